"""B200-native space-time Newton--FGMRES core for 2D resistive MHD
(drop-in for the hot path of the reference package ``stmhd``)."""

from .errors import (  # noqa: F401
    BreakdownError,
    ConfigurationError,
    ConvergenceError,
    CudaError,
    PreconditionerError,
    SingularMatrixError,
    StmhdError,
)
from .linalg import BlockVector, FieldLayout, LUFactor, lu_factor  # noqa: F401

__version__ = "0.1.0"
