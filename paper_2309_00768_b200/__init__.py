"""B200-native space-time Newton--FGMRES core for 2D resistive MHD.

Drop-in for the hot path of the reference package ``stmhd`` (arXiv
2309.00768): the same operator / preconditioner / GMRES API, backed by
hand-written sm_100a FP64 kernels behind the C-ABI in include/stmhd_b200.h.
"""

from .errors import (  # noqa: F401
    BreakdownError,
    ConfigurationError,
    ConvergenceError,
    CudaError,
    PreconditionerError,
    SingularMatrixError,
    StmhdError,
)
from .linalg import (  # noqa: F401
    BlockVector,
    FieldLayout,
    GmresConfig,
    GmresResult,
    LUFactor,
    gmres,
    lu_factor,
)
from .problems import (  # noqa: F401
    CONFIGS,
    BCKind,
    BCSpec,
    Condition,
    ProblemSpec,
    Side,
    dirichlet,
    enclosed_bcs,
    natural,
    slip,
    baseline_island,
    baseline_tearing,
    by_name,
    config_problem,
    island_coalescence,
    tearing_mode,
)
from .discretization import Discretization, discretize, discretize_config, initial_state  # noqa: F401
from .spacetime import (  # noqa: F401
    SlabBlocks,
    SpaceTimeJacobian,
    SpaceTimeState,
    apply_jacobian,
    assemble_jacobian,
    linearize_slab,
    residual,
)
from .precond import SpaceTimePreconditioner, Variant, compute_alfven_scaling  # noqa: F401
from .solver import (NewtonConfig, SolveStats, compute_overhead_ratios, solve_all_at_once,  # noqa: F401
                     solve_sequential)

__version__ = "0.1.0"
