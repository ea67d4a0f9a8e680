"""CPU oracle for the space-time Newton--FGMRES hot path (TEST INFRASTRUCTURE ONLY).

This package is a numpy/scipy restatement of the reference package ``stmhd``
(arXiv 2309.00768, mounted read-only at /root/reference during development)
restricted to the hot path listed in SURVEY.md section 8:

* finite-element spaces, quadrature and state-dependent assembly
  (reference ``pkg/src/stmhd/fem.py``),
* the space-time residual, Jacobian blocks and matvec
  (``pkg/src/stmhd/spacetime.py``),
* the block upper-triangular preconditioner P_T with SuperLU exact solves and
  sequential time sweeps (``pkg/src/stmhd/precond.py``),
* restarted right-preconditioned MGS GMRES and the Newton driver
  (``pkg/src/stmhd/linalg.py``, ``pkg/src/stmhd/solver.py``),
* the configuration-5 scalar advection-diffusion operator.

It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_2309_00768_b200``) never imports this package.

Parity pin: the oracle is checked against golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py`` imports
/root/reference/pkg/src/stmhd in the build container and writes
``tests/golden/*.npz``); ``tests/test_oracle_golden.py`` asserts agreement.
"""

from .configs import CONFIGS, baseline_problem, reference_problem, ProblemSpec  # noqa: F401
from .fe import Mesh, Space, rect_mesh  # noqa: F401
from .model import Disc, State, make_disc, initial_state, residual, jacobian, Jacobian  # noqa: F401
from .solvers import Precond, gmres_mgs, newton_solve  # noqa: F401
