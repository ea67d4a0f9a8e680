"""Golden fixture for the reference-shaped problem intake (ProblemSpec with its own
``bcs: BCSpec`` and ``a_eq_normal_flux_top``), generated from the UNMODIFIED
reference package ``stmhd`` (build container only; ``python
tests/golden/make_golden_bcs.py``).

The problem is NOT one of the reference's built-ins: it uses the island
coalescence closures with a boundary specification the built-ins never exercise --
a Dirichlet (lid-driven) velocity pair on the top side, slip on the other three,
and a Dirichlet potential on the top AND left sides (natural elsewhere).  Written
with the reference's own record and BC vocabulary (problems.py:25-47,
fem.py:478-529), P3/P2, dx=0.25, dt=0.5, T=1 (2 slabs).

  ref_bcs.npz  u/A constrained DOFs + values, current_flux, initial state,
               residual at a perturbed state, J.v, P_T^-1 v (TRIANGULAR), and the
               GMRES(50) rel 1e-8 iteration count of the first Newton step
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import stmhd  # noqa: E402
from stmhd.fem import BCSpec, dirichlet, natural, slip  # noqa: E402
from stmhd.linalg import BlockVector, GmresConfig, gmres  # noqa: E402
from stmhd.mesh import Side  # noqa: E402
from stmhd.precond import SpaceTimePreconditioner  # noqa: E402
from stmhd.problems import ProblemSpec  # noqa: E402
from stmhd.spacetime import SpaceTimeState, assemble_jacobian, residual  # noqa: E402


def lid_problem():
    """Island closures (reference problems.py:96-127 with beta=0.2, mu=eta=0.1) and
    a custom BCSpec."""
    ref = stmhd.by_name("island_coalescence", mu=0.1, eta=0.1)

    def lid_x(x, y):
        return 0.05 * np.sin(np.pi * x) + 0.0 * y

    def lid_y(x, y):
        return 0.0 * x

    bcs = BCSpec(conditions={
        "u": {Side.LEFT: slip(), Side.RIGHT: slip(), Side.BOTTOM: slip(),
              Side.TOP: dirichlet((lid_x, lid_y))},
        "p": {s: natural() for s in Side},
        "j": {s: natural() for s in Side},
        "A": {Side.LEFT: dirichlet(ref.a_eq), Side.RIGHT: natural(), Side.BOTTOM: natural(),
              Side.TOP: dirichlet(ref.a_eq)},
    })
    return ProblemSpec(name="island_lid", domain=ref.domain, mu=ref.mu, eta=ref.eta, mu0=ref.mu0,
                       eps=ref.eps, a_eq=ref.a_eq, e_eq=ref.e_eq, p_eq=ref.p_eq,
                       a_perturbation=ref.a_perturbation,
                       a_eq_normal_flux_top=ref.a_eq_normal_flux_top, bcs=bcs)


def main():
    disc = stmhd.discretize(lid_problem(), 0.25, 0.5, 1.0)
    st0 = stmhd.initial_state(disc)
    rng = np.random.default_rng(5)
    x = st0.vec.data + 1e-3 * rng.standard_normal(st0.vec.data.size)
    v = rng.standard_normal(x.size)
    st = SpaceTimeState(vec=BlockVector(disc.layout, disc.n_steps, x.copy()), ic_u=st0.ic_u, ic_a=st0.ic_a)
    r = residual(st, disc).data
    jac = assemble_jacobian(st, disc)
    pc = SpaceTimePreconditioner(jac, disc, st)
    jv = jac.apply(v)
    pv = pc.apply_inverse(v)
    # first Newton step from the initial state
    r0 = residual(st0, disc).data
    jac0 = assemble_jacobian(st0, disc)
    pc0 = SpaceTimePreconditioner(jac0, disc, st0)
    res = gmres(jac0.apply, pc0.apply_inverse, -r0,
                config=GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=1000, restart=50))
    np.savez_compressed(
        os.path.join(HERE, "ref_bcs.npz"),
        u_bc_idx=disc.u_bc_idx, u_bc_vals=disc.u_bc_vals, a_bc_idx=disc.a_bc_idx,
        a_bc_vals=disc.a_bc_vals, current_flux=disc.current_flux, state0=st0.vec.data,
        ic_u=st0.ic_u, ic_a=st0.ic_a, x=x, v=v, r=r, Jv=jv, Pv=pv, r0=r0,
        gmres_iters=res.iterations, gmres_x=res.x)
    print("ref_bcs ok", disc.layout.slab_size, disc.n_steps, res.iterations)


if __name__ == "__main__":
    main()
