"""Golden fixtures for the sequential driver and the single-step preconditioner,
generated from the UNMODIFIED reference package ``stmhd`` (build container only:
``python tests/golden/make_golden_seq.py``; the reference is imported read-only
from /root/reference/pkg/src).

  seq_tearing.npz   tearing_mode dx=0.25, dt=0.5, T=1: solve_sequential and
                    solve_all_at_once (default NewtonConfig) -> states, per-step
                    Newton / GMRES counts, overhead ratios
  seq_frozen.npz    island_coalescence eps=0, dx=0.5, dt=0.25, T=1: frozen steps
  seq_single.npz    island_coalescence dx=0.5, dt=0.5, T=1 at the initial guess:
                    single-step P_k^{-1} x and P_k x for k = 0, 1
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import stmhd  # noqa: E402
from stmhd.precond import SpaceTimePreconditioner  # noqa: E402
from stmhd.solver import compute_overhead_ratios  # noqa: E402
from stmhd.spacetime import assemble_jacobian  # noqa: E402


def main():
    disc = stmhd.discretize(stmhd.by_name("tearing_mode"), 0.25, 0.5, 1.0)
    seq_state, seq = stmhd.solve_sequential(disc)
    st_state, st = stmhd.solve_all_at_once(disc)
    nr, gr = compute_overhead_ratios(st, seq)
    np.savez_compressed(
        os.path.join(HERE, "seq_tearing.npz"),
        seq_x=seq_state.vec.data, st_x=st_state.vec.data,
        seq_newton=np.array(seq.per_step_newton),
        seq_gmres=np.array([g for gs in seq.per_step_gmres for g in gs]),
        seq_gmres_ptr=np.cumsum([0] + [len(g) for g in seq.per_step_gmres]),
        st_newton=st.newton_iters, st_gmres=np.array(st.gmres_iters), ratios=np.array([nr, gr]))
    print("seq_tearing", seq.per_step_newton, seq.per_step_gmres, st.newton_iters, st.gmres_iters, nr, gr)

    disc = stmhd.discretize(stmhd.by_name("island_coalescence", eps=0.0), 0.5, 0.25, 1.0)
    _, seq = stmhd.solve_sequential(disc)
    np.savez_compressed(os.path.join(HERE, "seq_frozen.npz"), frozen=np.array(seq.frozen_steps),
                        seq_newton=np.array(seq.per_step_newton))
    print("seq_frozen", seq.frozen_steps, seq.per_step_newton)

    disc = stmhd.discretize(stmhd.by_name("island_coalescence"), 0.5, 0.5, 1.0)
    state = stmhd.initial_state(disc)
    jac = assemble_jacobian(state, disc)
    prec = SpaceTimePreconditioner(jac, disc, state)
    rng = np.random.default_rng(11)
    out = {"state": state.vec.data, "ic_u": state.ic_u, "ic_a": state.ic_a}
    for k in range(disc.n_steps):
        x = rng.standard_normal(disc.layout.slab_size)
        out[f"x{k}"] = x
        out[f"inv{k}"] = prec.apply_single_step_inverse(k, x)
        out[f"fwd{k}"] = prec.apply_single_step(k, x)
    np.savez_compressed(os.path.join(HERE, "seq_single.npz"), **out)
    print("seq_single ok", disc.n_steps)


if __name__ == "__main__":
    main()
