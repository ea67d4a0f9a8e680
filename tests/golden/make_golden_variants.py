"""Golden vectors of the three P_T variants (TRIANGULAR / SIMPLIFIED / FULL),
inverse and forward application, from the UNMODIFIED reference ``stmhd``
(build container only: ``python tests/golden/make_golden_variants.py``).

  variants_island.npz   island_coalescence dx=0.5, dt=0.5, T=1 at the initial guess
  variants_tearing.npz  tearing_mode dx=0.25, dt=0.5, T=1 at the initial guess
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import stmhd  # noqa: E402
from stmhd.precond import SpaceTimePreconditioner, Variant  # noqa: E402
from stmhd.spacetime import assemble_jacobian  # noqa: E402


def main():
    for name, prob, dx in (("island", "island_coalescence", 0.5), ("tearing", "tearing_mode", 0.25)):
        disc = stmhd.discretize(stmhd.by_name(prob), dx, 0.5, 1.0)
        state = stmhd.initial_state(disc)
        jac = assemble_jacobian(state, disc)
        x = np.random.default_rng(21).standard_normal(jac.size)
        out = {"state": state.vec.data, "ic_u": state.ic_u, "ic_a": state.ic_a, "x": x}
        for v in Variant:
            prec = SpaceTimePreconditioner(jac, disc, state, v)
            out[f"inv_{v.value}"] = prec.apply_inverse(x.copy())
            out[f"fwd_{v.value}"] = prec.apply_forward(x.copy())
        np.savez_compressed(os.path.join(HERE, f"variants_{name}.npz"), **out)
        print(name, jac.size)


if __name__ == "__main__":
    main()
