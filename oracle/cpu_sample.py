"""Bounded CPU sample of the reference algorithm (TEST/BASELINE INFRASTRUCTURE ONLY).

Times the oracle port on the BASELINE configuration's mesh restricted to its
first `slabs` time slabs: one Newton step's residual, Jacobian and P_T setup,
then `iters` GMRES(50) iterations (reference MGS, P_T^{-1} and J applies).
Every per-slab cost of the reference scales linearly with the slab count
(causal block structure), so callers extrapolate to the full Nt.
Prints one JSON line.  Run in a subprocess so thread env vars take effect.
"""

from __future__ import annotations

import argparse
import json
import os
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--slabs", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import numpy as np

    from oracle import configs, model, solvers

    c = configs.CONFIGS[args.config]
    prob = configs.baseline_problem(c["problem"], c["visc"])
    t0 = time.perf_counter()
    d = model.make_disc(prob, c["n"], c["dt"], args.slabs)
    t_disc = time.perf_counter() - t0
    st = model.initial_state(d)
    t0 = time.perf_counter()
    r = model.residual(st, d)
    t1 = time.perf_counter()
    jac = model.jacobian(st, d)
    t2 = time.perf_counter()
    pc = solvers.Precond(jac, d, st)
    t3 = time.perf_counter()
    # rel_tol 0: a timing sample runs exactly `iters` iterations (a prefix of a few slabs
    # would converge early and under-weight the growing MGS basis)
    res = solvers.gmres_mgs(jac.apply, pc.apply_inverse, -r, rel_tol=0.0, abs_tol=1e-300,
                            max_iters=100000, restart=50, max_total=args.iters)
    t4 = time.perf_counter()
    print(json.dumps(dict(config=args.config, slabs=args.slabs, iters=res.iterations,
                          t_disc=t_disc, t_residual=t1 - t0, t_jacobian=t2 - t1, t_pc_setup=t3 - t2,
                          t_gmres=t4 - t3, t_iter=(t4 - t3) / max(res.iterations, 1),
                          threads=os.environ.get("OMP_NUM_THREADS", "all"),
                          numpy=np.__version__)))


if __name__ == "__main__":
    main()
