"""Full Newton-FGMRES solve of a custom BASELINE-physics grid (progress printed)."""
import argparse
import time

import paper_2309_00768_b200 as p

ap = argparse.ArgumentParser()
ap.add_argument("--problem", default="tearing")
ap.add_argument("--n", type=int, default=32)
ap.add_argument("--dt", type=float, default=0.02)
ap.add_argument("--nt", type=int, default=16)
ap.add_argument("--visc", type=float, default=None)
ap.add_argument("--rel", type=float, default=1e-6)
ap.add_argument("--maxit", type=int, default=3000)
a = ap.parse_args()
visc = a.visc if a.visc is not None else (1e-3 if a.problem == "tearing" else 1e-2)
prob = p.baseline_tearing(visc) if a.problem == "tearing" else p.baseline_island(visc)
d = p.discretize(prob, 2.0 / a.n, a.dt, a.nt * a.dt)
cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=a.rel, max_iters=6,
                     gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=a.maxit, restart=50))
t = time.perf_counter()
st, stats = p.solve_all_at_once(d, cfg)
r = stats.residual_norms
print(f"{a.problem} n={a.n} dt={a.dt} nt={a.nt}: newton {stats.newton_iters} gmres {stats.gmres_iters} "
      f"rel {[f'{x/r[0]:.2e}' for x in r]} time {time.perf_counter()-t:.1f}s", flush=True)
