"""C3 (tearing 64^2, Nt=128, mu=eta=1e-3): first Newton step's FGMRES(50) with P_T run
for many iterations, relative residual every 50 (the stagnation finding of DESIGN 7)."""
import argparse
import json
import time

import torch

import paper_2309_00768_b200 as p

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3000)
ap.add_argument("--restart", type=int, default=50)
args = ap.parse_args()
d = p.discretize_config("C3")
st = p.initial_state(d)
r = p.residual(st, d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
torch.cuda.synchronize()
t = time.perf_counter()
res = p.gmres(jac.apply, pc.apply_inverse, -r.data,
              config=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=args.iters, restart=args.restart))
torch.cuda.synchronize()
wall = time.perf_counter() - t
rr = [x / res.residuals[0] for x in res.residuals]
print(json.dumps({"config": "C3 Newton step 1", "restart": args.restart, "iterations": res.iterations,
                  "converged": res.converged, "wall_s": wall, "ms_per_iteration": 1e3 * wall / max(res.iterations, 1),
                  "relative_residual_every_50": rr[::50] + [rr[-1]],
                  "true_residual_rel": res.true_residual / res.residuals[0]}))
