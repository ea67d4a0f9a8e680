"""Capped FGMRES run on a config's first Newton step, printing progress."""
import sys
import time

import torch

import paper_2309_00768_b200 as p

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 600
d = p.discretize_config(cfg_name)
st = p.initial_state(d)
r = p.residual(st, d).data
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
t = time.perf_counter()
res = p.gmres(jac.apply, pc.apply_inverse, -r, config=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=cap, restart=50))
dt = time.perf_counter() - t
rs = res.residuals
print(f"{cfg_name}: {res.iterations} its in {dt:.1f}s ({1e3*dt/max(res.iterations,1):.1f} ms/it), converged={res.converged}")
for i in range(0, len(rs), 50):
    print(i, f"{rs[i]/rs[0]:.3e}")
print("final", f"{rs[-1]/rs[0]:.3e}", "true", res.true_residual / rs[0])
