"""Small 64^2 runs of the production sweep paths (sanitizer / debugging target):
tearing 64^2, mu=eta=1e-3, dt=0.02, NT slabs (default 3): P_T setup, solve_velocity,
apply_inverse, J.v.  python tools/prefix_probe.py [nt]"""
import sys

import torch

import paper_2309_00768_b200 as p

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 3
d = p.discretize(p.baseline_tearing(1e-3), 2.0 / 64, 0.02, nt * 0.02)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
x = pc.solve_velocity(v[: nt * d.layout.n_u])
y = pc.apply_inverse(v)
z = jac.apply(v)
torch.cuda.synchronize()
print("ok", float(x.norm()), float(y.norm()), float(z.norm()))
