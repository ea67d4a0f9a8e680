"""Repeated P_T^{-1} applications on C2 (launch-list / trace target)."""
import sys
import torch
import paper_2309_00768_b200 as p

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d = p.discretize_config(cfg)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
v = torch.randn(d.n_steps * d.layout.slab_size, dtype=torch.float64, device="cuda")
out = torch.empty_like(v)
for _ in range(reps):
    pc._into(v, out)
torch.cuda.synchronize()
print("ok")
