"""Run the velocity sweep of config C2 a few times (ncu target)."""
import sys
import torch
import paper_2309_00768_b200 as p

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
d = p.discretize_config(cfg)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
vu = torch.randn(d.n_steps * d.layout.n_u, dtype=torch.float64, device="cuda")
for _ in range(3):
    pc.solve_velocity(vu)
torch.cuda.synchronize()
print("ok")
