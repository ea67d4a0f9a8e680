"""Run every preconditioner sweep of a configuration once (trace/profile target)."""
import sys
import torch
import paper_2309_00768_b200 as p

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
d = p.discretize_config(cfg)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
L = d.layout
for name, nloc in (("solve_velocity", L.n_u), ("solve_wave", L.n_a), ("magnetic_schur_inverse", L.n_a),
                   ("pressure_schur_inverse", L.n_p)):
    v = torch.randn(d.n_steps * nloc, dtype=torch.float64, device="cuda")
    for _ in range(2):
        getattr(pc, name)(v)
    torch.cuda.synchronize()
    print("done", name, flush=True)
