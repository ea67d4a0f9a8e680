"""Time repeated preconditioner construction (factorisations + allocations)."""
import sys
import time
import torch
import paper_2309_00768_b200 as p

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
d = p.discretize_config(cfg)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pcs = []
for i in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    pc = p.SpaceTimePreconditioner(jac, d, st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    v = torch.randn(d.n_steps * d.layout.slab_size, dtype=torch.float64, device="cuda")
    pc.apply_inverse(v)  # forward factors (F_A, F_p) are created lazily
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"pc {i}: create {1e3 * (t1 - t):.1f} ms  first apply {1e3 * (t2 - t1):.1f} ms", flush=True)
    pcs = [pc]  # keep one alive (as Newton does while building the next)
