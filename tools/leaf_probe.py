"""P_T^-1 / solve_velocity time for several nested-dissection leaf sizes of the
velocity factor (diagnostics):  python tools/leaf_probe.py C4_64 24 32 48"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_00768_b200 as p  # noqa: E402


def tm(fn, r=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(r):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / r


cfg = sys.argv[1]
for leaf in [int(x) for x in sys.argv[2:]]:
    d = p.discretize_config(cfg, leaf={"fu": leaf})
    st = p.initial_state(d)
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    print(f"{cfg} leaf {leaf}: apply_inverse {tm(lambda: pc._into(v, out)):.3f} ms", flush=True)
    del pc, jac, d
