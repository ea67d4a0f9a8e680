"""Preconditioner setup split at one configuration (device-synchronised wall times):
assembly, SpaceTimePreconditioner() (factorisations + C~_A), the first P_T^-1 apply
(dense-top K build + coupling gathers), and a steady-state apply.
  python tools/setup_probe.py C4_512
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_00768_b200 as p  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4_64"
d = p.discretize_config(cfg)
st = p.initial_state(d)


def wall(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


for rep in range(2):
    jac, t_j = wall(lambda: p.assemble_jacobian(st, d))
    pc, t_pc = wall(lambda: p.SpaceTimePreconditioner(jac, d, st))
    v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    _, t_first = wall(lambda: pc._into(v, out))
    _, t_second = wall(lambda: pc._into(v, out))
    _, t_jv = wall(lambda: jac._into(v, out))
    print(f"{cfg} rep {rep}: jacobian {t_j * 1e3:.1f} ms, pc setup {t_pc * 1e3:.1f} ms, first apply "
          f"{t_first * 1e3:.1f} ms, second apply {t_second * 1e3:.1f} ms, J.v {t_jv * 1e3:.2f} ms", flush=True)
    del pc, jac
