"""Per-step trace of the sweeps at one configuration (diagnostics).  Run once plain
(timings), then with STMHD_SWEEP_TRACE=1 (slab 1's step durations of the traced
stage) or STMHD_SWEEP_PROF=1 (per-warp counters + CTA 0 timeline):
  python tools/trace_probe.py C4_64 [stage] [what]
stage: traced stage of the pipelined P_T^-1 (0 wave, 1 M_j, 2 velocity);
what: 'both' (solve_velocity and apply_inverse, default) or 'pinv'.
"""
import os
import sys

stage = sys.argv[2] if len(sys.argv) > 2 else "2"
what = sys.argv[3] if len(sys.argv) > 3 else "both"
os.environ.setdefault("STMHD_SWEEP_PLAN_INFO", "1")
os.environ["STMHD_SWEEP_TRACE_STAGE"] = stage
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_00768_b200 as p  # noqa: E402

cfg = sys.argv[1]
d = p.discretize_config(cfg)
st = p.initial_state(d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=g)
L = d.layout
vu = v[: d.n_steps * L.n_u].clone()
out = torch.empty_like(v)


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


msg = f"{cfg}: apply_inverse {tm(lambda: pc._into(v, out)):.3f} ms"
if what == "both":
    msg += f", solve_velocity {tm(lambda: pc.solve_velocity(vu)):.3f} ms"
print(msg + f", jac {tm(lambda: jac._into(v, out)):.3f} ms", flush=True)
