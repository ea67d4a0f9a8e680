"""Per-kernel GPU time of one Newton solve (or one preconditioner setup + applies)
through the CUDA activity API (torch.profiler / CUPTI: every kernel of the
process, ours included).  Diagnostics only; numbers from a profiled run are never
bench values.

  python tools/kernel_summary.py C4_512 [--what solve|setup] [--out file.json]
"""
import argparse
import collections
import json

import torch
from torch.profiler import ProfilerActivity, profile

import paper_2309_00768_b200 as p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--what", default="solve", choices=["solve", "setup"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    d = p.discretize_config(args.config)
    _, _, _, _, rel = p.config_problem(args.config)
    cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=rel, max_iters=1 if rel is None else 25,
                         gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))
    st = p.initial_state(d)
    if args.what == "solve":
        p.solve_all_at_once(d, cfg)  # warm-up (plans, K, pools)
    else:
        jac = p.assemble_jacobian(st, d)
        p.SpaceTimePreconditioner(jac, d, st).apply_inverse(torch.zeros(jac.size, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        if args.what == "solve":
            _, stats = p.solve_all_at_once(d, cfg)
            info = {"gmres": stats.gmres_iters}
        else:
            jac = p.assemble_jacobian(st, d)
            pc = p.SpaceTimePreconditioner(jac, d, st)
            pc.apply_inverse(torch.zeros(jac.size, dtype=torch.float64, device="cuda"))
            info = {}
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.split("(")[0][:90]
            tot[k][0] += 1
            tot[k][1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    total = sum(v[1] for v in tot.values())
    rows = sorted(tot.items(), key=lambda kv: -kv[1][1])
    print(f"{args.config} {args.what} {info}: total GPU kernel time {total / 1e3:.1f} ms, {sum(v[0] for v in tot.values())} launches")
    for k, (n, t) in rows[:30]:
        print(f"{t / 1e3:10.2f} ms {100 * t / total:5.1f}% {n:7d}  {k}")
    if args.out:
        json.dump({"config": args.config, "what": args.what, "info": info, "total_ms": total / 1e3,
                   "kernels": [{"name": k, "count": n, "ms": t / 1e3} for k, (n, t) in rows]}, open(args.out, "w"),
                  indent=1)


if __name__ == "__main__":
    main()
