"""Configuration-5 operator microbenchmark (BASELINE configs[4]): the space-time
block-bidiagonal scalar advection-diffusion block on an n x n P1 mesh, Nt slabs;
times `spmv` batched block-bidiagonal SpMVs and `apply` exact inverse applications
(sequential sweep) with CUDA events.  Prints one JSON line."""

import argparse
import json
import time

import torch

from paper_2309_00768_b200.c5 import C5Operator


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--nt", type=int, default=1024)
    ap.add_argument("--spmv", type=int, default=100)
    ap.add_argument("--apply", type=int, default=20)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    t0 = time.perf_counter()
    op = C5Operator(args.n, args.nt, seed=args.seed)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    op.factor()
    torch.cuda.synchronize()
    t_factor = time.perf_counter() - t0
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(args.nt * op.n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty_like(x)
    op.apply(x, y)
    op.solve(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.spmv):
        op.apply(x, y)
    e1.record()
    e1.synchronize()
    spmv_ms = e0.elapsed_time(e1) / args.spmv
    e0.record()
    for _ in range(args.apply):
        op.solve(x, y)
    e1.record()
    e1.synchronize()
    solve_ms = e0.elapsed_time(e1) / args.apply
    # SpMV algorithmic bytes: per-slab values, x and y once, shared indices and coupling
    c = op.coupling
    # round trip F (F^{-1} x) = x on the full operator (size-independent parity check)
    op.solve(x, y)
    z = op.apply(y)
    round_trip = float(torch.linalg.norm(z - x) / torch.linalg.norm(x))
    spmv_bytes = (8 * args.nt * op.nnz + 2 * 8 * args.nt * op.n + 4 * op.nnz + 4 * (op.n + 1)
                  + 12 * c.nnz + 4 * (op.n + 1))
    peak = 6543.4
    info = op._lu.info()
    print(json.dumps({
        "config": f"C5 {args.n}x{args.n} P1 scalar, Nt={args.nt}, dt=1e-2, eps=1e-3",
        "unknowns": args.nt * op.n, "nnz_per_slab": op.nnz,
        "spmv_ms": spmv_ms, "spmv_GBps": spmv_bytes / (spmv_ms * 1e-3) / 1e9,
        "spmv_frac_of_hbm": spmv_bytes / (spmv_ms * 1e-3) / 1e9 / peak,
        "apply_inverse_ms": solve_ms, "apply_inverse_per_slab_us": 1e3 * solve_ms / args.nt,
        "factor_doubles_per_slab": info["factor_doubles"], "factor_GB": 8e-9 * info["factor_doubles"] * args.nt,
        "setup_s": {"host_tables_and_assembly": t_build, "factorisation": t_factor},
        "round_trip_rel": round_trip,
        "timed": f"{args.spmv} SpMVs, {args.apply} exact-inverse applications (CUDA events)"}))


if __name__ == "__main__":
    main()
