"""Batched space-time SpMV microbenchmark: J.v (stmhd_jac_apply) at C2/C3 and the
configuration-5 block-bidiagonal operator (stmhd_spmv_apply), CUDA-event timed,
algorithmic bytes per SURVEY 8(d).  One JSON line per operator."""
import argparse
import json

import torch

import paper_2309_00768_b200 as p
from paper_2309_00768_b200.c5 import C5Operator

PEAK = 6534.5


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C5")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    for cfg in args.configs.split(","):
        if cfg == "C5":
            op = C5Operator(256, 1024, seed=0)
            x = torch.randn(op.nt * op.n, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            ms = timeit(lambda: op.apply(x, y), args.reps)
            c = op.coupling
            byt = 8 * op.nt * op.nnz + 16 * op.nt * op.n + 4 * op.nnz + 12 * c.nnz
            name, unk = "C5 bidiagonal F_k/-M/dt", op.nt * op.n
        else:
            d = p.discretize_config(cfg)
            st = p.initial_state(d)
            jac = p.assemble_jacobian(st, d)
            v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
            out = torch.empty_like(v)
            ms = timeit(lambda: jac._into(v, out), args.reps)
            L = d.layout
            nnz = d.pattern.nnz
            byt = d.n_steps * (8 * nnz + 16 * L.slab_size) + 12 * d.jc_nnz + 8 * L.n_p + 4 * nnz
            name, unk = f"{cfg} J.v", jac.size
        gbs = byt / (ms * 1e-3) / 1e9
        print(json.dumps({"op": name, "unknowns": unk, "ms": ms, "algorithmic_GB": byt / 1e9, "GBps": gbs,
                          "frac_of_hbm": gbs / PEAK}), flush=True)


if __name__ == "__main__":
    main()
