"""Assembly timing: residual and assemble_jacobian (clamp + element-matrix patch
values + Alfven) per config, CUDA events; algorithmic bytes per SURVEY 8(d)."""
import argparse
import json

import torch

import paper_2309_00768_b200 as p


def timeit(fn, reps=10):
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
    ap.add_argument("--configs", default="C2,C3")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    for cfg in args.configs.split(","):
        d = p.discretize_config(cfg)
        st = p.initial_state(d)
        st.vec.data += 1e-3 * torch.randn_like(st.vec.data)
        r_ms = timeit(lambda: p.residual(st, d), args.reps)
        j_ms = timeit(lambda: p.assemble_jacobian(st, d), args.reps)
        L, P, nt = d.layout, d.pattern, d.n_steps
        res_b = nt * 8 * 2 * L.slab_size
        jac_b = nt * 8 * (P.nnz + P.fp_nnz)
        print(json.dumps({"config": cfg, "residual_ms": r_ms, "jacobian_ms": j_ms,
                          "assembly_GBps": (res_b + jac_b) / ((r_ms + j_ms) * 1e-3) / 1e9,
                          "jacobian_GBps": jac_b / (j_ms * 1e-3) / 1e9, "residual_GBps": res_b / (r_ms * 1e-3) / 1e9}),
              flush=True)


if __name__ == "__main__":
    main()
