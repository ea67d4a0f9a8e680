"""Per-phase timing of one space-time Newton-FGMRES solve on the GPU."""
import argparse
import time

import torch

import paper_2309_00768_b200 as p


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--solve", type=int, default=1)
    ap.add_argument("--leaf", type=int, default=32)
    ap.add_argument("--leaf-fu", type=int, default=None)
    ap.add_argument("--leaf-ca", type=int, default=None)
    args = ap.parse_args()
    t0 = time.perf_counter()
    d = p.discretize_config(args.config, leaf={"fu": args.leaf_fu or args.leaf, "ca": args.leaf_ca or args.leaf,
                                               "const": args.leaf})
    torch.cuda.synchronize()
    print(f"discretize {time.perf_counter()-t0:.2f}s  device bytes {d.device_bytes()/1e9:.2f} GB  N={d.n_steps*d.layout.slab_size}")
    st = p.initial_state(d)
    r = p.residual(st, d)
    print("|r0|", r.norm())
    ms = timeit(lambda: p.residual(st, d))
    print(f"residual {ms:.3f} ms")
    jac = p.assemble_jacobian(st, d)
    print(f"assemble_jacobian {timeit(lambda: p.assemble_jacobian(st, d)):.3f} ms")
    t = time.perf_counter()
    pc = p.SpaceTimePreconditioner(jac, d, st)
    torch.cuda.synchronize()
    print(f"pc setup {1e3*(time.perf_counter()-t):.1f} ms")
    v = torch.randn(jac.size, dtype=torch.float64, device="cuda")
    out = torch.empty_like(v)
    print(f"J.apply {timeit(lambda: jac._into(v, out), 20):.3f} ms")
    print(f"P.apply_inverse {timeit(lambda: pc._into(v, out), 5):.3f} ms")
    L = d.layout
    nt = d.n_steps
    vu = torch.randn(nt * L.n_u, dtype=torch.float64, device="cuda")
    va = torch.randn(nt * L.n_a, dtype=torch.float64, device="cuda")
    vp = torch.randn(nt * L.n_p, dtype=torch.float64, device="cuda")
    print(f"  solve_velocity {timeit(lambda: pc.solve_velocity(vu), 5):.3f} ms")
    print(f"  solve_wave {timeit(lambda: pc.solve_wave(va), 5):.3f} ms")
    print(f"  magnetic_schur_inverse {timeit(lambda: pc.magnetic_schur_inverse(va), 5):.3f} ms")
    print(f"  pressure_schur_inverse {timeit(lambda: pc.pressure_schur_inverse(vp), 5):.3f} ms")
    if args.solve:
        _, _, _, _, rel = p.config_problem(args.config)
        cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=rel, max_iters=1 if rel is None else 25,
                             gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))
        t = time.perf_counter()
        state, stats = p.solve_all_at_once(d, cfg)
        print(f"solve {time.perf_counter()-t:.2f}s newton {stats.newton_iters} gmres {stats.gmres_iters} "
              f"res {stats.residual_norms} timings {stats.timings}")


if __name__ == "__main__":
    main()
