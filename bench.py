#!/usr/bin/env python
"""Benchmark: space-time Newton--FGMRES solve of BASELINE config C2 on B200.

Metric (BASELINE.json): preconditioned FGMRES iterations per second over a full
Newton solve (FP64), plus the Newton solve time.  One "step" = one complete
all-at-once solve of configuration C2 (island coalescence, 32x32 P2/P1,
dt=0.05, Nt=64; Newton to relative residual 1e-6, FGMRES(50) rel 1e-8, P_T
preconditioner) from the equilibrium-projection initial state.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun, one rank per GPU): the space-time sweeps do not shard
(SURVEY 8(e)), so every rank solves an independent replica; value = all
ranks' iterations / max-over-ranks device time ("scaling": "weak").

`--impl reference` times the reference algorithm on the host CPU through the
oracle port (oracle/, the reference is pure Python): a bounded sample (C2 mesh,
first 8 slabs, one Newton linearisation + one 50-iteration FGMRES cycle) per
step, extrapolated linearly in the slab count to the full C2 solve with the
reference's own iteration counts (458 + 413).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "C2"
# Reference iteration counts for C2 (Newton steps 1,2); the oracle and the GPU
# path both reproduce them (tests).
REF_GMRES = [458, 413]
SAMPLE_SLABS, SAMPLE_ITERS = 8, 50


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3-kernels", action="store_true", help="skip the C3 J.v / assembly roofline entries")
    return ap.parse_args()


# ---------------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "500"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(threads_one=True):
    """One bounded oracle sample in a subprocess (so thread env vars apply)."""
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    cmd = [sys.executable, "-m", "oracle.cpu_sample", "--config", CONFIG, "--slabs", str(SAMPLE_SLABS),
           "--iters", str(SAMPLE_ITERS)]
    if threads_one:
        env.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        if shutil_which("taskset"):
            cmd = ["taskset", "-c", "0"] + cmd
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        raise RuntimeError("cpu sample failed: " + out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def shutil_which(name):
    import shutil

    return shutil.which(name)


def extrapolate(sample, nt_full, gmres_iters):
    """Full-solve CPU time from a slab-prefix sample (linear in the slab count)."""
    scale = nt_full / sample["slabs"]
    newton = len(gmres_iters)
    t = scale * ((newton + 1) * sample["t_residual"] + newton * (sample["t_jacobian"] + sample["t_pc_setup"])
                 + sum(gmres_iters) * sample["t_iter"])
    return t, sum(gmres_iters) / t


# ---------------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy  # noqa: F401  (threads: all the host threads it can use)

    times = []
    sample = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        sample = cpu_sample(threads_one=False)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append((dt, sample))
    samples = [s for _, s in times]
    t_iter = statistics.median(s["t_iter"] for s in samples)
    agg = dict(samples[-1])
    agg["t_iter"] = t_iter
    for k in ("t_residual", "t_jacobian", "t_pc_setup"):
        agg[k] = statistics.median(s[k] for s in samples)
    t_full, value = extrapolate(agg, 64, REF_GMRES)
    cores = os.cpu_count()
    line = {
        "impl": "reference",
        "metric": "FGMRES iterations/s (C2 Newton solve, P_T preconditioner, FP64)",
        "value": value, "unit": "FGMRES it/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(t for t, _ in times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE C2 analytic problem)",
        "config": {"workload": "C2 island coalescence 32x32 P2/P1, dt=0.05, Nt=64, Newton rel 1e-6, FGMRES(50) rel 1e-8",
                   "l2": "n/a (CPU)"},
        "newton_solve_s_extrapolated": t_full,
        "cpu_baseline": {"value": value, "unit": "FGMRES it/s", "cores": cores, "kind": "port",
                         "sample": f"oracle port (reference algorithm: SuperLU P_T, MGS GMRES) on C2 mesh, first "
                                   f"{SAMPLE_SLABS} of 64 slabs: 1 residual+Jacobian+P_T setup and "
                                   f"{SAMPLE_ITERS} FGMRES iterations per step; extrapolated x{64 // SAMPLE_SLABS} "
                                   f"to the full solve with the reference counts {REF_GMRES}"},
        "e2e": {"value": value, "unit": "FGMRES it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------
def run_ours(args, rank, world):
    import numpy as np
    import scipy.sparse.linalg as spla
    import torch
    import torch.distributed as dist

    import paper_2309_00768_b200 as p
    from paper_2309_00768_b200 import _lib

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    lib = _lib.load()
    disc = p.discretize_config(CONFIG)
    _, _, _, nt, rel = p.config_problem(CONFIG)
    cfg = p.NewtonConfig(abs_tol=1e-300, rel_tol=rel, max_iters=25,
                         gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))
    st0 = p.initial_state(disc)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # > L2 (126 MB)

    def barrier():
        if world > 1:
            dist.barrier()

    def solve_once(state=None):
        st = state if state is not None else p.SpaceTimeState(st0.vec.copy(), st0.ic_u.clone(), st0.ic_a.clone())
        return p.solve_all_at_once(disc, cfg, state=st)

    for _ in range(args.warmup):
        solve_once()
    torch.cuda.synchronize()

    # ---- device-resident timed region ----
    clocks = Clocks(dev.index)
    iters, ms, breakdown = 0, [], {}
    barrier()
    torch.cuda.synchronize()
    launches0 = int(lib.stmhd_launch_count())
    clocks.start()
    stats_last = None
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (untimed)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, stats = solve_once()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        iters += stats.total_gmres
        for k, v in stats.timings.items():
            breakdown[k] = breakdown.get(k, 0.0) + v
        stats_last = stats
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = int(lib.stmhd_launch_count()) - launches0
    barrier()
    from paper_2309_00768_b200.replicas import aggregate

    total_s, iters_all = aggregate(sum(ms) / 1e3, iters, dev)
    value = iters_all / total_s

    # ---- e2e through the public API with host buffers ----
    h_state = st0.vec.data.cpu().pin_memory()
    h_icu, h_ica = st0.ic_u.cpu().pin_memory(), st0.ic_a.cpu().pin_memory()
    h_out = torch.empty_like(h_state).pin_memory()
    e2e_ms, e2e_iters = [], 0
    barrier()
    clocks2 = Clocks(dev.index)  # same sampler load as the device-resident region
    clocks2.start()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        vec = h_state.to(dev, non_blocking=True)
        icu, ica = h_icu.to(dev, non_blocking=True), h_ica.to(dev, non_blocking=True)
        state = p.SpaceTimeState(p.BlockVector(disc.layout, disc.n_steps, vec), icu, ica)
        state, stats = solve_once(state)
        h_out.copy_(state.vec.data, non_blocking=True)
        e1.record()
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        e2e_iters += stats.total_gmres
    clocks2.stop()
    e2e_s, e2e_iters = aggregate(sum(e2e_ms) / 1e3, e2e_iters, dev)
    e2e_value = e2e_iters / e2e_s
    h2d = (h_state.numel() + h_icu.numel() + h_ica.numel()) * 8
    d2h = h_out.numel() * 8

    # ---- roofline of the dominant kernel: the F_u time sweep (nd_solve_kernel) ----
    jac = p.assemble_jacobian(st0, disc)
    pc = p.SpaceTimePreconditioner(jac, disc, st0)
    L = disc.layout
    vu = torch.randn(nt * L.n_u, dtype=torch.float64, device=dev)
    pc.solve_velocity(vu)
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pc.solve_velocity(vu)
    e1.record()
    e1.synchronize()
    sweep_ms = e0.elapsed_time(e1) / reps
    # algorithmic bytes use the structural fill: factor slab 0 at a perturbed state
    # (at u = 0 scipy drops the vanishing cross-component entries)
    stp = p.SpaceTimeState(st0.vec.copy(), st0.ic_u, st0.ic_a)
    stp.vec.data += 1e-3 * torch.randn(stp.vec.data.shape, dtype=torch.float64, device=dev,
                                       generator=torch.Generator(device=dev).manual_seed(0))
    f_u0 = p.assemble_jacobian(stp, disc).slabs[0].f_u.tocsc()
    lu = spla.splu(f_u0)
    fill = int(lu.L.nnz + lu.U.nnz)  # reference SuperLU (COLAMD) fill, SURVEY 8(d)
    nnz_mu = disc.mass_u_dt_bc.nnz
    sweep_bytes = nt * 8 * fill + 12 * nnz_mu + 16 * nt * L.n_u
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = sweep_bytes / (sweep_ms / 1e3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "sweep_traffic.json")))
        if prof.get("config") == CONFIG:
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    # per-iteration operator costs
    v = torch.randn(jac.size, dtype=torch.float64, device=dev)
    out = torch.empty_like(v)

    def tmeas(fn, r=10):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(r):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / r

    per_iter = {"J_apply_ms": tmeas(lambda: jac._into(v, out), 50),
                "P_apply_ms": tmeas(lambda: pc._into(v, out), 5),
                "assembly_ms": tmeas(lambda: p.assemble_jacobian(st0, disc), 5),
                "residual_ms": tmeas(lambda: p.residual(st0, disc), 5)}
    # the other north-star kernels against the same peak (SURVEY 8(d) algorithmic bytes)
    P_ = disc.pattern
    jv_bytes = nt * (8 * P_.nnz + 16 * L.slab_size) + 12 * disc.jc_nnz + 8 * L.n_p + 4 * P_.nnz
    asm_bytes = nt * 8 * (2 * L.slab_size + P_.nnz + P_.fp_nnz)
    asm_ms = per_iter["assembly_ms"] + per_iter["residual_ms"]
    kernel_rooflines = {
        "J_apply (sell_spmv_kernel)": {"algorithmic_bytes": jv_bytes, "ms": per_iter["J_apply_ms"],
                                       "GBps": jv_bytes / per_iter["J_apply_ms"] / 1e6,
                                       "frac": jv_bytes / per_iter["J_apply_ms"] / 1e6 / peak},
        "assembly (residual_patch + values_patch)": {"algorithmic_bytes": asm_bytes, "ms": asm_ms,
                                                     "GBps": asm_bytes / asm_ms / 1e6,
                                                     "frac": asm_bytes / asm_ms / 1e6 / peak},
        "note": "C2 operators are partly L2-resident (168 MB); the C3 entries are measured in this run after "
                "the timed region; tools/bench_spmv.py and tools/asm_probe.py give the C5 figures"}

    # the same kernels at C3 (tearing 64^2, Nt=128: 1.37 GB per J.v, beyond L2)
    if rank == 0 and not args.no_c3_kernels:
        try:
            d3 = p.discretize_config("C3")
            s3 = p.initial_state(d3)
            j3 = p.assemble_jacobian(s3, d3)
            v3 = torch.randn(j3.size, dtype=torch.float64, device=dev)
            o3 = torch.empty_like(v3)
            L3, P3, nt3 = d3.layout, d3.pattern, d3.n_steps
            jv3 = tmeas(lambda: j3._into(v3, o3), 30)
            as3 = tmeas(lambda: p.assemble_jacobian(s3, d3), 5) + tmeas(lambda: p.residual(s3, d3), 5)
            jb3 = nt3 * (8 * P3.nnz + 16 * L3.slab_size) + 12 * d3.jc_nnz + 8 * L3.n_p + 4 * P3.nnz
            ab3 = nt3 * 8 * (2 * L3.slab_size + P3.nnz + P3.fp_nnz)
            kernel_rooflines["C3"] = {
                "J_apply (sell_spmv_kernel)": {"algorithmic_bytes": jb3, "ms": jv3, "GBps": jb3 / jv3 / 1e6,
                                               "frac": jb3 / jv3 / 1e6 / peak},
                "assembly (residual_patch + values_patch)": {"algorithmic_bytes": ab3, "ms": as3,
                                                             "GBps": ab3 / as3 / 1e6, "frac": ab3 / as3 / 1e6 / peak}}
            del d3, s3, j3, v3, o3
            torch.cuda.empty_cache()
        except Exception as exc:  # keep the line
            kernel_rooflines["C3"] = {"error": str(exc)[:200]}

    line = {
        "metric": "FGMRES iterations/s (C2 Newton solve, P_T preconditioner, FP64)",
        "value": value, "unit": "FGMRES it/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE C2 analytic problem, equilibrium initial state)",
        "config": {"workload": "C2 island coalescence 32x32 P2/P1, dt=0.05, Nt=64, Newton rel 1e-6, FGMRES(50) rel 1e-8",
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "512 MB flush between timed solves; per-solve factors 0.6 GB > L2"},
        "newton_solve_s": total_s / args.steps,
        "newton_steps": stats_last.newton_iters, "fgmres_iters": stats_last.gmres_iters,
        "relative_residual": stats_last.residual_norms[-1] / stats_last.residual_norms[0],
        "phase_s_per_solve": {k: v / args.steps for k, v in breakdown.items()},
        "per_call_ms": per_iter,
        "kernel_rooflines": kernel_rooflines,
        "e2e": {"value": e2e_value, "unit": "FGMRES it/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": {"kernel": "nd_sweep_kernel (F_u time sweep, solve_velocity)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes_per_launch": sweep_bytes,
                     "launch_ms": sweep_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            smp = cpu_sample(threads_one=True)
            t_full, cv = extrapolate(smp, nt, stats_last.gmres_iters)
            line["cpu_baseline"] = {
                "value": cv, "unit": "FGMRES it/s", "cores": 1, "kind": "port",
                "sample": f"oracle port (SuperLU P_T + MGS GMRES, 1 pinned core) on C2 mesh, first {SAMPLE_SLABS} "
                          f"of {nt} slabs: residual+Jacobian+P_T setup + {SAMPLE_ITERS} FGMRES iterations; "
                          f"extrapolated x{nt // SAMPLE_SLABS} with this run's counts {stats_last.gmres_iters} "
                          f"-> {t_full:.0f} s per solve"}
        except Exception as exc:  # keep the GPU line even if the CPU sample fails
            line["cpu_baseline"] = {"value": None, "unit": "FGMRES it/s", "cores": 1, "kind": "port",
                                    "sample": f"failed: {exc}"[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group(backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
