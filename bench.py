#!/usr/bin/env python
"""Benchmark: space-time Newton--FGMRES solve of BASELINE config C4 at Nt=512 on B200.

Metric (BASELINE.json): preconditioned FGMRES iterations per second over a full
Newton solve (FP64), plus the Newton solve time.  The N=1 workload is the largest
single-GPU Newton--FGMRES configuration of BASELINE.json: C4 at Nt=512
-- island coalescence on a 64x64 P2/P1 mesh, T=1, dt=1/512 (23.5 M unknowns),
Newton to relative residual 1e-6, FGMRES(50) rel 1e-8, P_T preconditioner, from the
equilibrium-projection initial state.  One "step" = one complete solve.

Every timed step copies the initial state from pinned host memory to the device,
solves, and reads the solution back; CUDA events split the step into the copy-in,
the device-resident solve (`value`) and the copy-out (`e2e` = the whole step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun, one rank per GPU): the space-time sweeps do not shard (SURVEY
8(e)), so every rank solves an independent replica; value = all ranks'
iterations / max-over-ranks device time ("scaling": "weak").

After the timed region (rank 0, N=1) the line adds: rooflines of the P_T^-1 apply
(the dominant kernel, nd_sweep_kernel), J.v and assembly at C4_512; the other
BASELINE configurations (C2 full solve, C4 at Nt=64/128/256, the C5 operator
micro-benchmark in a child process); and `cpu_baseline` -- the oracle port (the
reference algorithm: SuperLU P_T, sparsetools SpMV, MGS GMRES) pinned to one host
core on a bounded slab-prefix sample, extrapolated (labelled) to the full solve.

`--impl reference` times that CPU implementation alone (the reference is pure
Python and does not exist on the GPU box; the oracle port pinned to it by golden
vectors stands in for it): each step one bounded sample, per-op costs scaled to
the full C4_512 solve with the reference iteration counts.
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

CONFIG = "C4_512"
NT_FULL = 512
# FGMRES counts of this configuration (Newton steps 1, 2), measured on the B200 and
# used by the reference arm's extrapolation; the unmodified reference gives the same
# counts at C4_64 ([96, 89], tests/golden/cfg_c4_64.npz) and C2 ([458, 413]).
REF_GMRES = [108, 98]
# CPU samples: first SAMPLE_SLABS slabs of the configuration, one Newton linearisation
# and SAMPLE_ITERS FGMRES(50) iterations
SAMPLE_SLABS, SAMPLE_ITERS = 4, 40
REF_SLABS, REF_ITERS = 2, 20  # --impl reference: per step (K + W steps must fit minutes)
WORKLOAD = ("C4 island coalescence 64x64 P2/P1, T=1, dt=1/512, Nt=512 (23.5 M unknowns), "
            "Newton rel 1e-6, FGMRES(50) rel 1e-8, P_T")
METRIC = "FGMRES iterations/s (C4 Nt=512 Newton solve, P_T preconditioner, FP64)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the other configurations")
    ap.add_argument("--c5-child", action="store_true", help=argparse.SUPPRESS)
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


def cpu_sample(config=CONFIG, slabs=SAMPLE_SLABS, iters=SAMPLE_ITERS):
    """One bounded oracle sample in a subprocess pinned to one core (BASELINE.md 3:
    the reference is single-threaded by construction -- SuperLU, sparsetools, Python
    loops -- so one core with OMP/OPENBLAS=1)."""
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    env.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "oracle.cpu_sample", "--config", config, "--slabs", str(slabs),
           "--iters", str(iters)]
    if shutil_which("taskset"):
        try:
            core = sorted(os.sched_getaffinity(0))[0]
        except (AttributeError, OSError):
            core = 0
        cmd = ["taskset", "-c", str(core)] + cmd
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    if out.returncode != 0:
        raise RuntimeError("cpu sample failed: " + out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def shutil_which(name):
    import shutil

    return shutil.which(name)


def host_info():
    cpu = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count()}


# Unmodified reference over the port's extrapolation, measured on full solves on one
# core of the build container (profiles/r02_cpu_calibration.json): C4_64 1.669 (the
# factor used: same 64^2 mesh as C4_512), C2 1.711.
CAL_FACTOR = 1.669


def extrapolate(sample, nt_full, gmres_iters):
    """Full-solve CPU seconds from a slab-prefix sample.  Every per-slab cost of the
    reference is linear in the slab count (causal block structure: residual, Jacobian,
    P_T setup, J.v, P_T^-1 and the MGS basis all loop over slabs), so the per-op times
    scale by nt_full / slabs; Newton does (newton + 1) residuals."""
    scale = nt_full / sample["slabs"]
    newton = len(gmres_iters)
    t = scale * ((newton + 1) * sample["t_residual"] + newton * (sample["t_jacobian"] + sample["t_pc_setup"])
                 + sum(gmres_iters) * sample["t_iter"])
    return t, sum(gmres_iters) / t


def sample_text(smp, nt_full, counts, t_full):
    return (f"oracle port of the reference algorithm (SuperLU P_T, sparsetools SpMV, MGS GMRES; pinned "
            f"to one core) on the {CONFIG} mesh restricted to its first {smp['slabs']} of {nt_full} slabs: "
            f"residual + Jacobian + P_T setup + {smp['iters']} FGMRES(50) iterations "
            f"({smp['t_iter'] * 1e3:.0f} ms each); per-op times x{nt_full // smp['slabs']} with the counts "
            f"{counts} -> {t_full:.0f} s per solve, x{CAL_FACTOR} calibration to the unmodified reference "
            f"(full C4_64/C2 solves, profiles/r02_cpu_calibration.json) -> {t_full * CAL_FACTOR:.0f} s "
            f"(EXTRAPOLATED)")


# ---------------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    times, samples = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        smp = cpu_sample(CONFIG, REF_SLABS, REF_ITERS)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            samples.append(smp)
    agg = dict(samples[-1])
    for k in ("t_residual", "t_jacobian", "t_pc_setup", "t_iter"):
        agg[k] = statistics.median(s[k] for s in samples)
    t_full, value = extrapolate(agg, NT_FULL, REF_GMRES)
    value /= CAL_FACTOR
    line = {
        "impl": "reference", "metric": METRIC,
        "value": value, "unit": "FGMRES it/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE C4 analytic problem)",
        "config": {"workload": WORKLOAD, "l2": "n/a (CPU)"},
        "newton_solve_s_extrapolated": t_full * CAL_FACTOR,
        "port_extrapolated_s_uncalibrated": t_full,
        "cpu_baseline": {"value": value, "unit": "FGMRES it/s", "cores": 1, "kind": "port",
                         "sample": sample_text(agg, NT_FULL, REF_GMRES, t_full) + "; one sample per step",
                         "host": host_info()},
        "e2e": {"value": value, "unit": "FGMRES it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------
def splu_fill(m):
    """L+U nnz of the reference's SuperLU factorisation (scipy splu, COLAMD)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    lu = spla.splu(sp.csc_matrix(m))
    return int(lu.L.nnz + lu.U.nnz)


def pt_algorithmic_bytes(p, disc, state, torch, dev):
    """SURVEY 8(d) P_T^-1 bytes: Nt 8 [fill(F_u) + fill(C_A) + nnz(f_a, f_p, z_j, z_a, sub1)]
    + 12 [fill(M_A, M_j, K_p, M_p) + nnz(M_A/dt, K_jA, M_p, sub2, B^T, M_u/dt)] + 16 N, with
    the reference SuperLU (COLAMD) fills of slab 0 at a perturbed state (structural fill)."""
    stp = p.SpaceTimeState(state.vec.copy(), state.ic_u, state.ic_a)
    stp.vec.data += 1e-3 * torch.randn(stp.vec.data.shape, dtype=torch.float64, device=dev,
                                       generator=torch.Generator(device=dev).manual_seed(0))
    jac = p.assemble_jacobian(stp, disc)
    pc = p.SpaceTimePreconditioner(jac, disc, stp)
    s0 = jac.slabs[0]
    nt, L = disc.n_steps, disc.layout
    per_slab = (splu_fill(s0.f_u) + splu_fill(pc.c_a[0]) + s0.f_a.nnz + pc.f_p[0].nnz + s0.z_j.nnz + s0.z_a.nnz
                + pc.c_a_sub1[0].nnz)
    const = (splu_fill(disc.mass_a_bc) + splu_fill(disc.mass_j) + splu_fill(disc.stiff_p_pinned)
             + splu_fill(disc.mass_p) + disc.mass_a_dt_bc.nnz + disc.mixed_ja_bc.nnz + disc.mass_p.nnz
             + pc.c_a_sub2.nnz + disc.div_t_bc.nnz + disc.mass_u_dt_bc.nnz)
    del pc, jac
    return nt * 8 * per_slab + 12 * const + 16 * nt * L.slab_size


def tmeas(torch, fn, r=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(r):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / r


def newton_cfg(p, rel):
    return p.NewtonConfig(abs_tol=1e-300, rel_tol=rel, max_iters=1 if rel is None else 25,
                          gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))


def other_configs(p, torch, dev, peak):
    """The other BASELINE configurations (not bench lines): C2 full solve, C4 at
    Nt=64/128/256 (one solve each, device-timed), C3 per-call operator times."""
    out = {}
    for name in ("C2", "C4_64", "C4_128", "C4_256"):
        d = p.discretize_config(name)
        _, _, _, nt, rel = p.config_problem(name)
        cfg = newton_cfg(p, rel)
        p.solve_all_at_once(d, cfg)  # warm-up (plans, dense tops, pools)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, st = p.solve_all_at_once(d, cfg)
        e1.record()
        e1.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        out[name] = {"solve_s": s, "newton": st.newton_iters, "fgmres": st.gmres_iters,
                     "fgmres_it_per_s": st.total_gmres / s,
                     "relative_residual": st.residual_norms[-1] / st.residual_norms[0]}
        del d
        torch.cuda.empty_cache()
    out["C2"]["reference_counts"] = [458, 413]
    out["C4_64"]["reference_counts"] = [96, 89]
    # C3: tearing 64^2, mu=eta=1e-3, Nt=128 -- stagnates in the reference algorithm itself
    # (DESIGN 7), so per-call operator times only
    d3 = p.discretize_config("C3")
    s3 = p.initial_state(d3)
    j3 = p.assemble_jacobian(s3, d3)
    pc3 = p.SpaceTimePreconditioner(j3, d3, s3)
    v3 = torch.randn(j3.size, dtype=torch.float64, device=dev)
    o3 = torch.empty_like(v3)
    out["C3"] = {"J_apply_ms": tmeas(torch, lambda: j3._into(v3, o3), 30),
                 "P_apply_ms": tmeas(torch, lambda: pc3._into(v3, o3), 5),
                 "assembly_ms": tmeas(torch, lambda: p.assemble_jacobian(s3, d3), 5),
                 "residual_ms": tmeas(torch, lambda: p.residual(s3, d3), 5),
                 "note": "FGMRES(50) with P_T stagnates at C3 in the reference algorithm (DESIGN 7)"}
    del d3, s3, j3, pc3, v3, o3
    torch.cuda.empty_cache()
    return out


def c5_child():
    """C5 operator micro-benchmark (BASELINE configs[4]; child process so its 77 GB of
    factors never meet the C4 solve's): 100 batched block-bidiagonal SpMVs and 20
    exact-inverse applications (the preconditioner application) over
    1024 slabs of a 256^2 P1 scalar advection-diffusion block."""
    import torch

    from paper_2309_00768_b200.c5 import C5Operator

    peak = peak_gbs()
    nt, n = 1024, 256
    t0 = time.perf_counter()
    op = C5Operator(n, nt, seed=0)
    op.factor()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(nt * op.n, dtype=torch.float64, device="cuda", generator=g)
    y = torch.empty_like(x)
    spmv_ms = tmeas(torch, lambda: op.apply(x, y), 100)
    inv_ms = tmeas(torch, lambda: op.solve(x, y), 20)
    op.solve(x, y)
    rt = float(torch.linalg.norm(op.apply(y) - x) / torch.linalg.norm(x))
    c = op.coupling
    spmv_bytes = nt * (8 * op.nnz + 16 * op.n) + 12 * c.nnz + 4 * op.nnz
    fill = splu_fill(op.matrix(0))
    sweep_bytes = nt * 8 * fill + 12 * c.nnz + 16 * nt * op.n
    print("C5JSON " + json.dumps({
        "workload": "C5 256x256 P1 scalar advection-diffusion, Nt=1024 (67.6 M unknowns), dt=1e-2, eps=1e-3",
        "spmv_ms": spmv_ms, "spmv_100_s": spmv_ms * 0.1,
        "spmv": {"algorithmic_bytes": spmv_bytes, "GBps": spmv_bytes / spmv_ms / 1e6,
                 "frac": spmv_bytes / spmv_ms / 1e6 / peak},
        "inverse_ms": inv_ms, "inverse_20_s": inv_ms * 0.02, "inverse_per_slab_us": 1e3 * inv_ms / nt,
        "inverse": {"algorithmic_bytes": sweep_bytes, "GBps": sweep_bytes / inv_ms / 1e6,
                    "frac": sweep_bytes / inv_ms / 1e6 / peak, "superlu_fill_per_slab": fill},
        "round_trip_rel": rt, "setup_s": setup,
        "timed": "100 SpMVs + 20 exact-inverse applications, CUDA events (the inverse is the exact "
                 "sequential block forward substitution, SURVEY 8(d) interpretation)"}), flush=True)


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6534.5))
    except Exception:
        return 6534.5  # fallback: the pool's measured copy peak of round 1


def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2309_00768_b200 as p
    from paper_2309_00768_b200 import _lib
    from paper_2309_00768_b200.replicas import aggregate

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    c5 = None
    if rank == 0 and world == 1 and not args.no_extras:
        # C5 first, in a child process: its 77 GB of factors must not meet this process's pools
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--c5-child"], cwd=ROOT,
                               capture_output=True, text=True, timeout=900)
            c5l = [ln for ln in r.stdout.splitlines() if ln.startswith("C5JSON ")]
            c5 = json.loads(c5l[0][7:]) if c5l else {"error": r.stderr[-300:]}
        except Exception as exc:
            c5 = {"error": str(exc)[:300]}
    torch.cuda.set_device(dev)
    lib = _lib.load()
    disc = p.discretize_config(CONFIG)
    _, _, _, nt, rel = p.config_problem(CONFIG)
    cfg = newton_cfg(p, rel)
    st0 = p.initial_state(disc)
    # pinned host copies of the inputs (the initial state and the initial conditions)
    h_state = st0.vec.data.cpu().pin_memory()
    h_icu, h_ica = st0.ic_u.cpu().pin_memory(), st0.ic_a.cpu().pin_memory()
    h_out = torch.empty_like(h_state).pin_memory()
    h2d = (h_state.numel() + h_icu.numel() + h_ica.numel()) * 8
    d2h = h_out.numel() * 8
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)  # > L2 (126 MB)

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        vec = h_state.to(dev, non_blocking=True)
        icu, ica = h_icu.to(dev, non_blocking=True), h_ica.to(dev, non_blocking=True)
        ev[1].record()
        state = p.SpaceTimeState(p.BlockVector(disc.layout, disc.n_steps, vec), icu, ica)
        state, stats = p.solve_all_at_once(disc, cfg, state=state)
        ev[2].record()
        h_out.copy_(state.vec.data, non_blocking=True)
        ev[3].record()
        ev[3].synchronize()
        return ev[1].elapsed_time(ev[2]), ev[0].elapsed_time(ev[3]), stats

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = Clocks(dev.index)
    dev_ms, e2e_ms, iters, breakdown = [], [], 0, {}
    barrier()
    torch.cuda.synchronize()
    launches0 = int(lib.stmhd_launch_count())
    clocks.start()
    stats_last = None
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed solves (untimed)
        torch.cuda.synchronize()
        dms, ems, stats = step()
        dev_ms.append(dms)
        e2e_ms.append(ems)
        iters += stats.total_gmres
        for k, v in stats.timings.items():
            breakdown[k] = breakdown.get(k, 0.0) + v
        stats_last = stats
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = int(lib.stmhd_launch_count()) - launches0
    barrier()
    total_s, iters_all = aggregate(sum(dev_ms) / 1e3, iters, dev)
    e2e_s, _ = aggregate(sum(e2e_ms) / 1e3, iters, dev)
    value = iters_all / total_s
    e2e_value = iters_all / e2e_s
    peak = peak_gbs()
    line = {
        "metric": METRIC, "value": value, "unit": "FGMRES it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE C4 analytic problem: island coalescence, equilibrium initial state)",
        "config": {"workload": WORKLOAD, "parallelism": "replicas" if world > 1 else "single",
                   "l2": "512 MB flush between timed solves; per-solve factors ~26 GB > L2"},
        "newton_solve_s": total_s / args.steps, "newton_steps": stats_last.newton_iters,
        "fgmres_iters": stats_last.gmres_iters,
        "relative_residual": stats_last.residual_norms[-1] / stats_last.residual_norms[0],
        "phase_s_per_solve": {k: v / args.steps for k, v in breakdown.items()},
        "e2e": {"value": e2e_value, "unit": "FGMRES it/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "same timed solves: pinned-host state in, device solve, solution out"},
        "gpu_launches": launches, "clocks": clk,
    }
    if rank != 0:
        return
    # ---- rooflines at C4_512 (after the timed region): P_T^-1 (dominant), J.v, assembly ----
    jac = p.assemble_jacobian(st0, disc)
    pc = p.SpaceTimePreconditioner(jac, disc, st0)
    L = disc.layout
    v = torch.randn(jac.size, dtype=torch.float64, device=dev)
    out = torch.empty_like(v)
    pt_ms = tmeas(torch, lambda: pc._into(v, out), 10)
    pt_bytes = pt_algorithmic_bytes(p, disc, st0, torch, dev)
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "sweep_traffic.json")))
        if prof.get("config") == CONFIG:
            traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    achieved = pt_bytes / (pt_ms / 1e3) / 1e9
    line["roofline"] = {
        "kernel": "nd_sweep_kernel: one P_T^-1 apply (pipelined wave | M_j | F_u sweeps, ~95% of the apply) "
                  "+ its batched pre-steps", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": pt_bytes, "launch_ms": pt_ms,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json"))
        else "fallback 6534.5 GB/s (round-1 measured copy peak)",
        "bytes_formula": "SURVEY 8(d): reference SuperLU (COLAMD) fills, so independent of the GPU factorisation"}
    P_ = disc.pattern
    jv_bytes = nt * (8 * P_.nnz + 16 * L.slab_size) + 12 * disc.jc_nnz + 8 * L.n_p + 4 * P_.nnz
    asm_bytes = nt * 8 * (2 * L.slab_size + P_.nnz + P_.fp_nnz)
    jv_ms = tmeas(torch, lambda: jac._into(v, out), 30)
    asm_ms = tmeas(torch, lambda: p.assemble_jacobian(st0, disc), 5) + tmeas(torch, lambda: p.residual(st0, disc), 5)
    line["kernel_rooflines"] = {
        "P_T^-1 apply": {"algorithmic_bytes": pt_bytes, "ms": pt_ms, "GBps": achieved, "frac": achieved / peak},
        "J_apply (sell_spmv_kernel)": {"algorithmic_bytes": jv_bytes, "ms": jv_ms, "GBps": jv_bytes / jv_ms / 1e6,
                                       "frac": jv_bytes / jv_ms / 1e6 / peak},
        "assembly (residual_patch + values_patch)": {"algorithmic_bytes": asm_bytes, "ms": asm_ms,
                                                     "GBps": asm_bytes / asm_ms / 1e6,
                                                     "frac": asm_bytes / asm_ms / 1e6 / peak},
        "config": CONFIG}
    del jac, pc, v, out
    torch.cuda.empty_cache()
    if world == 1 and not args.no_extras:
        try:
            line["other_configs"] = other_configs(p, torch, dev, peak)
        except Exception as exc:
            line["other_configs"] = {"error": str(exc)[:300]}
        line["c5_operator"] = c5
    if world == 1 and not args.no_cpu_baseline:
        try:
            smp = cpu_sample()
            t_full, cv = extrapolate(smp, nt, stats_last.gmres_iters)
            cv /= CAL_FACTOR
            line["cpu_baseline"] = {"value": cv, "unit": "FGMRES it/s", "cores": 1, "kind": "port",
                                    "sample": sample_text(smp, nt, stats_last.gmres_iters, t_full),
                                    "host": host_info(),
                                    "calibration": {"factor": CAL_FACTOR, "file": "profiles/r02_cpu_calibration.json",
                                                    "points": "unmodified reference full solves on one core of "
                                                              "the build container: C2 737.7 s [458, 413], C4_64 "
                                                              "939.9 s [96, 89]"}}
        except Exception as exc:  # keep the GPU line even if the CPU sample fails
            line["cpu_baseline"] = {"value": None, "unit": "FGMRES it/s", "cores": 1, "kind": "port",
                                    "sample": f"failed: {exc}"[:300]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.c5_child:
        c5_child()
        return
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
