"""Golden fixtures at BASELINE-config scale from the UNMODIFIED reference ``stmhd``.

Run in the build container only (``/root/reference`` does not exist on the GPU
box), one case per process, pinned to one core as BASELINE.md section 3 asks::

    OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 taskset -c 0 \
        python tests/golden/make_golden_configs.py c2

It reuses the SURVEY 0.1 adapter of ``make_golden.py`` (P2/P1 degree swap,
[-1,1]^2, Dirichlet A top and bottom with the bottom flux) and only *wraps* the
reference's own functions with timers (``stmhd.solver`` module globals), it
never edits the reference.

Cases (file -> content):
  cfg_c2.npz        C2 (island 32^2, dt=0.05, Nt=64): full Newton solve to rel 1e-6 --
                    per-step FGMRES counts, residual norms, the final state (all N
                    entries) and the per-phase wall times of the reference on 1 core
  cfg_c3p.npz       C3 prefix (tearing 64^2, mu=eta=1e-3, dt=0.02, first 3 of 128 slabs;
                    causality makes the prefix exact): perturbed-state residual, J.v,
                    P_T^-1 v, Alfven scalings, plus sampled per-slab Jacobian values
  cfg_c4_64.npz     C4 at Nt=64 (island 64^2, dt=1/64): full Newton solve -- counts,
                    residual norms, sampled final state + per-slab norms, phase times
  cfg_c5p.npz       C5 (256^2 P1 scalar, dt=1e-2) 32-slab prefix: F x and the exact
                    inverse F^-1 x sampled (every 61st entry) + per-slab norms, per-op times
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import baseline_disc, c5_case, csr_dump  # noqa: E402  (adapter + reference import)

import stmhd  # noqa: E402
from stmhd import solver as ref_solver  # noqa: E402
from stmhd.precond import SpaceTimePreconditioner  # noqa: E402
from stmhd.spacetime import assemble_jacobian, residual  # noqa: E402

STRIDE = 61  # sampled fixtures keep every 61st entry


class PhaseTimer:
    """Accumulates wall time of the reference's hot-path calls made by _newton."""

    NAMES = ("residual", "assemble_jacobian", "SpaceTimePreconditioner", "gmres")

    def __init__(self):
        self.t = {n: 0.0 for n in self.NAMES}
        self.n = {n: 0 for n in self.NAMES}
        self.orig = {}

    def __enter__(self):
        for name in self.NAMES:
            fn = getattr(ref_solver, name)
            self.orig[name] = fn

            def wrapped(*a, _fn=fn, _name=name, **k):
                t0 = time.perf_counter()
                out = _fn(*a, **k)
                self.t[_name] += time.perf_counter() - t0
                self.n[_name] += 1
                return out

            setattr(ref_solver, name, wrapped)
        return self

    def __exit__(self, *exc):
        for name, fn in self.orig.items():
            setattr(ref_solver, name, fn)


def host_info():
    import scipy

    cpu = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu": cpu, "nproc": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "numpy": np.__version__, "scipy": scipy.__version__,
            "omp": os.environ.get("OMP_NUM_THREADS"), "openblas": os.environ.get("OPENBLAS_NUM_THREADS")}


def newton_solve(disc, rel):
    gm = stmhd.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50)
    st = stmhd.initial_state(disc)
    r0 = residual(st, disc).norm()
    cfg = ref_solver.NewtonConfig(abs_tol=rel * r0, max_iters=25, gmres=gm)
    t0 = time.perf_counter()
    with PhaseTimer() as pt:
        state, stats = ref_solver.solve_all_at_once(disc, cfg)
    wall = time.perf_counter() - t0
    return state, stats, wall, pt


def case_solve(name, kind, visc, n, dt, nt, full_x):
    t0 = time.perf_counter()
    disc = baseline_disc(kind, visc, n, dt, nt)
    t_disc = time.perf_counter() - t0
    state, stats, wall, pt = newton_solve(disc, 1e-6)
    x = state.vec.data
    out = {"gmres_iters": np.array(stats.gmres_iters), "newton_iters": stats.newton_iters,
           "residual_norms": np.array(stats.residual_norms), "converged": stats.converged,
           "slab_norms": np.linalg.norm(x.reshape(nt, -1), axis=1), "x_norm": np.linalg.norm(x)}
    if full_x:
        out["x"] = x
    else:
        out["x_sample"] = x[::STRIDE].copy()
    times = {"discretize_s": t_disc, "solve_wall_s": wall, "phase_s": pt.t, "phase_calls": pt.n,
             "host": host_info(), "gmres_iters": [int(g) for g in stats.gmres_iters],
             "residual_norms": [float(r) for r in stats.residual_norms]}
    out["times_json"] = np.array(json.dumps(times))
    np.savez_compressed(os.path.join(HERE, f"cfg_{name}.npz"), **out)
    print(name, json.dumps(times), flush=True)


def case_c3_prefix(nslab=3, seed=11):
    disc = baseline_disc("tearing", 1e-3, 64, 0.02, nslab)
    rng = np.random.default_rng(seed)
    st = stmhd.initial_state(disc)
    out = {"seed": seed, "nslab": nslab}
    # the reference's initial state is one slab repeated; keep it (and the IC) so the
    # device side perturbs exactly the same state
    assert np.array_equal(st.vec.data.reshape(nslab, -1), np.tile(st.vec.data.reshape(nslab, -1)[0], (nslab, 1)))
    out["state0_slab"] = st.vec.data.reshape(nslab, -1)[0].copy()
    out["ic_u"], out["ic_a"] = st.ic_u, st.ic_a
    st.vec.data += 1e-3 * rng.standard_normal(st.vec.data.size)
    t = {}
    t0 = time.perf_counter()
    out["r"] = residual(st, disc).data
    t["residual_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    jac = assemble_jacobian(st, disc)
    t["jacobian_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    prec = SpaceTimePreconditioner(jac, disc, st)
    t["pc_setup_s"] = time.perf_counter() - t0
    v = rng.standard_normal(jac.size)
    t0 = time.perf_counter()
    out["Jv"] = jac.apply(v)
    t["jv_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    out["Pv"] = prec.apply_inverse(v)
    t["pinv_s"] = time.perf_counter() - t0
    out["alfven"] = np.asarray(prec.alfven)
    # Jacobian blocks of the last slab (the one coupled to its predecessors), sampled
    b = jac.slabs[nslab - 1]
    for name in ("f_u", "z_j", "z_a", "y", "f_a"):
        m = getattr(b, name).tocoo()
        sel = np.arange(0, m.nnz, 31)
        out[f"blk_{name}_row"] = m.row[sel].astype(np.int32)
        out[f"blk_{name}_col"] = m.col[sel].astype(np.int32)
        out[f"blk_{name}_val"] = m.data[sel]
        out[f"blk_{name}_nnz"] = m.nnz
    nt, n_u, n_p, n_a = nslab, disc.layout.n_u, disc.layout.n_p, disc.layout.n_a
    out["sv_u_sample"] = prec.solve_velocity(v[: nt * n_u].copy())[::7].copy()
    out["sw_a_sample"] = prec.solve_wave(v[: nt * n_a].copy())[::7].copy()
    t["host"] = host_info()
    out["times_json"] = np.array(json.dumps(t))
    np.savez_compressed(os.path.join(HERE, "cfg_c3p.npz"), **out)
    print("c3p", json.dumps(t), "|r|", np.linalg.norm(out["r"]), flush=True)


def case_c5_prefix(nslab=32):
    raw = {}
    t0 = time.perf_counter()
    c5_case(raw, n=256, nt=nslab, seed=0)
    total = time.perf_counter() - t0
    out = {"nslab": nslab, "stride": STRIDE}
    for key in ("Fx", "Finv_x"):
        a = raw[key]
        out[key + "_sample"] = a.reshape(-1)[::STRIDE].copy()
        out[key + "_slab_norms"] = np.linalg.norm(a, axis=1)
    out["x_slab_norms"] = np.linalg.norm(raw["x"], axis=1)
    out["times_json"] = np.array(json.dumps({"c5_case_s": total, "host": host_info()}))
    np.savez_compressed(os.path.join(HERE, "cfg_c5p.npz"), **out)
    print("c5p", total, flush=True)


if __name__ == "__main__":
    which = sys.argv[1]
    if which == "c2":
        case_solve("c2", "island", 1e-2, 32, 0.05, 64, full_x=True)
    elif which == "c4_64":
        case_solve("c4_64", "island", 1e-2, 64, 1.0 / 64, 64, full_x=False)
    elif which == "c3p":
        case_c3_prefix()
    elif which == "c5p":
        case_c5_prefix()
    else:
        raise SystemExit("usage: make_golden_configs.py c2|c4_64|c3p|c5p")
