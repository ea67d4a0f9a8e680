"""Experiment sweeps on the device solvers with the reference's CSV rows (SURVEY
8(f)-4; reference cli.py:26, 68-100 ResultRow, 148-208 run_sweep/_run_cell/emit_csv).

Only the sweep/row layer is mirrored (same header, same 6-significant-digit
formatting, same per-cell semantics for the 'spacetime', 'sequential' and 'both'
modes, failures recorded in the status column); there is no command-line front
end.  ``run_baseline_configs`` runs BASELINE configurations by name (C1..C4_512)
with their Newton relative stop and adds device throughput columns.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

from .errors import ConfigurationError, ConvergenceError, StmhdError
from .linalg import GmresConfig
from .precond import Variant
from .solver import NewtonConfig, compute_overhead_ratios, solve_all_at_once, solve_sequential

CSV_HEADER = "problem,dx,dt,T,Nt,mode,newton,avg_gmres,effective_steps,newton_ratio,gmres_ratio,status,wall_s"
MODES = ("spacetime", "sequential", "both")


@dataclass
class ExperimentConfig:
    """Sweep configuration with the reference's fields, defaults, validation and
    Newton/GMRES settings (cli.py:32-65): Newton abs 1e-10, GMRES rel 1e-2 / abs 1e-14."""

    problem: str = "tearing_mode"
    dx: list = field(default_factory=lambda: [0.25])
    dt: list = field(default_factory=lambda: [0.25])
    t_final: list = field(default_factory=lambda: [1.0])
    mode: str = "spacetime"
    precond: str = "triangular"
    out: str = "results.csv"
    newton_tol: float = 1e-10
    gmres_rtol: float = 1e-2
    gmres_atol: float = 1e-14
    max_newton: int = 25
    eps: float = 1e-3
    seed: int = 0  # reserved; the solver itself is deterministic

    def validate(self):
        if not self.dx or not self.dt or not self.t_final:
            raise ConfigurationError("dx, dt, and T sweep lists must be nonempty")
        if self.mode not in MODES:
            raise ConfigurationError(f"mode must be one of {MODES}, got '{self.mode}'")
        if any(v <= 0 for v in list(self.dx) + list(self.dt) + list(self.t_final)):
            raise ConfigurationError("all dx, dt, T values must be positive")
        for t in self.t_final:
            if any(dt > t for dt in self.dt):
                raise ConfigurationError("dt must not exceed T")
        Variant(self.precond)

    def newton_config(self) -> NewtonConfig:
        return NewtonConfig(abs_tol=self.newton_tol, max_iters=self.max_newton,
                            gmres=GmresConfig(rel_tol=self.gmres_rtol, abs_tol=self.gmres_atol),
                            variant=Variant(self.precond))


@dataclass
class ResultRow:
    problem: str
    dx: float
    dt: float
    t_final: float
    n_steps: int
    mode: str
    newton: float
    avg_gmres: float
    effective_steps: int | None
    newton_ratio: float | None
    gmres_ratio: float | None
    status: str
    wall_s: float

    def to_csv(self) -> str:
        def fmt(v):
            if v is None:
                return ""
            if isinstance(v, float):
                return f"{v:.6g}"
            return str(v)

        return ",".join(fmt(v) for v in (self.problem, self.dx, self.dt, self.t_final, self.n_steps, self.mode,
                                         self.newton, self.avg_gmres, self.effective_steps, self.newton_ratio,
                                         self.gmres_ratio, self.status, self.wall_s))


def run_cell(problem_name: str, problem, dx: float, dt: float, t_final: float, mode: str,
             ncfg: NewtonConfig) -> ResultRow:
    """One sweep cell (reference cli.py:165-198)."""
    from .discretization import discretize

    if mode not in MODES:
        raise ConfigurationError(f"mode must be one of {MODES}, got '{mode}'")
    disc = discretize(problem, dx, dt, t_final)
    base = dict(problem=problem_name, dx=dx, dt=dt, t_final=t_final, n_steps=disc.n_steps)
    try:
        if mode == "spacetime":
            _, st = solve_all_at_once(disc, ncfg)
            return ResultRow(**base, mode="spacetime", newton=st.newton_iters, avg_gmres=st.avg_gmres,
                             effective_steps=None, newton_ratio=None, gmres_ratio=None,
                             status="ok" if st.converged else "nonconverged", wall_s=st.wall_time)
        if mode == "sequential":
            _, seq = solve_sequential(disc, ncfg)
            return ResultRow(**base, mode="sequential", newton=seq.avg_newton_per_step,
                             avg_gmres=(seq.avg_gmres if seq.newton_iters else 0.0),
                             effective_steps=seq.effective_steps, newton_ratio=None, gmres_ratio=None,
                             status="ok" if seq.converged else "nonconverged", wall_s=seq.wall_time)
        _, st = solve_all_at_once(disc, ncfg)
        _, seq = solve_sequential(disc, ncfg)
        nr, gr = compute_overhead_ratios(st, seq)
        return ResultRow(**base, mode="both", newton=st.newton_iters, avg_gmres=st.avg_gmres,
                         effective_steps=seq.effective_steps, newton_ratio=nr, gmres_ratio=gr,
                         status="ok" if (st.converged and seq.converged) else "nonconverged",
                         wall_s=st.wall_time + seq.wall_time)
    except (ConvergenceError, StmhdError) as exc:
        return ResultRow(**base, mode=mode, newton=0, avg_gmres=0.0, effective_steps=None, newton_ratio=None,
                         gmres_ratio=None, status=f"failed: {exc}", wall_s=0.0)


def run_sweep(problem_name, problem=None, dxs=None, dts=None, t_finals=None, mode: str = "spacetime",
              ncfg: NewtonConfig | None = None) -> list[ResultRow]:
    """Rows ordered dx outer, then dt, then T (reference cli.py:148-162).

    ``run_sweep(ExperimentConfig(...))`` is the reference's call (problem by name with
    the config's eps, its Newton/GMRES settings and variant); the long form takes the
    problem object, the sweep lists, the mode and a NewtonConfig."""
    if isinstance(problem_name, ExperimentConfig):
        from .problems import by_name

        cfg = problem_name
        cfg.validate()
        return run_sweep(cfg.problem, by_name(cfg.problem, eps=cfg.eps), cfg.dx, cfg.dt, cfg.t_final, cfg.mode,
                         cfg.newton_config())
    if not dxs or not dts or not t_finals:
        raise ConfigurationError("dx, dt, and T sweep lists must be nonempty")
    if any(v <= 0 for v in list(dxs) + list(dts) + list(t_finals)):
        raise ConfigurationError("all dx, dt, T values must be positive")
    for t in t_finals:
        if any(dt > t for dt in dts):
            raise ConfigurationError("dt must not exceed T")
    ncfg = ncfg or NewtonConfig(variant=Variant.TRIANGULAR)
    return [run_cell(problem_name, problem, dx, dt, t, mode, ncfg) for dx in dxs for dt in dts for t in t_finals]


def emit_csv(rows: list[ResultRow], path: str) -> None:
    """LF endings, 6-significant-digit floats (reference cli.py:201-208)."""
    if not rows:
        raise ConfigurationError("no result rows to write")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(CSV_HEADER + "\n")
        for row in rows:
            fh.write(row.to_csv() + "\n")


def run_baseline_configs(names, gmres_max_iters: int = 20000) -> list[dict]:
    """BASELINE configurations by name: Newton to the configuration's relative stop
    (one step for C1), FGMRES(50) rel 1e-8; the CSV row plus iteration counts and
    device throughput (FGMRES iterations per second of solve time)."""
    import torch

    from .discretization import discretize_config
    from .problems import config_problem

    out = []
    for name in names:
        prob, n, dt, nt, rel = config_problem(name)
        x0, x1, _, _ = prob.domain
        cfg = NewtonConfig(abs_tol=1e-300, rel_tol=rel, max_iters=1 if rel is None else 25,
                           gmres=GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=gmres_max_iters, restart=50))
        disc = discretize_config(name)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            _, st = solve_all_at_once(disc, cfg)
            status = "ok" if (st.converged or rel is None) else "nonconverged"  # C1: one Newton step
        except (ConvergenceError, StmhdError) as exc:
            st, status = None, f"failed: {exc}"
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        row = ResultRow(problem=name, dx=(x1 - x0) / n, dt=dt, t_final=nt * dt, n_steps=nt, mode="spacetime",
                        newton=st.newton_iters if st else 0, avg_gmres=st.avg_gmres if st else 0.0,
                        effective_steps=None, newton_ratio=None, gmres_ratio=None, status=status, wall_s=wall)
        rec = {"csv": row.to_csv(), "config": name, "unknowns": nt * disc.layout.slab_size,
               "newton": row.newton, "gmres": list(st.gmres_iters) if st else [],
               "relative_residual": (st.residual_norms[-1] / st.residual_norms[0]) if st else None,
               "wall_s": wall, "fgmres_it_per_s": (st.total_gmres / wall) if st else None}
        out.append(rec)
        del disc
        torch.cuda.empty_cache()
    return out
