"""Experiment rows (reference cli.py:26, 68-100, 148-208): CSV header and
formatting, sweep validation (CPU), and one device sweep cell per mode (GPU)."""

import numpy as np
import pytest

from paper_2309_00768_b200 import experiments as ex
from paper_2309_00768_b200.errors import ConfigurationError


def test_csv_rows_match_reference_format(tmp_path):
    row = ex.ResultRow("tearing_mode", 0.25, 0.125, 1.0, 8, "both", 3, 41.333333333, 8, 1.2345678, None, "ok", 2.5)
    assert row.to_csv() == "tearing_mode,0.25,0.125,1,8,both,3,41.3333,8,1.23457,,ok,2.5"
    path = tmp_path / "r.csv"
    ex.emit_csv([row, row], str(path))
    lines = open(path, newline="").read().split("\n")
    assert lines[0] == ex.CSV_HEADER and lines[1] == row.to_csv() and lines[-1] == ""
    with pytest.raises(ConfigurationError):
        ex.emit_csv([], str(path))


def test_sweep_validation():
    with pytest.raises(ConfigurationError):
        ex.run_sweep("x", None, [], [0.1], [1.0])
    with pytest.raises(ConfigurationError):
        ex.run_sweep("x", None, [0.5], [2.0], [1.0])  # dt > T
    with pytest.raises(ConfigurationError):
        ex.run_sweep("x", None, [0.5], [-0.1], [1.0])


@pytest.mark.gpu
def test_sweep_cells_on_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p

    prob = p.by_name("island_coalescence")
    cfg = p.NewtonConfig(abs_tol=1e-8, gmres=p.GmresConfig(rel_tol=1e-2, abs_tol=1e-14))
    rows = ex.run_sweep("island_coalescence", prob, [0.5], [0.5], [1.0], mode="both", ncfg=cfg)
    assert len(rows) == 1
    r = rows[0]
    assert r.status == "ok" and r.n_steps == 2 and r.newton >= 1 and r.effective_steps >= 1
    assert np.isfinite(r.newton_ratio) and np.isfinite(r.gmres_ratio)
    assert len(r.to_csv().split(",")) == len(ex.CSV_HEADER.split(","))


def test_experiment_config_mirrors_reference():
    cfg = ex.ExperimentConfig()
    assert (cfg.problem, cfg.dx, cfg.dt, cfg.t_final, cfg.mode, cfg.precond) == (
        "tearing_mode", [0.25], [0.25], [1.0], "spacetime", "triangular")
    n = cfg.newton_config()
    assert (n.abs_tol, n.max_iters, n.gmres.rel_tol, n.gmres.abs_tol) == (1e-10, 25, 1e-2, 1e-14)
    for bad in (dict(dx=[]), dict(mode="x"), dict(dt=[-1.0]), dict(dt=[2.0]), dict(precond="nope")):
        with pytest.raises(Exception):
            ex.ExperimentConfig(**bad).validate()


@pytest.mark.gpu
def test_sweep_rows_match_reference(golden_json):
    """Rows of the reference's own harness (tests/golden/make_golden_sweep.py: cli.run_sweep
    with its ExperimentConfig defaults) reproduced by the device solvers: problem, grid,
    Nt, mode, Newton counts, effective steps and status exactly; the GMRES averages and
    the overhead ratios within one GMRES iteration per Newton step."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref = golden_json("sweep_rows")
    for name, case in ref.items():
        rows = ex.run_sweep(ex.ExperimentConfig(**case["config"]))
        assert len(rows) == len(case["rows"]), name
        for mine, want in zip(rows, case["rows"]):
            m = mine.to_csv().split(",")[:-1]
            w = want.split(",")
            assert m[:6] == w[:6] and m[6] == w[6] and m[8] == w[8] and m[11] == w[11], (name, m, w)
            newton = float(w[6]) if w[6] else 1.0
            assert abs(float(m[7]) - float(w[7])) <= 1.0 + 1e-9, (name, m, w)
            for i in (9, 10):
                if w[i]:
                    assert abs(float(m[i]) - float(w[i])) <= 1.0 / max(newton, 1.0) + 0.05 * float(w[i]), (name, m, w)
