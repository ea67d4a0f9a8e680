"""Golden sweep rows from the UNMODIFIED reference's experiment harness
(``stmhd.cli.run_sweep``, cli.py:148-208; build container only:
``python tests/golden/make_golden_sweep.py``).  Small grids, every mode, the
reference's ExperimentConfig defaults (Newton abs 1e-10, GMRES rel 1e-2 / abs 1e-14,
TRIANGULAR).  The wall-time column is dropped (machine dependent).

  sweep_rows.json   {case name: [csv row without wall_s, ...]}
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from stmhd.cli import ExperimentConfig, run_sweep  # noqa: E402

CASES = {
    "island_spacetime": dict(problem="island_coalescence", dx=[0.5], dt=[0.5, 0.25], t_final=[1.0],
                             mode="spacetime"),
    "island_sequential": dict(problem="island_coalescence", dx=[0.5], dt=[0.5, 0.25], t_final=[1.0],
                              mode="sequential"),
    "island_both": dict(problem="island_coalescence", dx=[0.5], dt=[0.5], t_final=[1.0, 2.0], mode="both"),
    "tearing_both": dict(problem="tearing_mode", dx=[0.25], dt=[0.5], t_final=[1.0], mode="both"),
    "tearing_full": dict(problem="tearing_mode", dx=[0.25], dt=[0.5], t_final=[1.0], mode="spacetime",
                         precond="full"),
}


def main():
    out = {}
    for name, kw in CASES.items():
        rows = run_sweep(ExperimentConfig(**kw))
        out[name] = {"config": kw, "rows": [",".join(r.to_csv().split(",")[:-1]) for r in rows]}
        print(name, out[name]["rows"])
    with open(os.path.join(HERE, "sweep_rows.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
