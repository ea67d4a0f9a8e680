"""BASELINE configs[3] (time-step refinement, island 64x64, T = 1, Nt in {64..512})
and any other named configs through experiments.run_baseline_configs; writes the
reference-format CSV and one JSON line per configuration."""
import argparse
import json

from paper_2309_00768_b200 import experiments

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C4_64,C4_128,C4_256,C4_512")
ap.add_argument("--csv", default="gpurun_out/c4.csv")
args = ap.parse_args()
recs = []
for name in args.configs.split(","):
    rec = experiments.run_baseline_configs([name])[0]
    print(json.dumps(rec), flush=True)
    recs.append(rec)
with open(args.csv, "w", newline="\n") as fh:
    fh.write(experiments.CSV_HEADER + "\n")
    for r in recs:
        fh.write(r["csv"] + "\n")
