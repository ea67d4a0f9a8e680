"""Opcode histogram of selected kernels in the built library (cuobjdump -sass), with
the Blackwell mnemonics that show how data moves: UBLKCP (cp.async.bulk / TMA bulk
copy), SYNCS (mbarrier), UBLKPF (bulk L2 prefetch), LDGSTS (cp.async), DMMA (FP64
tensor-core mma), DFMA, LDG/STG/LDS/STS.
  python tools/sass_summary.py [kernel-substring ...] > profiles/rNN_sass_summary.md
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2309_00768_b200", "_lib",
                   "libstmhd_b200.so")
KEY = ["UBLKCP", "SYNCS", "UBLKPF", "LDGSTS", "DMMA", "DFMA", "DADD", "DMUL", "LDG", "STG", "LDS", "STS", "LD", "ST",
       "SHFL", "BAR", "RED", "ATOM", "MEMBAR"]


def main():
    want = sys.argv[1:] or ["nd_sweep_kernel", "values_patch_kernel", "residual_patch_kernel", "sell_spmv_kernel",
                            "topk_kernel", "nd_factor_level", "dense_gemm_kernel", "update_partial"]
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            funcs[cur][m.group(1)] += 1
    print(f"# SASS opcode summary ({os.path.basename(LIB)}, sm_100a)\n")
    print("| kernel | instructions | " + " | ".join(KEY) + " |")
    print("|---|---|" + "---|" * len(KEY))
    for name, c in funcs.items():
        if not any(w in name for w in want):
            continue
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        print(f"| `{dem[:70]}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in KEY) + " |")


if __name__ == "__main__":
    main()
