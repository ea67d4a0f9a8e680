"""Build and load tools/microbench.cu (barrier / pointer-chase micro-benchmarks; not
part of the product library) as tools/_lib/libstmhd_microbench.so."""

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(os.path.dirname(HERE), "paper_2309_00768_b200", "csrc")
OUT = os.path.join(HERE, "_lib", "libstmhd_microbench.so")


def load():
    src = os.path.join(HERE, "microbench.cu")
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-Xcompiler", "-fPIC", "-shared", "-I", CSRC, src, "-o", OUT])
    return ctypes.CDLL(OUT)
