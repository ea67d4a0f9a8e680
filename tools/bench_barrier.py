import ctypes
import _microbench
lib = _microbench.load()
for bps in (1, 2):
    us = ctypes.c_double()
    lib.stmhd_bench_barrier(bps, 256, 2000, ctypes.byref(us))
    print(f"grid barrier blocks/SM={bps}: {us.value:.2f} us")
for nelem, label in ((1 << 14, "64KB (L1)"), (1 << 22, "16MB (L2)"), (1 << 27, "512MB (HBM)")):
    for cl, th in ((1, 32), (16, 1024)):
        lat, bar = ctypes.c_double(), ctypes.c_double()
        st = lib.stmhd_bench_chase(nelem, 2000, cl, th, 2000, ctypes.byref(lat), ctypes.byref(bar))
        print(f"chase {label} cluster={cl} threads={th}: {lat.value:.1f} ns/load, cluster barrier {bar.value:.1f} ns (st={st})")
