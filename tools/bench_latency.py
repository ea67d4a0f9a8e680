import ctypes
import _microbench
lib = _microbench.load()
lib.stmhd_bench_chase2.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
for nelem, label in ((1 << 12, "16KB"), (1 << 18, "1MB"), (1 << 23, "32MB"), (1 << 27, "512MB")):
    for cl, th in ((2, 32), (16, 32), (16, 512)):
        for bar in (0, 1):
            c = ctypes.c_double()
            st = lib.stmhd_bench_chase2(nelem, 1000, cl, th, bar, ctypes.byref(c))
            print(f"{label:6s} cluster={cl:2d} threads={th:3d} barrier={bar}: {c.value:7.0f} cycles/step (st={st})")
