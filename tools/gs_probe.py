"""CGS2 kernels alone at a given vector length (default: C4_512's 23.5 M unknowns):
device time of the dots, update+dots, update+norm and normalise calls for j = 1..m basis
vectors, and a checksum of the coefficients (compare builds / STMHD_GS_V1=1)."""
import sys

import torch

from paper_2309_00768_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 23_527_424
m = int(sys.argv[2]) if len(sys.argv) > 2 else 50
lib = _lib.load()
sp_ = _lib.stream_ptr()
g = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(m + 1, n, dtype=torch.float64, device="cuda", generator=g)
dev = torch.zeros(2 * m + 8, dtype=torch.float64, device="cuda")
work = torch.empty(int(lib.stmhd_gs_work_size(n, m + 1)) + 8, dtype=torch.float64, device="cuda")
names = ["dots", "update+dots", "update+norm", "normalize"]
tot = [0.0] * 4
chk = 0.0
ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
for rep in range(2):
    tot = [0.0] * 4
    for j in range(m):
        nv = j + 1
        w = V[nv]
        h1, h2, nrm = dev[:nv], dev[m + 1: m + 1 + nv], dev[2 * m + 3: 2 * m + 4]
        ev[0].record()
        _lib.check(lib.stmhd_gs_dots(sp_, _lib.ptr(V), n, nv, _lib.ptr(w), n, _lib.ptr(h1), _lib.ptr(work)))
        ev[1].record()
        _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h1), _lib.ptr(w), n, _lib.ptr(h2), 0,
                                       _lib.ptr(work)))
        ev[2].record()
        _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h2), _lib.ptr(w), n, 0, _lib.ptr(nrm),
                                       _lib.ptr(work)))
        ev[3].record()
        _lib.check(lib.stmhd_gs_normalize(sp_, _lib.ptr(w), _lib.ptr(w), n, _lib.ptr(nrm)))
        ev[4].record()
        torch.cuda.synchronize()
        for i in range(4):
            tot[i] += ev[i].elapsed_time(ev[i + 1])
        if rep == 0:
            chk += float(h1.sum() + 3.0 * h2.sum() + 7.0 * nrm.sum())
    if rep == 0:
        # the basis was orthonormalised in place by the first pass: regenerate for the timed pass
        V = torch.randn(m + 1, n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
print(f"n={n} m={m} checksum {chk!r}")
for nm, t in zip(names, tot):
    print(f"  {nm:12s} {t / m:.3f} ms per step (avg over j=1..{m})")
print(f"  CGS2 total   {sum(tot) / m:.3f} ms per step; one V stream at avg j: {8e-9 * n * (m + 1) / 2:.2f} GB")
