"""Where an FGMRES iteration's time goes on C2 (device-timed): P_T^-1 + J.v alone,
plus the CGS2 kernels, and the full gmres() loop (host Givens, copies, syncs)."""
import sys
import time

import torch

import paper_2309_00768_b200 as p
from paper_2309_00768_b200 import _lib

d = p.discretize_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
st = p.initial_state(d)
r = p.residual(st, d)
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
n = jac.size
lib = _lib.load()
sp_ = _lib.stream_ptr()
m = 50
V = torch.randn(m + 1, n, dtype=torch.float64, device="cuda")
Z = torch.empty(m, n, dtype=torch.float64, device="cuda")
dev = torch.zeros(2 * m + 8, dtype=torch.float64, device="cuda")
work = torch.empty(int(lib.stmhd_gs_work_size(n, m + 1)) + 8, dtype=torch.float64, device="cuda")
pc._into(V[0], Z[0])
jac._into(Z[0], V[1])
torch.cuda.synchronize()


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(reps):
        fn(j)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def pj(j):
    pc._into(V[j % m], Z[j % m])
    jac._into(Z[j % m], V[j % m + 1])


def gs(j):
    nv = j % m + 1
    w = V[nv]
    h1, h2, nrm = dev[:nv], dev[m + 1: m + 1 + nv], dev[2 * m + 3: 2 * m + 4]
    _lib.check(lib.stmhd_gs_dots(sp_, _lib.ptr(V), n, nv, _lib.ptr(w), n, _lib.ptr(h1), _lib.ptr(work)))
    _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h1), _lib.ptr(w), n, _lib.ptr(h2), 0,
                                   _lib.ptr(work)))
    _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h2), _lib.ptr(w), n, 0, _lib.ptr(nrm),
                                   _lib.ptr(work)))
    _lib.check(lib.stmhd_gs_normalize(sp_, _lib.ptr(w), _lib.ptr(w), n, _lib.ptr(nrm)))


print(f"P+J per iteration      {timed(pj, 50):.3f} ms")
print(f"CGS2 (avg j=25)        {timed(gs, 50):.3f} ms")
print(f"P+J+CGS2               {timed(lambda j: (pj(j), gs(j)), 50):.3f} ms")
cfg = p.GmresConfig(rel_tol=1e-14, abs_tol=1e-300, max_iters=100, restart=50)
b = -r.data
p.gmres(jac.apply, pc.apply_inverse, b, config=cfg)
torch.cuda.synchronize()
t = time.perf_counter()
res = p.gmres(jac.apply, pc.apply_inverse, b, config=cfg)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"gmres loop             {1e3 * dt / res.iterations:.3f} ms per iteration ({res.iterations} iterations)")
