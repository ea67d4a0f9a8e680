"""Layout contract, GPU sparse LU and device FGMRES (drop-ins for reference
``linalg.py``: FieldLayout/BlockVector :14-68, LUFactor :71-96, gmres :99-209).

Vectors are ``torch.float64`` CUDA tensors.  numpy inputs are accepted at the
boundary and copied to the device once.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .errors import BreakdownError, SingularMatrixError

DEV = "cuda"


def as_device(v, device=DEV) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        if v.dtype != torch.float64:
            v = v.to(torch.float64)
        return v if v.is_cuda else v.to(device)
    return torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64), device=device)


@dataclass(frozen=True)
class FieldLayout:
    """Per-slab segment sizes of (u, p, j, A) (reference linalg.py:14-32)."""

    n_u: int
    n_p: int
    n_j: int
    n_a: int

    @property
    def slab_size(self) -> int:
        return self.n_u + self.n_p + self.n_j + self.n_a

    def offsets(self) -> dict:
        o_p = self.n_u
        o_j = o_p + self.n_p
        o_a = o_j + self.n_j
        return {"u": (0, o_p), "p": (o_p, o_j), "j": (o_j, o_a), "A": (o_a, self.slab_size)}


class BlockVector:
    """Slab-major space-time vector on the device; slab/field accessors are
    views (reference linalg.py:35-68)."""

    def __init__(self, layout: FieldLayout, n_steps: int, data=None):
        self.layout, self.n_steps = layout, n_steps
        size = n_steps * layout.slab_size
        if data is None:
            data = torch.zeros(size, dtype=torch.float64, device=DEV)
        data = as_device(data)
        if tuple(data.shape) != (size,):
            raise ValueError(f"data must have shape ({size},), got {tuple(data.shape)}")
        self.data = data
        self._off = layout.offsets()

    def slab(self, step: int):
        s = self.layout.slab_size
        return self.data[step * s:(step + 1) * s]

    def field(self, step: int, name: str):
        lo, hi = self._off[name]
        return self.slab(step)[lo:hi]

    def fields(self, name: str):
        """(n_steps, n_field) strided view of one field over all slabs."""
        lo, hi = self._off[name]
        return self.data.view(self.n_steps, self.layout.slab_size)[:, lo:hi]

    def copy(self) -> "BlockVector":
        return BlockVector(self.layout, self.n_steps, self.data.clone())

    def zeros_like(self) -> "BlockVector":
        return BlockVector(self.layout, self.n_steps)

    def norm(self) -> float:
        return float(torch.linalg.vector_norm(self.data))


class _LUHandle:
    """Owns an stmhd_lu handle (nested-dissection supernodal LU on device)."""

    def __init__(self, csr: sp.csr_matrix, nbatch=1, gx=None, gy=None, leaf=64):
        self.lib = _lib.load()
        csr = sp.csr_matrix(csr)
        csr.sort_indices()
        self.n = csr.shape[0]
        self.rowptr = np.ascontiguousarray(csr.indptr, dtype=np.int32)
        self.col = np.ascontiguousarray(csr.indices, dtype=np.int32)
        gx = None if gx is None else np.ascontiguousarray(gx, dtype=np.int32)
        gy = None if gy is None else np.ascontiguousarray(gy, dtype=np.int32)
        h = _lib.c_vp()
        _lib.check(self.lib.stmhd_lu_create(self.n, _lib.ptr(self.rowptr), _lib.ptr(self.col),
                                            _lib.ptr(gx), _lib.ptr(gy), nbatch, leaf, C_byref(h)))
        self.h = h
        self.nbatch = nbatch

    def info(self):
        out = np.zeros(5, dtype=np.int64)
        _lib.check(self.lib.stmhd_lu_info(self.h, _lib.ptr(out)))
        return dict(factor_doubles=int(out[0]), supernodes=int(out[1]), levels=int(out[2]),
                    max_front=int(out[3]), sym_nnz=int(out[4]))

    def factor(self, values: torch.Tensor, stride: int):
        st = self.lib.stmhd_lu_factor(self.h, _lib.stream_ptr(), _lib.ptr(values), stride, 0)
        if st == 2:
            raise SingularMatrixError((self.lib.stmhd_last_error() or b"").decode())
        _lib.check(st)

    def solve(self, rhs: torch.Tensor, out: torch.Tensor, nrhs: int, ld_rhs: int, ld_x: int):
        _lib.check(self.lib.stmhd_lu_solve(self.h, _lib.stream_ptr(), _lib.ptr(rhs), ld_rhs,
                                           _lib.ptr(out), ld_x, nrhs))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.stmhd_lu_destroy(self.h)
        except Exception:
            pass


def C_byref(h):
    import ctypes

    return ctypes.byref(h)


class LUFactor:
    """Drop-in for reference ``LUFactor`` (linalg.py:71-96): a sparse LU of one
    matrix on the device.  Zero pivots (after partial pivoting inside the
    supernode blocks) raise ``SingularMatrixError``; non-finite solves too."""

    def __init__(self, matrix, coords=None, leaf=64):
        mat = sp.csr_matrix(matrix, dtype=np.float64)
        mat.sort_indices()
        if mat.shape[0] != mat.shape[1]:
            raise ValueError("LUFactor needs a square matrix")
        gx, gy = (None, None) if coords is None else coords
        self._h = _LUHandle(mat, 1, gx, gy, leaf)
        self.shape = mat.shape
        self._vals = torch.as_tensor(mat.data, device=DEV)
        self._h.factor(self._vals, 0)

    def solve(self, b):
        was_np = not isinstance(b, torch.Tensor)
        bd = as_device(b).contiguous()
        nrhs = 1 if bd.dim() == 1 else bd.shape[1]
        if bd.dim() == 2:
            bd = bd.t().contiguous()
        x = torch.empty_like(bd)
        self._h.solve(bd, x, nrhs, self.shape[0], self.shape[0])
        if not bool(torch.isfinite(x).all()):
            raise SingularMatrixError("LU solve produced non-finite values")
        if bd.dim() == 2 and nrhs > 1:
            x = x.t()
        return x.cpu().numpy() if was_np else x


def lu_factor(matrix) -> LUFactor:
    return LUFactor(matrix)


# -- device FGMRES ------------------------------------------------------------------


@dataclass
class GmresConfig:
    rel_tol: float = 1e-2
    abs_tol: float = 1e-14
    max_iters: int = 200
    restart: int | None = None  # None = full GMRES

    def __post_init__(self):
        if self.rel_tol <= 0 or self.abs_tol <= 0:
            raise ValueError("tolerances must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")


@dataclass
class GmresResult:
    x: torch.Tensor
    iterations: int
    residuals: list = field(default_factory=list)
    converged: bool = True
    true_residual: float = 0.0


def _fast(fn):
    """(object, method) for callbacks that can write into a given buffer."""
    obj = getattr(fn, "__self__", None)
    if obj is not None and hasattr(obj, "_into") and getattr(fn, "__name__", "") in ("apply", "apply_inverse"):
        return obj
    return None


class _Workspace:
    """Krylov basis storage reused across gmres calls of the same size."""

    cache: dict = {}

    @classmethod
    def get(cls, n, m):
        key = (n, m)
        ws = cls.cache.get(key)
        if ws is None:
            cls.cache.clear()
            lib = _lib.load()
            ws = dict(V=torch.empty((m + 1, n), dtype=torch.float64, device=DEV),
                      Z=torch.empty((m, n), dtype=torch.float64, device=DEV),
                      dev=torch.zeros(2 * (m + 2), dtype=torch.float64, device=DEV),
                      host=torch.zeros(2 * (m + 2), dtype=torch.float64).pin_memory(),
                      host2=torch.zeros(2 * (m + 2), dtype=torch.float64).pin_memory(),
                      ev=[torch.cuda.Event(), torch.cuda.Event()],
                      work=torch.empty(int(lib.stmhd_gs_work_size(n, m + 1)) + 8, dtype=torch.float64, device=DEV),
                      y=torch.zeros(m, dtype=torch.float64, device=DEV),
                      r=torch.empty(n, dtype=torch.float64, device=DEV))
            cls.cache[key] = ws
        return ws


def gmres(apply_a, apply_pinv, b, x0=None, config: GmresConfig | None = None) -> GmresResult:
    """Right-preconditioned restarted FGMRES on the device (reference
    linalg.py:122-209 semantics: x0 = 0 unless given, tol = max(rel |r0|, abs)
    fixed at entry, Givens rotations, restart residual recomputed, true
    residual at exit).  Orthogonalisation is CGS2 with fused multi-vector
    kernels; the preconditioned basis Z is stored, so the cycle update is
    x += Z y (no extra preconditioner apply)."""
    cfg = config or GmresConfig()
    lib = _lib.load()
    sp_ = _lib.stream_ptr()
    b = as_device(b).contiguous()
    n = b.numel()
    if not bool(torch.isfinite(b).all()):
        raise BreakdownError("right-hand side contains non-finite values")
    ident = apply_pinv is None
    fa, fp = _fast(apply_a), (None if ident else _fast(apply_pinv))

    def A_into(v, out):
        if fa is not None:
            return fa._into(v, out)
        out.copy_(as_device(apply_a(v)).reshape(-1))
        return out

    def P_into(v, out):
        if ident:
            out.copy_(v)
        elif fp is not None:
            fp._into(v, out)
        else:
            out.copy_(as_device(apply_pinv(v)).reshape(-1))
        return out

    restart = cfg.restart or cfg.max_iters
    m_alloc = min(restart, cfg.max_iters)
    ws = _Workspace.get(n, m_alloc)
    V, Z, dev, host, work, ydev, r = ws["V"], ws["Z"], ws["dev"], ws["host"], ws["work"], ws["y"], ws["r"]
    x = torch.zeros(n, dtype=torch.float64, device=DEV) if x0 is None else as_device(x0).clone().reshape(-1)
    if x0 is not None:
        A_into(x, r)
        r.neg_().add_(b)
    else:
        r.copy_(b)
    beta = float(torch.linalg.vector_norm(r))
    residuals = [beta]
    tol = max(cfg.rel_tol * beta, cfg.abs_tol)
    if beta <= tol:
        return GmresResult(x, 0, residuals, True, beta)
    total, converged = 0, False
    while total < cfg.max_iters and not converged:
        m = min(restart, cfg.max_iters - total)
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        torch.div(r, beta, out=V[0])
        g[0] = beta
        last = -1
        hosts = (ws["host"], ws["host2"])
        evs = ws["ev"]

        def process(jj):
            """Givens update of column jj (its Hessenberg entries are in hosts[jj % 2]);
            returns True when the cycle stops at jj (converged or breakdown)."""
            nonlocal total, last, converged
            evs[jj % 2].synchronize()
            hv = hosts[jj % 2].numpy()
            nv = jj + 1
            col = hv[:nv] + hv[m_alloc + 1: m_alloc + 1 + nv]
            nrm2 = hv[2 * m_alloc + 3]
            if not (np.all(np.isfinite(col)) and np.isfinite(nrm2)):
                raise BreakdownError("non-finite vector in Arnoldi process")
            hnorm = float(np.sqrt(max(nrm2, 0.0)))
            H[:nv, jj] = col
            H[jj + 1, jj] = hnorm
            for i in range(jj):
                t = cs[i] * H[i, jj] + sn[i] * H[i + 1, jj]
                H[i + 1, jj] = -sn[i] * H[i, jj] + cs[i] * H[i + 1, jj]
                H[i, jj] = t
            den = np.hypot(H[jj, jj], H[jj + 1, jj])
            cs[jj], sn[jj] = H[jj, jj] / den, H[jj + 1, jj] / den
            H[jj, jj] = den
            H[jj + 1, jj] = 0.0
            g[jj + 1] = -sn[jj] * g[jj]
            g[jj] = cs[jj] * g[jj]
            total += 1
            last = jj
            residuals.append(abs(float(g[jj + 1])))
            if residuals[-1] <= tol:
                converged = True
                return True
            return den == 0.0

        # The host Givens update of column j-1 runs while iteration j is already on the
        # device (one-iteration lag): the GPU never waits for the host.  Numbers are
        # identical to the unlagged loop; a cycle that stops at j-1 discards iteration j.
        stopped = False
        for j in range(m):
            P_into(V[j], Z[j])
            w = V[j + 1]
            A_into(Z[j], w)
            nv = j + 1
            h1, h2, nrm = dev[:nv], dev[m_alloc + 1: m_alloc + 1 + nv], dev[2 * m_alloc + 3: 2 * m_alloc + 4]
            _lib.check(lib.stmhd_gs_dots(sp_, _lib.ptr(V), n, nv, _lib.ptr(w), n, _lib.ptr(h1), _lib.ptr(work)))
            _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h1), _lib.ptr(w), n, _lib.ptr(h2),
                                           0, _lib.ptr(work)))
            _lib.check(lib.stmhd_gs_update(sp_, _lib.ptr(V), n, nv, _lib.ptr(h2), _lib.ptr(w), n, 0,
                                           _lib.ptr(nrm), _lib.ptr(work)))
            hosts[j % 2].copy_(dev, non_blocking=True)
            evs[j % 2].record()
            _lib.check(lib.stmhd_gs_normalize(sp_, _lib.ptr(w), _lib.ptr(w), n, _lib.ptr(nrm)))
            if j > 0 and process(j - 1):
                stopped = True
                break
        if not stopped:
            process(m - 1)
        if last >= 0:
            y = np.zeros(last + 1)
            for i in range(last, -1, -1):
                y[i] = (g[i] - H[i, i + 1:last + 1] @ y[i + 1:last + 1]) / H[i, i]
            ydev[: last + 1].copy_(torch.from_numpy(y))
            _lib.check(lib.stmhd_gs_combine(sp_, _lib.ptr(Z), n, last + 1, _lib.ptr(ydev), _lib.ptr(x), n))
        if converged:
            break
        A_into(x, r)
        r.neg_().add_(b)
        beta = float(torch.linalg.vector_norm(r))
        if beta <= tol:
            converged = True
            break
    A_into(x, r)
    r.neg_().add_(b)
    true_res = float(torch.linalg.vector_norm(r))
    # a pipelined preconditioner launch that timed out (stages not co-resident) is
    # reported here instead of trapping on the device
    _lib.check(lib.stmhd_device_fault(sp_))
    return GmresResult(x, total, residuals, converged, true_res)
