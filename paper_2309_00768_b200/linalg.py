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
