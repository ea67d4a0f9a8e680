"""Space-time block preconditioner on the device (drop-in for reference
``precond.py``: Variant :40-43, compute_alfven_scaling :46-57,
SpaceTimePreconditioner :60-387).

Setup (one native call) builds C_A,k and the wave sub-diagonals with fixed
gather plans and factors F_u,k and C_A,k for every slab with the batched
nested-dissection LU; applications chain batched exact solves, bidiagonal
SpMVs and the two sequential time sweeps in the reference order.
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .errors import PreconditionerError
from .linalg import as_device
from .spacetime import SpaceTimeJacobian, _assemble, _bind_nt


class Variant(str, Enum):
    FULL = "full"
    SIMPLIFIED = "simplified"
    TRIANGULAR = "triangular"


_VARIANT_CODE = {Variant.TRIANGULAR: 0, Variant.SIMPLIFIED: 1, Variant.FULL: 2}

OPS = {"solve_velocity": (0, "u"), "apply_velocity": (1, "u"), "solve_wave": (2, "A"),
       "apply_wave": (3, "A"), "apply_potential": (4, "A"), "solve_potential": (5, "A"),
       "pressure_schur_inverse": (6, "p"), "pressure_schur_apply": (7, "p"),
       "magnetic_schur_inverse": (8, "A"), "magnetic_schur_apply": (9, "A"),
       "apply_pressure_cd": (10, "p"), "solve_pressure_cd": (11, "p")}


def compute_alfven_scaling(pot_space, a_coefs, mu0: float) -> np.ndarray:
    """||mean grad A_k||^2 / mu0 per row of a_coefs (reference precond.py:46-57).
    Host helper on P1 coefficient vectors (the Newton path computes it on the
    device inside assembly)."""
    a_coefs = np.atleast_2d(np.asarray(a_coefs.cpu() if isinstance(a_coefs, torch.Tensor) else a_coefs,
                                       dtype=float))
    m = pot_space.mesh
    from .fem import orientation_maps

    _, invs = orientation_maps(m.hx, m.hy)
    # P1 reference gradients of (1-x-y, x, y) mapped by invJ (rows r, cols d)
    gref = np.array([[-1.0, -1.0], [1.0, 0.0], [0.0, 1.0]])
    g = np.stack([gref @ inv for inv in invs])  # (2, 3, 2)
    o = np.arange(m.ne) & 1
    out = np.empty(len(a_coefs))
    for k, a in enumerate(a_coefs):
        ae = a[pot_space.elem]
        grads = np.einsum("en,end->ed", ae, g[o])
        mean = grads.sum(axis=0) * (0.5 * m.hx * m.hy) / m.area
        out[k] = float(mean @ mean) / mu0
    return out


class SpaceTimePreconditioner:
    """Factorised blocks at one Newton linearisation point (device)."""

    def __init__(self, jacobian: SpaceTimeJacobian, disc, state, variant=Variant.TRIANGULAR):
        self.disc = disc
        self.jac = jacobian
        self.variant = Variant(variant)
        self.n_steps = jacobian.n_steps
        self.layout = disc.layout
        nt = self.n_steps
        P = disc.pattern
        # F_p and the Alfven scaling come from `state` (precond.py:80-90)
        self.fp_values = torch.empty((nt, P.fp_nnz), dtype=torch.float64, device="cuda")
        self._alf = torch.empty(nt, dtype=torch.float64, device="cuda")
        _assemble(state, disc, fp=self.fp_values, alf=self._alf)
        _bind_nt(disc, nt)
        lib = _lib.load()
        h = ctypes.c_void_p()
        st = lib.stmhd_pc_create(disc.handle, _lib.stream_ptr(), _lib.ptr(jacobian.values),
                                 _lib.ptr(self.fp_values), _lib.ptr(self._alf),
                                 _VARIANT_CODE[self.variant], ctypes.byref(h))
        if st == 2:
            blk = (lib.stmhd_last_block() or b"").decode() or "F_u"
            raise PreconditionerError(blk, (lib.stmhd_last_error() or b"").decode())
        _lib.check(st)
        self._h = h
        self._lib = lib

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._lib.stmhd_pc_destroy(self._h)
        except Exception:
            pass

    # -- inspection (tests) ----------------------------------------------------------
    @property
    def alfven(self) -> np.ndarray:
        return self._alf.cpu().numpy()

    def _export(self, what, shape):
        out = torch.empty(shape, dtype=torch.float64, device="cuda")
        _lib.check(self._lib.stmhd_pc_export(self._h, _lib.stream_ptr(), what, _lib.ptr(out)))
        return out.cpu().numpy()

    @property
    def c_a(self):
        rp, col = self.disc._ca_pattern
        n = self.layout.n_a
        vals = self._export(0, (self.n_steps, len(col)))
        return [sp.csr_matrix((vals[k], col, rp), shape=(n, n)) for k in range(self.n_steps)]

    @property
    def c_a_sub1(self):
        rp, col = self.disc._s1_pattern
        n = self.layout.n_a
        if self.n_steps < 2:
            return []
        vals = self._export(1, (self.n_steps - 1, len(col)))
        return [sp.csr_matrix((vals[k], col, rp), shape=(n, n)) for k in range(self.n_steps - 1)]

    @property
    def pivot_ratio(self) -> dict:
        """Smallest restricted-pivoting ratio of the F_u and C~_A factorisations:
        |pivot| / max |entry of its column below the diagonal|, contribution-block rows
        included (the pivot search is restricted to the supernode's diagonal block; 1
        means as good as unrestricted partial pivoting).  A ratio below 1e-8 is also
        reported on stderr by the native library (STMHD_PIVOT_WARN)."""
        v = self._export(3, (2,))
        return {"F_u": float(v[0]), "C_A": float(v[1])}

    @property
    def c_a_sub2(self):
        return self.disc.c_a_sub2

    @property
    def f_p(self):
        P = self.disc.pattern
        n = self.layout.n_p
        v = self.fp_values.cpu().numpy()
        return [sp.csr_matrix((v[k], P.fp_col, P.fp_rowptr), shape=(n, n)) for k in range(self.n_steps)]

    # -- applications -------------------------------------------------------------------
    def _into(self, r: torch.Tensor, out: torch.Tensor, direction=0):
        _lib.check(self._lib.stmhd_pc_apply(self._h, _lib.stream_ptr(), direction, _lib.ptr(r), _lib.ptr(out)))
        return out

    def apply_inverse(self, r):
        """P^{-1} r for the selected variant (precond.py:270-301)."""
        r = as_device(r).contiguous()
        return self._into(r, torch.empty_like(r), 0)

    def apply_forward(self, x):
        """P x (round-trip checks, precond.py:303-340)."""
        x = as_device(x).contiguous()
        return self._into(x, torch.empty_like(x), 1)

    # -- single time-step counterpart (precond.py:344-387) -----------------------------
    def _single(self, k, v, direction):
        """Slab k of the space-time operator applied to e_k (x) v.  P_T^{-1} is block
        lower triangular in time and P_T block lower bidiagonal, so with zero input
        in every other slab this is exactly the single-step operator of slab k
        (no time coupling) -- computed with the same device kernels."""
        if not 0 <= k < self.n_steps:
            raise IndexError(f"slab {k} out of range 0..{self.n_steps - 1}")
        L = self.layout.slab_size
        full = torch.zeros(self.n_steps * L, dtype=torch.float64, device="cuda")
        full[k * L:(k + 1) * L] = as_device(v).reshape(-1)
        # directions 2/3 force the TRIANGULAR operator: the reference's single-step
        # preconditioner ignores the variant (precond.py:344-387)
        out = self._into(full, torch.empty_like(full), direction + 2)
        return out[k * L:(k + 1) * L].clone()

    def apply_single_step_inverse(self, k: int, r_slab):
        """Back-substitution of the single-step preconditioner at slab k (precond.py:344-366)."""
        return self._single(k, r_slab, 0)

    def apply_single_step(self, k: int, x_slab):
        """Forward application of the single-step preconditioner at slab k (precond.py:368-387)."""
        return self._single(k, x_slab, 1)

    def _op(self, name, v):
        code, field = OPS[name]
        v = as_device(v).contiguous()
        out = torch.empty_like(v)
        _lib.check(self._lib.stmhd_pc_op(self._h, _lib.stream_ptr(), code, _lib.ptr(v), _lib.ptr(out)))
        return out

    def solve_velocity(self, r):
        return self._op("solve_velocity", r)

    def apply_velocity(self, v):
        return self._op("apply_velocity", v)

    def apply_pressure_cd(self, v):
        return self._op("apply_pressure_cd", v)

    def solve_pressure_cd(self, r):
        return self._op("solve_pressure_cd", r)

    def apply_potential(self, v):
        return self._op("apply_potential", v)

    def solve_potential(self, r):
        return self._op("solve_potential", r)

    def apply_wave(self, v):
        return self._op("apply_wave", v)

    def solve_wave(self, r):
        return self._op("solve_wave", r)

    def pressure_schur_inverse(self, r):
        return self._op("pressure_schur_inverse", r)

    def pressure_schur_apply(self, x):
        return self._op("pressure_schur_apply", x)

    def magnetic_schur_inverse(self, r):
        return self._op("magnetic_schur_inverse", r)

    def magnetic_schur_apply(self, x):
        return self._op("magnetic_schur_apply", x)
