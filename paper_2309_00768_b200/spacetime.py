"""All-at-once residual and space-time Jacobian on the device (drop-in for
reference ``spacetime.py``: SpaceTimeState :26-39, residual :65-85,
SlabBlocks/linearize_slab :88-112, SpaceTimeJacobian :115-164,
assemble_jacobian :167-175, apply_jacobian :178-183)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib
from .linalg import BlockVector, as_device


@dataclass
class SpaceTimeState:
    """Field values on slabs 1..N_t plus the time-zero initial condition."""

    vec: BlockVector
    ic_u: torch.Tensor
    ic_a: torch.Tensor

    @property
    def n_steps(self) -> int:
        return self.vec.n_steps

    def copy(self) -> "SpaceTimeState":
        return SpaceTimeState(self.vec.copy(), self.ic_u.clone(), self.ic_a.clone())


def _bind_nt(disc, nt):
    """The native handle sizes every call by its current slab count."""
    if disc._bound_nt != nt:
        _lib.check(_lib.load().stmhd_disc_set_int(disc.handle, b"nt", int(nt)))
        disc._bound_nt = nt


def _assemble(state: SpaceTimeState, disc, residual=None, js=None, fp=None, alf=None):
    _bind_nt(disc, state.n_steps)
    lib = _lib.load()
    _lib.check(lib.stmhd_assemble(disc.handle, _lib.stream_ptr(), _lib.ptr(state.vec.data),
                                  _lib.ptr(state.ic_u), _lib.ptr(state.ic_a), _lib.ptr(residual),
                                  _lib.ptr(js), _lib.ptr(fp), _lib.ptr(alf)))


def residual(state: SpaceTimeState, disc) -> BlockVector:
    """Backward-Euler residual of every slab with constraint rows (K1)."""
    out = torch.empty_like(state.vec.data)
    _assemble(state, disc, residual=out)
    return BlockVector(disc.layout, state.n_steps, out)


@dataclass
class SlabBlocks:
    """Linearised blocks of one slab as scipy CSR views (tests / inspection)."""

    f_u: sp.csr_matrix
    z_j: sp.csr_matrix
    z_a: sp.csr_matrix
    y: sp.csr_matrix
    f_a: sp.csr_matrix


class SpaceTimeJacobian:
    """Per-slab values in the fixed merged pattern + shared couplings on the
    device.  ``apply`` is one batched SpMV launch over all slabs (K2)."""

    def __init__(self, disc, values: torch.Tensor, fp_values: torch.Tensor, alfven: torch.Tensor,
                 n_steps: int):
        self.disc = disc
        self.values = values
        self.fp_values = fp_values
        self.alfven = alfven
        self.n_steps = n_steps
        self.layout = disc.layout
        self.size = n_steps * disc.layout.slab_size
        self.block_multiplies = 0
        self._slabs = None
        self._sell = None

    def _sell_values(self):
        """Sliced-ELL copy of the slab values (stmhd_jac_relayout), made at the first
        apply; ``values`` is not modified after assembly (the reference builds fresh
        matrices, spacetime.py:167-175)."""
        if self._sell is None:
            lib = _lib.load()
            _bind_nt(self.disc, self.n_steps)
            n = lib.stmhd_jac_sell_size(self.disc.handle, _lib.stream_ptr())
            if n < 0:
                _lib.check(1)
            self._sell = torch.empty((self.n_steps, n), dtype=torch.float64, device=self.values.device)
            _lib.check(lib.stmhd_jac_relayout(self.disc.handle, _lib.stream_ptr(), _lib.ptr(self.values),
                                              _lib.ptr(self._sell)))
        return self._sell

    def _into(self, v: torch.Tensor, out: torch.Tensor):
        sell = self._sell_values()
        _bind_nt(self.disc, self.n_steps)
        _lib.check(_lib.load().stmhd_jac_apply_sell(self.disc.handle, _lib.stream_ptr(), _lib.ptr(sell),
                                                    _lib.ptr(v), _lib.ptr(out)))
        self.block_multiplies += 8 * self.n_steps + 2 * (self.n_steps - 1)
        return out

    def apply(self, v):
        v = as_device(v).contiguous()
        return self._into(v, torch.empty_like(v))

    @property
    def slabs(self):
        if self._slabs is None:
            self._slabs = [linearized_blocks(self.disc, self.values[k].cpu().numpy())
                           for k in range(self.n_steps)]
        return self._slabs

    def to_dense(self) -> np.ndarray:
        n = self.size
        out = np.empty((n, n))
        e = torch.zeros(n, dtype=torch.float64, device="cuda")
        for i in range(n):
            e[i] = 1.0
            out[:, i] = self.apply(e).cpu().numpy()
            e[i] = 0.0
        return out


def linearized_blocks(disc, vals: np.ndarray) -> SlabBlocks:
    """scipy views of one slab's f_u, z_j, z_a, y, f_a from its value row."""
    P, L = disc.pattern, disc.layout
    o_p, o_j, o_a = P.offsets
    return SlabBlocks(
        f_u=P.to_csr(vals, 0, L.n_u, 0, 0, L.n_u),
        z_j=P.to_csr(vals, 0, L.n_u, 1, o_j, o_j + L.n_j),
        z_a=P.to_csr(vals, 0, L.n_u, 2, o_a, o_a + L.n_a),
        y=P.to_csr(vals, o_a, o_a + L.n_a, 0, 0, L.n_u),
        f_a=P.to_csr(vals, o_a, o_a + L.n_a, 1, o_a, o_a + L.n_a),
    )


def linearize_slab(disc, u, j, a) -> SlabBlocks:
    """Blocks of one slab at given (clamped) fields (reference spacetime.py:99-112)."""
    L = disc.layout
    slab = torch.zeros(L.slab_size, dtype=torch.float64, device="cuda")
    o = L.offsets()
    slab[o["u"][0]:o["u"][1]] = as_device(u)
    slab[o["j"][0]:o["j"][1]] = as_device(j)
    slab[o["A"][0]:o["A"][1]] = as_device(a)
    st = SpaceTimeState(BlockVector(L, 1, slab), torch.zeros(L.n_u, dtype=torch.float64, device="cuda"),
                        as_device(a).clone())
    jac = assemble_jacobian(st, disc)
    return jac.slabs[0]


def assemble_jacobian(state: SpaceTimeState, disc) -> SpaceTimeJacobian:
    """Linearise at the given state, all slabs in one launch (K1)."""
    nt = state.n_steps
    P = disc.pattern
    js = torch.empty((nt, P.nnz), dtype=torch.float64, device="cuda")
    fp = torch.empty((nt, P.fp_nnz), dtype=torch.float64, device="cuda")
    alf = torch.empty(nt, dtype=torch.float64, device="cuda")
    _assemble(state, disc, js=js, fp=fp, alf=alf)
    return SpaceTimeJacobian(disc, js, fp, alf, nt)


def apply_jacobian(jacobian: SpaceTimeJacobian, v):
    if isinstance(v, BlockVector):
        return BlockVector(jacobian.layout, jacobian.n_steps, jacobian.apply(v.data))
    return jacobian.apply(v)
