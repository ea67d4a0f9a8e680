"""Configuration-5 synthetic inputs: the per-slab
divergence-free advection fields of the scalar advection-diffusion
micro-benchmark.

For each slab k, in order, from one ``np.random.default_rng(seed)``:
``kx, ky = rng.integers(1, 9, size=(8, 2))`` and ``a = rng.standard_normal(8)``;
psi_k = sum_m a_m sin(pi kx_m (x+1)/2) sin(pi ky_m (y+1)/2),
u_k = (d psi/dy, -d psi/dx) at the P1 nodes, scaled so max_node |u_k| = 1.
The same function feeds the GPU run, the CPU oracle and the golden fixture.
"""

from __future__ import annotations

import numpy as np


def c5_modes(nt: int, seed: int = 0) -> np.ndarray:
    """(nt, 8, 3) per-slab modes {kx, ky, amplitude} in the generator's draw order."""
    rng = np.random.default_rng(seed)
    out = np.empty((nt, 8, 3))
    for k in range(nt):
        out[k, :, :2] = rng.integers(1, 9, size=(8, 2))
        out[k, :, 2] = rng.standard_normal(8)
    return out


def c5_velocity_fields_device(coords: np.ndarray, nt: int, seed: int = 0):
    """The same fields as c5_velocity_fields, evaluated on the device
    (stmhd_c5_velocity): a (nt, n_nodes, 2) CUDA tensor."""
    import torch

    from . import _lib
    from .linalg import DEV

    xy = torch.as_tensor(np.ascontiguousarray(coords, dtype=np.float64), device=DEV)
    md = np.ascontiguousarray(c5_modes(nt, seed))
    u = torch.empty((nt, len(coords), 2), dtype=torch.float64, device=DEV)
    _lib.check(_lib.load().stmhd_c5_velocity(_lib.stream_ptr(), len(coords), nt, _lib.ptr(xy), md.ctypes.data,
                                             _lib.ptr(u)))
    return u


def c5_velocity_fields(coords: np.ndarray, nt: int, seed: int = 0) -> np.ndarray:
    """(nt, n_nodes, 2) nodal velocities for the slabs 0..nt-1 (host reference)."""
    rng = np.random.default_rng(seed)
    x = coords[:, 0] + 1.0
    y = coords[:, 1] + 1.0
    out = np.empty((nt, len(coords), 2))
    for k in range(nt):
        kk = rng.integers(1, 9, size=(8, 2))
        amp = rng.standard_normal(8)
        ux = np.zeros(len(coords))
        uy = np.zeros(len(coords))
        for (kx, ky), a in zip(kk, amp):
            sx, cx = np.sin(0.5 * np.pi * kx * x), np.cos(0.5 * np.pi * kx * x)
            sy, cy = np.sin(0.5 * np.pi * ky * y), np.cos(0.5 * np.pi * ky * y)
            ux += a * sx * (0.5 * np.pi * ky) * cy
            uy -= a * (0.5 * np.pi * kx) * cx * sy
        scale = np.sqrt(ux * ux + uy * uy).max()
        out[k, :, 0] = ux / scale
        out[k, :, 1] = uy / scale
    return out


def c5_host_tables(n: int, dt: float = 1e-2, eps: float = 1e-3) -> dict:
    """Host side of the configuration-5 operator: the fixed pattern (element couplings,
    Dirichlet rows and columns reduced to the diagonal as bc_identity leaves them), the constant
    part M/dt + eps K per entry, every entry's element contributions
    {element, local row, local col, orientation} for the device advection assembly, the
    P1 element mass / gradient tensors, and C = bc_zero(M/dt)."""
    import scipy.sparse as sp

    from . import fem

    mesh = fem.Mesh(-1.0, 1.0, -1.0, 1.0, n, n)
    p1 = fem.Space(mesh, 1)
    nn = p1.n_nodes
    T = fem.element_tensors(1, 1, mesh.hx, mesh.hy)
    bc = np.unique(np.concatenate([p1.side_nodes["top"], p1.side_nodes["bottom"]]))
    isbc = np.zeros(nn, dtype=bool)
    isbc[bc] = True
    el = p1.elem
    ne = len(el)
    rows = np.repeat(el[:, :, None], 3, axis=2).ravel()
    cols = np.repeat(el[:, None, :], 3, axis=1).ravel()
    keys = np.unique(rows * nn + cols)
    # bc_identity clears the rows AND columns of Dirichlet nodes, then sets the diagonal
    keys = keys[(~isbc[keys // nn] & ~isbc[keys % nn]) | (keys // nn == keys % nn)]
    keys = np.union1d(keys, bc * nn + bc)
    prow, pcol = keys // nn, keys % nn
    nnz = len(keys)
    o = np.arange(ne) & 1
    li = np.tile(np.repeat(np.arange(3), 3), ne)
    lj = np.tile(np.tile(np.arange(3), 3), ne)
    eid = np.repeat(np.arange(ne), 9)
    keep = ~isbc[rows] & ~isbc[cols]
    ent = np.searchsorted(keys, rows * nn + cols)
    # constant part M/dt + eps K: assembled on the device (fem._assemble, csrc/constops.cu),
    # picked at the entries bc_identity keeps
    a0 = fem._assemble(p1, p1, np.asarray(T["M1"])[None, :, :] / dt + eps * np.asarray(T["K1"]))
    akeys = np.repeat(np.arange(nn, dtype=np.int64), np.diff(a0.indptr)) * nn + a0.indices
    base = a0.data[np.searchsorted(akeys, keys)]
    base[isbc[prow] | isbc[pcol]] = 0.0
    base[np.searchsorted(keys, bc * nn + bc)] = 1.0
    order = np.argsort(ent[keep], kind="stable")
    ce = ent[keep][order]
    cinfo = np.column_stack([eid[keep][order], li[keep][order], lj[keep][order], o[eid[keep][order]]])
    m = fem._assemble(p1, p1, [T["M1"], T["M1"]]).tocsr()
    keepc = sp.diags((~isbc).astype(float))
    cmat = (keepc @ (m / dt) @ keepc).tocsr()
    cmat.eliminate_zeros()
    cmat.sort_indices()
    return dict(p1=p1, bc=bc, nnz=nnz, rowptr=np.searchsorted(prow, np.arange(nn + 1)).astype(np.int32),
                col=pcol.astype(np.int32), base=base, cptr=np.searchsorted(ce, np.arange(nnz + 1)).astype(np.int32),
                cinfo=cinfo.astype(np.int32),
                mloc=np.ascontiguousarray(np.asarray(T["M1"], dtype=np.float64).reshape(-1)),
                grad=np.ascontiguousarray(np.asarray(T["G1"], dtype=np.float64).reshape(-1)), coupling=cmat)


class C5Operator:
    """Configuration-5 scalar advection-diffusion space-time block on the device
    (SURVEY 8(d)); the same interface as the CPU restatement ``oracle/c5.py C5``.

    Per slab F_k = M/dt + eps K + W(u_k) on a P1 space of the n x n mesh of [-1,1]^2
    (W: reference fem.py:430-462, ``lin_a`` with a P1 vector velocity), Dirichlet
    rows/columns of the top/bottom nodes replaced by the identity (fem.py:593-600); sub-diagonal -C with
    C = bc_zero(M/dt) (fem.py:603-610).  ``apply`` is the block-bidiagonal batched
    SpMV, ``solve`` the exact inverse by sequential block forward substitution
    (reference solve_potential, precond.py:173-180) on the cluster sweep, with one
    nested-dissection LU per slab."""

    def __init__(self, n: int, nt: int, ufields=None, seed: int = 0, dt: float = 1e-2, eps: float = 1e-3,
                 leaf: int = 32):
        import torch

        from . import _lib
        from .linalg import DEV, _LUHandle

        self.n_cells, self.nt, self.dt, self.eps = n, nt, dt, eps
        h = c5_host_tables(n, dt, eps)
        p1 = h["p1"]
        self.p1, self.n, self.bc, self.nnz = p1, p1.n_nodes, h["bc"], h["nnz"]
        self.rowptr, self.col, self.coupling = h["rowptr"], h["col"], h["coupling"]
        self._mloc, self._grad = h["mloc"], h["grad"]
        base, cptr, cinfo, el, cmat = h["base"], h["cptr"], h["cinfo"], p1.elem, h["coupling"]
        tens = lambda a, dt_=torch.int32: torch.as_tensor(np.ascontiguousarray(a), dtype=dt_, device=DEV)
        self._d = dict(rowptr=tens(self.rowptr), col=tens(self.col), base=tens(base, torch.float64),
                       cptr=tens(cptr), cinfo=tens(cinfo.astype(np.int32)), elem=tens(el.astype(np.int32)),
                       c_rowptr=tens(cmat.indptr.astype(np.int32)), c_col=tens(cmat.indices.astype(np.int32)),
                       c_val=tens(cmat.data, torch.float64))
        if ufields is None:  # seeded fields, generated on the device
            self.u = c5_velocity_fields_device(p1.coords, nt, seed)
        else:
            self.u = torch.as_tensor(np.ascontiguousarray(ufields, dtype=np.float64), device=DEV)
        self.values = torch.empty(nt * self.nnz, dtype=torch.float64, device=DEV)
        self._lib = _lib.load()
        self._lu = None
        self._leaf = leaf
        self._grid = (p1.gi, p1.gj)
        self._handle_cls = _LUHandle
        self.assemble()

    def assemble(self):
        """Every slab's F_k values on the device (stmhd_c5_values)."""
        from . import _lib

        self._sell = None  # the sliced-ELL copy follows the values
        d = self._d
        _lib.check(self._lib.stmhd_c5_values(_lib.stream_ptr(), self.nnz, self.nt, _lib.ptr(d["base"]),
                                             _lib.ptr(d["cptr"]), _lib.ptr(d["cinfo"]), _lib.ptr(d["elem"]),
                                             _lib.ptr(self.u), self.n, _lib.ptr(self._mloc), _lib.ptr(self._grad),
                                             _lib.ptr(self.values)))

    def matrix(self, k: int):
        """F_k as scipy CSR (tests / inspection)."""
        import scipy.sparse as sp

        v = self.values[k * self.nnz:(k + 1) * self.nnz].cpu().numpy()
        return sp.csr_matrix((v, self.col, self.rowptr), shape=(self.n, self.n))

    def apply(self, x, out=None):
        """y_k = F_k x_k - C x_{k-1} (oracle C5.apply)."""
        import torch

        from . import _lib
        from .linalg import as_device

        x = as_device(x).reshape(-1).contiguous()
        out = torch.empty_like(x) if out is None else out
        _lib.check(self._lib.stmhd_spmv_apply(self._spmv_plan(), _lib.stream_ptr(), self.nt, _lib.ptr(self._sell),
                                              1.0, -1.0, _lib.ptr(x), _lib.ptr(out)))
        return out

    def _spmv_plan(self):
        """Row-block plan of the slab-looped SpMV (stmhd_spmv_create), built once."""
        import ctypes

        from . import _lib

        if getattr(self, "_plan", None) is None:
            h = ctypes.c_void_p()
            rp = np.ascontiguousarray(self.rowptr, dtype=np.int32)
            cl = np.ascontiguousarray(self.col, dtype=np.int32)
            crp = np.ascontiguousarray(self.coupling.indptr, dtype=np.int32)
            ccl = np.ascontiguousarray(self.coupling.indices, dtype=np.int32)
            cvl = np.ascontiguousarray(self.coupling.data, dtype=np.float64)
            _lib.check(self._lib.stmhd_spmv_create(self.n, rp.ctypes.data, cl.ctypes.data, crp.ctypes.data,
                                                   ccl.ctypes.data, cvl.ctypes.data, -self.n, _lib.stream_ptr(),
                                                   ctypes.byref(h)))
            self._plan = h.value
            self._sell = None
        if self._sell is None:
            import torch

            n = self._lib.stmhd_spmv_sell_size(self._plan)
            self._sell = torch.empty(self.nt * n, dtype=torch.float64, device=self.values.device)
            _lib.check(self._lib.stmhd_spmv_relayout(self._plan, _lib.stream_ptr(), self.nt, _lib.ptr(self.values),
                                                     self.nnz, _lib.ptr(self._sell)))
        return self._plan

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan is not None:
            try:
                self._lib.stmhd_spmv_destroy(plan)
            except Exception:
                pass

    def factor(self):
        """One nested-dissection LU per slab (batched, shared symbolic structure)."""
        import scipy.sparse as sp

        if self._lu is None:
            pat = sp.csr_matrix((np.ones(self.nnz), self.col, self.rowptr), shape=(self.n, self.n))
            self._lu = self._handle_cls(pat, self.nt, self._grid[0], self._grid[1], self._leaf)
        self._lu.factor(self.values, self.nnz)

    def solve(self, r, out=None):
        """x_k = F_k^{-1}(r_k + C x_{k-1}) sequentially (oracle C5.solve)."""
        import torch

        from . import _lib
        from .linalg import as_device

        if self._lu is None:
            self.factor()
        r = as_device(r).reshape(-1).contiguous()
        out = torch.empty_like(r) if out is None else out
        d = self._d
        _lib.check(self._lib.stmhd_lu_sweep(self._lu.h, _lib.stream_ptr(), _lib.ptr(r), self.n, _lib.ptr(out),
                                            self.n, self.nt, _lib.ptr(d["c_rowptr"]), _lib.ptr(d["c_col"]),
                                            _lib.ptr(d["c_val"]), 1.0))
        return out
