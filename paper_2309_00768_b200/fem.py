"""Host-side finite-element setup for the device kernels (one-time, CPU).

Everything here is state-independent and runs once per discretisation:
mesh and DOF maps (reference ``mesh.py:96-132``, ``fem.py:84-189``), exact
per-orientation element tensors, constant operators, loads and boundary
index sets (``fem.py:211-335``, ``fem.py:529-610``).

Unlike the reference, which re-integrates every state-dependent form with a
25-point rule inside each Newton step, the device kernels contract the state
against *exact* reference-element tensors.  On the structured mesh there are
only two element orientations, so every tensor exists
twice:

  MV[i,j]          = det int phi_i phi_j                    (velocity mass)
  KV[o,i,j]        = det int grad phi_i . grad phi_j        (velocity stiffness)
  TV[o,i,m,j,c]    = det int phi_i phi_m d_c phi_j          (transport/reaction)
  MX[i,n]          = det int phi_i psi_n                    (velocity x P1)
  G1[o,n,c]        = d_c psi_n                              (P1 gradients)
  M1, K1[o]        P1 mass / stiffness
  MP, KP[o]        pressure mass / stiffness
  TP[o,m,l,n,c]    = det int q_m phi_l d_c q_n              (PCD advection)
  BD[o,m,n,c]      = -det int q_m d_c phi_n                 (negative divergence)

Polynomials are integrated exactly with int_T x^p y^q = p! q! / (p+q+2)!.
"""

from __future__ import annotations

from functools import lru_cache
from math import factorial

import numpy as np
import scipy.sparse as sp
from numpy.polynomial.legendre import leggauss

SIDES = ("left", "right", "bottom", "top")
NORMAL_COMP = {"left": 0, "right": 0, "bottom": 1, "top": 1}


# -- mesh and spaces -----------------------------------------------------------

class Mesh:
    """Uniform right-triangle mesh; cell (i,j) -> elements 2(j nx+i) =
    (v00,v10,v11) [orientation 0] and 2(j nx+i)+1 = (v00,v11,v01)
    [orientation 1] (reference mesh.py:112-121)."""

    def __init__(self, x0, x1, y0, y1, nx, ny):
        self.x0, self.x1, self.y0, self.y1, self.nx, self.ny = x0, x1, y0, y1, nx, ny
        self.hx, self.hy = (x1 - x0) / nx, (y1 - y0) / ny
        self.area = (x1 - x0) * (y1 - y0)
        cj, ci = np.divmod(np.arange(nx * ny), nx)
        v00 = cj * (nx + 1) + ci
        tri = np.empty((2 * nx * ny, 3), dtype=np.int64)
        tri[0::2] = np.column_stack([v00, v00 + 1, v00 + nx + 2])
        tri[1::2] = np.column_stack([v00, v00 + nx + 2, v00 + nx + 1])
        self.tris = tri
        self.ne = len(tri)
        self.vi = np.arange((nx + 1) * (ny + 1)) % (nx + 1)
        self.vj = np.arange((nx + 1) * (ny + 1)) // (nx + 1)


def lattice(k):
    """Barycentric node triples, c outer (reference fem.py:48-50)."""
    return [(k - b - c, b, c) for c in range(k + 1) for b in range(k + 1 - c)]


class Space:
    """Pk Lagrange space on the refined grid: node (gi,gj) -> gj*(k nx+1)+gi,
    vector DOF = comp*n_nodes + node (reference fem.py:9-11, 97-123)."""

    def __init__(self, mesh: Mesh, k: int, ncomp: int = 1):
        self.mesh, self.k, self.ncomp = mesh, k, ncomp
        self.gnx, self.gny = k * mesh.nx, k * mesh.ny
        self.n_nodes = (self.gnx + 1) * (self.gny + 1)
        self.ndof = ncomp * self.n_nodes
        self.gi = np.arange(self.n_nodes) % (self.gnx + 1)
        self.gj = np.arange(self.n_nodes) // (self.gnx + 1)
        self.coords = np.column_stack([mesh.x0 + self.gi * mesh.hx / k,
                                       mesh.y0 + self.gj * mesh.hy / k])
        lat = np.array(lattice(k))
        gx = (k * mesh.vi[mesh.tris]) @ lat.T // k
        gy = (k * mesh.vj[mesh.tris]) @ lat.T // k
        self.elem = (gy * (self.gnx + 1) + gx).astype(np.int64)
        self.nloc = self.elem.shape[1]
        self.side_nodes = {
            "left": np.flatnonzero(self.gi == 0), "right": np.flatnonzero(self.gi == self.gnx),
            "bottom": np.flatnonzero(self.gj == 0), "top": np.flatnonzero(self.gj == self.gny),
        }

    def interp(self, fn):
        return np.asarray(fn(self.coords[:, 0], self.coords[:, 1]), dtype=float) + np.zeros(self.n_nodes)

    def node_elements(self):
        """CSR (ptr, code) of the elements touching each node, code =
        e*16 + local index, sorted by element."""
        ne, nl = self.elem.shape
        node = self.elem.ravel()
        code = (np.repeat(np.arange(ne), nl) * 16 + np.tile(np.arange(nl), ne))
        order = np.lexsort((code, node))
        ptr = np.zeros(self.n_nodes + 1, dtype=np.int64)
        np.add.at(ptr, node + 1, 1)
        return np.cumsum(ptr).astype(np.int32), code[order].astype(np.int32)


# -- exact polynomial algebra on the reference triangle ------------------------

def _mono_exps(k):
    return [(p, q) for q in range(k + 1) for p in range(k + 1 - q)]


@lru_cache(maxsize=None)
def basis_polys(k):
    """Monomial coefficient arrays C[i][p,q] of the k-th degree Lagrange basis
    (monomial Vandermonde inverse, reference fem.py:53-81)."""
    nodes = [(b / k, c / k) for (_, b, c) in lattice(k)]
    exps = _mono_exps(k)
    vand = np.array([[x**p * y**q for (p, q) in exps] for (x, y) in nodes])
    coef = np.linalg.inv(vand)  # column i = coefficients of basis i
    polys = []
    for i in range(len(nodes)):
        c = np.zeros((k + 1, k + 1))
        for t, (p, q) in enumerate(exps):
            c[p, q] = coef[t, i]
        polys.append(c)
    return polys


def _dx(c):
    out = np.zeros_like(c)
    out[:-1, :] = c[1:, :] * np.arange(1, c.shape[0])[:, None]
    return out


def _dy(c):
    out = np.zeros_like(c)
    out[:, :-1] = c[:, 1:] * np.arange(1, c.shape[1])[None, :]
    return out


def _mul(*cs):
    out = np.ones((1, 1))
    for c in cs:
        r = np.zeros((out.shape[0] + c.shape[0] - 1, out.shape[1] + c.shape[1] - 1))
        for p in range(c.shape[0]):
            for q in range(c.shape[1]):
                if c[p, q] != 0.0:
                    r[p:p + out.shape[0], q:q + out.shape[1]] += c[p, q] * out
        out = r
    return out


@lru_cache(maxsize=None)
def _mono_int(pmax):
    t = np.zeros((pmax + 1, pmax + 1))
    for p in range(pmax + 1):
        for q in range(pmax + 1):
            t[p, q] = factorial(p) * factorial(q) / factorial(p + q + 2)
    return t


def _int(c):
    t = _mono_int(max(c.shape))
    return float(np.sum(c * t[: c.shape[0], : c.shape[1]]))


def orientation_maps(hx, hy):
    """(det, invJ[o]) of the two element orientations (reference fem.py:126-135)."""
    e = [((hx, 0.0), (hx, hy)), ((hx, hy), (0.0, hy))]
    inv = []
    for e1, e2 in e:
        det = e1[0] * e2[1] - e1[1] * e2[0]
        inv.append(np.array([[e2[1], -e2[0]], [-e1[1], e1[0]]]) / det)
    return hx * hy, inv


def _phys_grads(polys, invj):
    """Physical gradient polynomials g[i][c] = sum_r d_r phi_i invJ[r,c]."""
    out = []
    for c0 in polys:
        d = (_dx(c0), _dy(c0))
        out.append([d[0] * invj[0, c] + d[1] * invj[1, c] for c in range(2)])
    return out


def element_tensors(kv: int, kp: int, hx: float, hy: float) -> dict:
    """All element tensors the assembly kernels contract against."""
    det, invs = orientation_maps(hx, hy)
    pv, pp, p1 = basis_polys(kv), basis_polys(kp), basis_polys(1)
    nv, npl = len(pv), len(pp)
    T = {}
    T["MV"] = np.array([[det * _int(_mul(a, b)) for b in pv] for a in pv])
    T["M1"] = np.array([[det * _int(_mul(a, b)) for b in p1] for a in p1])
    T["MP"] = np.array([[det * _int(_mul(a, b)) for b in pp] for a in pp])
    T["MX"] = np.array([[det * _int(_mul(a, b)) for b in p1] for a in pv])
    KV, K1, KP, TV, TP, BD, G1 = [], [], [], [], [], [], []
    for inv in invs:
        gv, g1, gp = _phys_grads(pv, inv), _phys_grads(p1, inv), _phys_grads(pp, inv)
        KV.append([[det * sum(_int(_mul(gv[i][c], gv[j][c])) for c in range(2))
                    for j in range(nv)] for i in range(nv)])
        K1.append([[det * sum(_int(_mul(g1[i][c], g1[j][c])) for c in range(2))
                    for j in range(3)] for i in range(3)])
        KP.append([[det * sum(_int(_mul(gp[i][c], gp[j][c])) for c in range(2))
                    for j in range(npl)] for i in range(npl)])
        tv = np.zeros((nv, nv, nv, 2))
        for i in range(nv):
            for m in range(i, nv):
                pm = _mul(pv[i], pv[m])
                for j in range(nv):
                    for c in range(2):
                        tv[i, m, j, c] = tv[m, i, j, c] = det * _int(_mul(pm, gv[j][c]))
        TV.append(tv)
        tp = np.zeros((npl, nv, npl, 2))
        for m in range(npl):
            for l in range(nv):
                pm = _mul(pp[m], pv[l])
                for n in range(npl):
                    for c in range(2):
                        tp[m, l, n, c] = det * _int(_mul(pm, gp[n][c]))
        TP.append(tp)
        BD.append([[[-det * _int(_mul(pp[m], gv[n][c])) for c in range(2)] for n in range(nv)]
                   for m in range(npl)])
        G1.append([[float(g1[n][c][0, 0]) for c in range(2)] for n in range(3)])
    T["KV"], T["K1"], T["KP"] = np.array(KV), np.array(K1), np.array(KP)
    T["TV"], T["TP"], T["BD"], T["G1"] = np.array(TV), np.array(TP), np.array(BD), np.array(G1)
    T["det"] = det
    return T


# -- constant operators (state independent; values assembled on the device) ----------

def _assemble(sr: Space, sc: Space, local_by_o, roff=0, coff=0, shape=None):
    """CSR of a per-orientation local matrix (no, nr, nc) summed over the elements:
    reference assemble_mass / assemble_stiffness / assemble_divergence (fem.py:211-271).
    The pattern and the values come from the device kernels of csrc/constops.cu
    (C-ABI stmhd_const_assemble); there is no host fallback."""
    from . import _lib

    lib = _lib.load()
    loc = np.ascontiguousarray(np.asarray(local_by_o, dtype=np.float64))
    nr, nc = sr.elem.shape[1], sc.elem.shape[1]
    assert loc.shape == (2, nr, nc)
    ne = sr.mesh.ne
    ptr, code = sr.node_elements()
    elem_c = np.ascontiguousarray(sc.elem, dtype=np.int32)
    cap = int(ne) * nr * nc
    rowptr = np.empty(sr.n_nodes + 1, np.int32)
    col = np.empty(cap, np.int32)
    val = np.empty(cap, np.float64)
    nnz = np.zeros(1, np.int64)
    _lib.check(lib.stmhd_const_assemble(_lib.stream_ptr(), sr.n_nodes, nr, nc, ne, _lib.ptr(ptr), _lib.ptr(code),
                                        _lib.ptr(elem_c), _lib.ptr(loc), _lib.ptr(rowptr), _lib.ptr(col),
                                        _lib.ptr(val), cap, _lib.ptr(nnz)))
    n = int(nnz[0])
    shape = shape or (sr.n_nodes, sc.n_nodes)
    rp = rowptr
    if roff or shape[0] != sr.n_nodes:
        rp = np.concatenate([np.zeros(roff, np.int32), rowptr, np.full(shape[0] - roff - sr.n_nodes, n, np.int32)])
    return sp.csr_matrix((val[:n].copy(), col[:n] + np.int32(coff), rp), shape=shape)


def blockdiag2(m):
    return sp.block_diag((m, m), format="csr")


def constant_operators(vel: Space, prs: Space, p1: Space, T: dict) -> dict:
    ops = {}
    ops["mass_u"] = blockdiag2(_assemble(vel, vel, [T["MV"], T["MV"]]))
    ops["stiff_u"] = blockdiag2(_assemble(vel, vel, T["KV"]))
    ops["mass_p"] = _assemble(prs, prs, [T["MP"], T["MP"]])
    ops["stiff_p"] = _assemble(prs, prs, T["KP"])
    ops["mass_1"] = _assemble(p1, p1, [T["M1"], T["M1"]])
    ops["stiff_1"] = _assemble(p1, p1, T["K1"])
    blocks = [_assemble(prs, vel, T["BD"][:, :, :, c], coff=c * vel.n_nodes,
                        shape=(prs.ndof, vel.ndof)) for c in range(2)]
    ops["div"] = (blocks[0] + blocks[1]).tocsr()
    return ops


# -- loads (high-order rules; non-polynomial data) -----------------------------------

def duffy_rule(n):
    t, w = leggauss(n)
    t, w = 0.5 * (t + 1.0), 0.5 * w
    a, b = np.meshgrid(t, t, indexing="ij")
    wa, wb = np.meshgrid(w, w, indexing="ij")
    return np.column_stack([a.ravel(), (b * (1.0 - a)).ravel()]), (wa * wb * (1.0 - a)).ravel()


def _eval_poly(c, x, y):
    out = np.zeros_like(x)
    for p in range(c.shape[0]):
        for q in range(c.shape[1]):
            if c[p, q] != 0.0:
                out = out + c[p, q] * x**p * y**q
    return out


def load_vector(s: Space, fn, nq=10):
    """int fn * basis with the 100-point collapsed rule (as reference
    fem.py:274-284), evaluated on both orientations."""
    pts, w = duffy_rule(nq)
    tab = np.array([_eval_poly(c, pts[:, 0], pts[:, 1]) for c in basis_polys(s.k)])
    m = s.mesh
    verts = np.column_stack([m.x0 + m.vi * m.hx, m.y0 + m.vj * m.hy])
    p = verts[m.tris]
    e1, e2 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]
    det = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
    xq = p[:, 0, None, 0] + e1[:, None, 0] * pts[None, :, 0] + e2[:, None, 0] * pts[None, :, 1]
    yq = p[:, 0, None, 1] + e1[:, None, 1] * pts[None, :, 0] + e2[:, None, 1] * pts[None, :, 1]
    fv = np.asarray(fn(xq, yq), dtype=float) + np.zeros(xq.shape)
    loc = np.einsum("eq,iq,q->ei", fv, tab, w) * det[:, None]
    out = np.zeros(s.ndof)
    np.add.at(out, s.elem, loc)
    return out


def edge_load_vector(s: Space, side: str, fn):
    """int_side fn * basis ds with k+2 Gauss points per segment (reference
    fem.py:287-318)."""
    k = s.k
    t, w = leggauss(k + 2)
    t, w = 0.5 * (t + 1.0), 0.5 * w
    coef = np.linalg.inv(np.vander(np.arange(k + 1) / k, k + 1, increasing=True))
    tab = np.vander(t, k + 1, increasing=True) @ coef
    horiz = side in ("bottom", "top")
    m = s.mesh
    length = m.hx if horiz else m.hy
    nodes = s.side_nodes[side]
    ordered = nodes[np.argsort(s.coords[nodes, 0 if horiz else 1])]
    out = np.zeros(s.ndof)
    for cell in range(m.nx if horiz else m.ny):
        seg = ordered[cell * k: cell * k + k + 1]
        x = s.coords[seg[0], 0] + (t * length if horiz else 0.0)
        y = s.coords[seg[0], 1] + (0.0 if horiz else t * length)
        fv = np.asarray(fn(x, y), dtype=float) + np.zeros(len(t))
        out[seg] += length * (tab.T @ (w * fv))
    return out


def mean_integral(s: Space, coef, T_mass_local):
    """Exact integral of a scalar FE field: sum_e sum_ij M_loc[i,j] c_j /
    sum over basis (int phi_i = row sums of the local mass)."""
    w = T_mass_local.sum(axis=1)
    return float(np.sum(coef[s.elem] @ w))


# -- boundary conditions (reference fem.py:529-610) ------------------------------------

def slip_dofs(vel: Space):
    return np.unique(np.concatenate([vel.side_nodes[s] + NORMAL_COMP[s] * vel.n_nodes
                                     for s in SIDES]))


def dirichlet_dofs(s: Space, sides, fn):
    parts, vals = [], []
    for side in SIDES:
        if side in sides:
            nodes = s.side_nodes[side]
            parts.append(nodes)
            vals.append(np.asarray(fn(s.coords[nodes, 0], s.coords[nodes, 1]), dtype=float)
                        + np.zeros(len(nodes)))
    if not parts:
        return np.empty(0, dtype=np.int64), np.empty(0)
    idx, first = np.unique(np.concatenate(parts), return_index=True)
    return idx, np.concatenate(vals)[first]


def keep_mask(n, idx):
    d = np.ones(n)
    d[idx] = 0.0
    return sp.diags(d).tocsr()


def bc_identity(m, idx):
    n = m.shape[0]
    if len(idx) == 0:
        return m.tocsr()
    z = keep_mask(n, idx)
    return (z @ m @ z + sp.coo_matrix((np.ones(len(idx)), (idx, idx)), shape=(n, n))).tocsr()


def bc_zero(m, rows=None, cols=None):
    out = m
    if rows is not None and len(rows):
        out = keep_mask(out.shape[0], np.asarray(rows)) @ out
    if cols is not None and len(cols):
        out = out @ keep_mask(out.shape[1], np.asarray(cols))
    return out.tocsr()
