"""Structured triangle mesh, Pk Lagrange spaces and Galerkin assembly
(TEST INFRASTRUCTURE ONLY -- CPU restatement of reference ``mesh.py`` and
``fem.py``; see the citations on each function).

Everything is evaluated with the reference's 25-point collapsed Gauss rule so
the oracle reproduces the reference's rounding closely; sparse matrices are
built with scipy COO->CSR exactly like the reference (duplicates summed,
explicit zeros kept until a product or sum drops them).
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import scipy.sparse as sp
from numpy.polynomial.legendre import leggauss

SIDES = ("left", "right", "bottom", "top")
NORMAL_COMP = {"left": 0, "right": 0, "bottom": 1, "top": 1}  # fem.py:505


class Mesh:
    """[x0,x1]x[y0,y1] split into nx*ny squares, two CCW triangles each:
    (v00,v10,v11) and (v00,v11,v01); vertex (i,j) -> j*(nx+1)+i
    (reference mesh.py:96-132)."""

    def __init__(self, x0, x1, y0, y1, nx, ny):
        self.x0, self.x1, self.y0, self.y1 = x0, x1, y0, y1
        self.nx, self.ny = nx, ny
        xs = np.linspace(x0, x1, nx + 1)
        ys = np.linspace(y0, y1, ny + 1)
        gx, gy = np.meshgrid(xs, ys, indexing="xy")
        self.verts = np.column_stack([gx.ravel(), gy.ravel()])
        i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
        i, j = i.ravel(), j.ravel()
        v00 = j * (nx + 1) + i
        v10, v01, v11 = v00 + 1, v00 + nx + 1, v00 + nx + 2
        tri = np.empty((2 * nx * ny, 3), dtype=np.int64)
        tri[0::2] = np.column_stack([v00, v10, v11])
        tri[1::2] = np.column_stack([v00, v11, v01])
        self.tris = tri

    @property
    def hx(self):
        return (self.x1 - self.x0) / self.nx

    @property
    def hy(self):
        return (self.y1 - self.y0) / self.ny

    @property
    def area(self):
        return (self.x1 - self.x0) * (self.y1 - self.y0)

    @property
    def ne(self):
        return len(self.tris)


def rect_mesh(x0, x1, y0, y1, dx) -> Mesh:
    nx = int(round((x1 - x0) / dx))
    ny = int(round((y1 - y0) / dx))
    return Mesh(x0, x1, y0, y1, nx, ny)


def duffy_rule(n):
    """Collapsed Gauss rule on the unit triangle (reference fem.py:36-45)."""
    t, w = leggauss(n)
    t = 0.5 * (t + 1.0)
    w = 0.5 * w
    a, b = np.meshgrid(t, t, indexing="ij")
    wa, wb = np.meshgrid(w, w, indexing="ij")
    pts = np.column_stack([a.ravel(), (b * (1.0 - a)).ravel()])
    return pts, (wa * wb * (1.0 - a)).ravel()


def lattice(k):
    """(a,b,c) barycentric index triples, c outer (reference fem.py:48-50)."""
    return [(k - b - c, b, c) for c in range(k + 1) for b in range(k + 1 - c)]


def _mono_exps(k):
    return [(p, q) for q in range(k + 1) for p in range(k + 1 - q)]


def _mono_eval(exps, pts):
    x, y = pts[:, 0], pts[:, 1]
    v = np.column_stack([x**p * y**q for p, q in exps])
    dx = np.column_stack([p * x ** max(p - 1, 0) * y**q if p else 0.0 * x for p, q in exps])
    dy = np.column_stack([q * x**p * y ** max(q - 1, 0) if q else 0.0 * x for p, q in exps])
    return v, dx, dy


@lru_cache(maxsize=None)
def _coeffs(k):
    nodes = np.array([(b / k, c / k) for (_, b, c) in lattice(k)])
    v, _, _ = _mono_eval(_mono_exps(k), nodes)
    return np.linalg.inv(v)


def ref_basis(k, pts):
    """Values (nloc,nq) and reference gradients (nloc,nq,2) of the Lagrange
    basis through the monomial Vandermonde inverse (reference fem.py:53-81)."""
    c = _coeffs(k)
    v, dx, dy = _mono_eval(_mono_exps(k), pts)
    return (v @ c).T, np.stack([(dx @ c).T, (dy @ c).T], axis=-1)


class Space:
    """Scalar or 2-vector Pk space on the refined (k nx+1)x(k ny+1) node grid
    (reference fem.py:84-189)."""

    def __init__(self, mesh: Mesh, k: int, ncomp: int = 1):
        self.mesh, self.k, self.ncomp = mesh, k, ncomp
        self.gnx, self.gny = k * mesh.nx, k * mesh.ny
        self.n_nodes = (self.gnx + 1) * (self.gny + 1)
        self.ndof = ncomp * self.n_nodes
        gi = np.arange(self.n_nodes) % (self.gnx + 1)
        gj = np.arange(self.n_nodes) // (self.gnx + 1)
        self.coords = np.column_stack([mesh.x0 + gi * mesh.hx / k, mesh.y0 + gj * mesh.hy / k])
        self.side_nodes = {
            "left": np.flatnonzero(gi == 0), "right": np.flatnonzero(gi == self.gnx),
            "bottom": np.flatnonzero(gj == 0), "top": np.flatnonzero(gj == self.gny),
        }
        vi = np.arange(len(mesh.verts)) % (mesh.nx + 1)
        vj = np.arange(len(mesh.verts)) // (mesh.nx + 1)
        lat = np.array(lattice(k))
        gx = (k * vi[mesh.tris]) @ lat.T // k
        gy = (k * vj[mesh.tris]) @ lat.T // k
        self.elem = gy * (self.gnx + 1) + gx
        p = mesh.verts[mesh.tris]
        e1, e2 = p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]
        self.det = e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]
        inv = np.empty((mesh.ne, 2, 2))
        inv[:, 0, 0], inv[:, 0, 1] = e2[:, 1], -e2[:, 0]
        inv[:, 1, 0], inv[:, 1, 1] = -e1[:, 1], e1[:, 0]
        self.invj = inv / self.det[:, None, None]
        self.jmat = np.stack([e1, e2], axis=-1)
        self.origin = p[:, 0]
        pts, self.w = duffy_rule(5)
        self.tab, g = ref_basis(k, pts)
        self.grads = np.einsum("iqr,erd->eiqd", g, self.invj)

    def comp(self, v, c):
        return v[c * self.n_nodes:(c + 1) * self.n_nodes]

    def scalar_at_q(self, coef):
        ce = coef[self.elem]
        return ce @ self.tab, np.einsum("ei,eiqd->eqd", ce, self.grads)

    def vector_at_q(self, coef):
        vals = np.empty((self.mesh.ne, len(self.w), 2))
        grads = np.empty((self.mesh.ne, len(self.w), 2, 2))
        for d in range(2):
            vals[:, :, d], grads[:, :, d, :] = self.scalar_at_q(self.comp(coef, d))
        return vals, grads

    def interp(self, fn):
        x, y = self.coords[:, 0], self.coords[:, 1]
        return np.asarray(fn(x, y), dtype=float) + np.zeros(self.n_nodes)


def _coo(rows, cols, vals, shape):
    return sp.coo_matrix((np.ravel(vals), (np.ravel(rows), np.ravel(cols))), shape=shape).tocsr()


def _pairs(sr: Space, sc: Space, roff=0, coff=0):
    er, ec = sr.elem + roff, sc.elem + coff
    return (np.repeat(er[:, :, None], ec.shape[1], axis=2),
            np.repeat(ec[:, None, :], er.shape[1], axis=1))


def _blockdiag2(m):
    return sp.block_diag((m, m), format="csr")


# -- constant operators (reference fem.py:211-335) ------------------------------

def mass(s: Space):
    loc = np.einsum("iq,jq,q->ij", s.tab, s.tab, s.w)
    r, c = _pairs(s, s)
    m = _coo(r, c, np.broadcast_to(loc[None] * s.det[:, None, None], r.shape),
             (s.n_nodes, s.n_nodes))
    return m if s.ncomp == 1 else _blockdiag2(m)


def stiffness(s: Space):
    loc = np.einsum("eiqd,ejqd,q->eij", s.grads, s.grads, s.w) * s.det[:, None, None]
    r, c = _pairs(s, s)
    m = _coo(r, c, loc, (s.n_nodes, s.n_nodes))
    return m if s.ncomp == 1 else _blockdiag2(m)


def neg_divergence(vel: Space, prs: Space):
    rs, cs, vs = [], [], []
    for c in range(2):
        loc = -np.einsum("mq,enq,q->emn", prs.tab, vel.grads[:, :, :, c], vel.w) * vel.det[:, None, None]
        r, cc = _pairs(prs, vel, coff=c * vel.n_nodes)
        rs.append(r.ravel()), cs.append(cc.ravel()), vs.append(loc.ravel())
    return _coo(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), (prs.ndof, vel.ndof))


def mixed_grad(sr: Space, sc: Space):
    loc = np.einsum("eiqd,ejqd,q->eij", sr.grads, sc.grads, sr.w) * sr.det[:, None, None]
    r, c = _pairs(sr, sc)
    return _coo(r, c, loc, (sr.ndof, sc.ndof))


def load(s: Space, fn):
    """High-order (10x10 collapsed Gauss) load vector, reference fem.py:274-284."""
    pts, w = duffy_rule(10)
    tab, _ = ref_basis(s.k, pts)
    xq = np.einsum("eds,qs->eqd", s.jmat, pts) + s.origin[:, None, :]
    fv = np.asarray(fn(xq[:, :, 0], xq[:, :, 1]), dtype=float) + np.zeros(xq.shape[:2])
    out = np.zeros(s.ndof)
    np.add.at(out, s.elem, np.einsum("eq,iq,q->ei", fv, tab, w) * s.det[:, None])
    return out


def edge_load(s: Space, side: str, fn):
    """Boundary load on one side, 1D Gauss with k+2 points per segment
    (reference fem.py:287-318)."""
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
    for c in range(m.nx if horiz else m.ny):
        seg = ordered[c * k:c * k + k + 1]
        x = s.coords[seg[0], 0] + (t * length if horiz else 0.0)
        y = s.coords[seg[0], 1] + (0.0 if horiz else t * length)
        fv = np.asarray(fn(x, y), dtype=float) + np.zeros(len(t))
        out[seg] += length * (tab.T @ (w * fv))
    return out


def integral(s: Space, coef):
    v, _ = s.scalar_at_q(coef)
    return float(np.einsum("eq,q,e->", v, s.w, s.det))


def mean_grad(s: Space, coef):
    """reference fem.py:331-335."""
    _, g = s.scalar_at_q(coef)
    return np.einsum("eqd,q,e->d", g, s.w, s.det) / s.mesh.area


# -- state-dependent blocks (reference fem.py:341-472) --------------------------

def momentum_advection(vel: Space, u):
    """(residual, transport, reaction) of (u.grad)u, reference fem.py:341-381."""
    uv, ug = vel.vector_at_q(u)
    det, w, nn = vel.det, vel.w, vel.n_nodes
    conv = np.einsum("eqc,eqdc->eqd", uv, ug)
    loc = np.einsum("eqd,iq,q->eid", conv, vel.tab, w) * det[:, None, None]
    res = np.zeros(vel.ndof)
    for d in range(2):
        np.add.at(res, vel.elem + d * nn, loc[:, :, d])
    ug_dot = np.einsum("eqc,ejqc->ejq", uv, vel.grads)
    tv = np.einsum("iq,ejq,q->eij", vel.tab, ug_dot, w) * det[:, None, None]
    r, c = _pairs(vel, vel)
    transport = _coo(np.concatenate([r.ravel(), (r + nn).ravel()]),
                     np.concatenate([c.ravel(), (c + nn).ravel()]),
                     np.concatenate([tv.ravel(), tv.ravel()]), (vel.ndof, vel.ndof))
    rv = np.einsum("iq,jq,eqdc,q->eijdc", vel.tab, vel.tab, ug, w) * det[:, None, None, None, None]
    rs, cs, vs = [], [], []
    for d in range(2):
        for cd in range(2):
            rs.append((r + d * nn).ravel()), cs.append((c + cd * nn).ravel())
            vs.append(rv[:, :, :, d, cd].ravel())
    reaction = _coo(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), (vel.ndof, vel.ndof))
    return res, transport, reaction


def lorentz(vel: Space, cur: Space, pot: Space, j, a):
    """(residual, Z_j(A), Z_A(j)), reference fem.py:391-427."""
    jv, _ = cur.scalar_at_q(j)
    _, ag = pot.scalar_at_q(a)
    det, w, nn = vel.det, vel.w, vel.n_nodes
    loc = np.einsum("eq,eqd,iq,q->eid", jv, ag, vel.tab, w) * det[:, None, None]
    res = np.zeros(vel.ndof)
    for d in range(2):
        np.add.at(res, vel.elem + d * nn, loc[:, :, d])
    zj = np.einsum("nq,eqd,iq,q->eind", cur.tab, ag, vel.tab, w) * det[:, None, None, None]
    za = np.einsum("eq,enqd,iq,q->eind", jv, pot.grads, vel.tab, w) * det[:, None, None, None]

    def build(vals, col):
        rs, cs, vs = [], [], []
        for d in range(2):
            r, c = _pairs(vel, col, roff=d * nn)
            rs.append(r.ravel()), cs.append(c.ravel()), vs.append(vals[:, :, :, d].ravel())
        return _coo(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), (vel.ndof, col.ndof))

    return res, build(zj, cur), build(za, pot)


def potential_advection(pot: Space, vel: Space, u, a):
    """(residual, lin_a, lin_u) of u.grad A, reference fem.py:430-462."""
    uv, _ = vel.vector_at_q(u)
    _, ag = pot.scalar_at_q(a)
    det, w = pot.det, pot.w
    conv = np.einsum("eqc,eqc->eq", uv, ag)
    res = np.zeros(pot.ndof)
    np.add.at(res, pot.elem, np.einsum("eq,mq,q->em", conv, pot.tab, w) * det[:, None])
    ugd = np.einsum("eqc,enqc->enq", uv, pot.grads)
    fa = np.einsum("mq,enq,q->emn", pot.tab, ugd, w) * det[:, None, None]
    r, c = _pairs(pot, pot)
    lin_a = _coo(r, c, fa, (pot.ndof, pot.ndof))
    yv = np.einsum("mq,nq,eqc,q->emnc", pot.tab, vel.tab, ag, w) * det[:, None, None, None]
    rs, cs, vs = [], [], []
    for cd in range(2):
        r, c = _pairs(pot, vel, coff=cd * vel.n_nodes)
        rs.append(r.ravel()), cs.append(c.ravel()), vs.append(yv[:, :, :, cd].ravel())
    lin_u = _coo(np.concatenate(rs), np.concatenate(cs), np.concatenate(vs), (pot.ndof, vel.ndof))
    return res, lin_a, lin_u


def pcd_advection(prs: Space, vel: Space, u):
    """reference fem.py:465-472."""
    uv, _ = vel.vector_at_q(u)
    ugd = np.einsum("eqc,enqc->enq", uv, prs.grads)
    vals = np.einsum("mq,enq,q->emn", prs.tab, ugd, prs.w) * prs.det[:, None, None]
    r, c = _pairs(prs, prs)
    return _coo(r, c, vals, (prs.ndof, prs.ndof))


# -- boundary conditions (reference fem.py:529-610) -----------------------------

def _keep(n, idx):
    d = np.ones(n)
    d[idx] = 0.0
    return sp.diags(d).tocsr()


def bc_identity(m, idx):
    n = m.shape[0]
    if len(idx) == 0:
        return m.tocsr()
    z = _keep(n, idx)
    one = sp.coo_matrix((np.ones(len(idx)), (idx, idx)), shape=(n, n)).tocsr()
    return (z @ m @ z + one).tocsr()


def bc_zero(m, rows=None, cols=None):
    out = m
    if rows is not None and len(rows):
        out = _keep(out.shape[0], np.asarray(rows)) @ out
    if cols is not None and len(cols):
        out = out @ _keep(out.shape[1], np.asarray(cols))
    return out.tocsr()


def slip_dofs(vel: Space):
    """Normal-component DOFs of every side (slip everywhere)."""
    idx = np.concatenate([vel.side_nodes[s] + NORMAL_COMP[s] * vel.n_nodes for s in SIDES])
    return np.unique(idx)


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
