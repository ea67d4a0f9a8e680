"""Discretisation, space-time residual, Jacobian blocks and matvec
(TEST INFRASTRUCTURE ONLY -- CPU restatement of reference ``problems.py``
``Discretization``/``initial_state`` and ``spacetime.py``)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fe
from .configs import ProblemSpec


class SingularMatrix(Exception):
    pass


class LU:
    """SuperLU factor with the reference's non-finite check (linalg.py:71-86)."""

    def __init__(self, m):
        try:
            self._lu = spla.splu(sp.csc_matrix(m))
        except RuntimeError as exc:
            raise SingularMatrix(str(exc)) from exc
        self.shape = m.shape

    def solve(self, b):
        x = self._lu.solve(np.asarray(b, dtype=float))
        if not np.all(np.isfinite(x)):
            raise SingularMatrix("non-finite LU solve")
        return x


class Disc:
    """All state-independent data of one space-time grid (reference
    problems.py:141-256), with the adapter's velocity degree."""

    def __init__(self, prob: ProblemSpec, nx: int, ny: int, dt: float, nt: int):
        self.prob, self.dt, self.nt = prob, dt, nt
        x0, x1, y0, y1 = prob.domain
        self.mesh = fe.Mesh(x0, x1, y0, y1, nx, ny)
        kv = prob.vel_degree
        self.vel = fe.Space(self.mesh, kv, 2)
        self.prs = fe.Space(self.mesh, kv - 1)
        self.cur = fe.Space(self.mesh, 1)
        self.pot = fe.Space(self.mesh, 1)
        self.n_u, self.n_p = self.vel.ndof, self.prs.ndof
        self.n_j, self.n_a = self.cur.ndof, self.pot.ndof
        self.slab = self.n_u + self.n_p + self.n_j + self.n_a
        self.off = {"u": 0, "p": self.n_u, "j": self.n_u + self.n_p,
                    "A": self.n_u + self.n_p + self.n_j}
        self.mu, self.eta, self.mu0 = prob.mu, prob.eta, prob.mu0

        self.mass_u, self.stiff_u = fe.mass(self.vel), fe.stiffness(self.vel)
        self.mass_p, self.stiff_p = fe.mass(self.prs), fe.stiffness(self.prs)
        self.mass_j = fe.mass(self.cur)
        self.mass_a, self.stiff_a = fe.mass(self.pot), fe.stiffness(self.pot)
        self.mixed_ja = fe.mixed_grad(self.cur, self.pot)
        self.div = fe.neg_divergence(self.vel, self.prs)
        self.e_load = fe.load(self.pot, prob.e_eq)
        flux = np.zeros(self.n_j)
        for side in fe.SIDES:  # problems.py:185-188 (+ bottom edge)
            if side in prob.flux:
                flux = flux + fe.edge_load(self.cur, side, prob.flux[side])
        self.current_flux = flux / prob.mu0

        self.u_bc = fe.slip_dofs(self.vel)
        self.u_bc_vals = np.zeros(len(self.u_bc))
        self.a_bc, self.a_bc_vals = fe.dirichlet_dofs(self.pot, prob.a_dirichlet, prob.a_eq)

        self.p_pin = 0  # problems.py:199-206
        m = fe.load(self.prs, lambda x, y: 1.0 + 0.0 * x)
        self.p_mean_row = m / np.linalg.norm(m)
        self.p_mean_mass = float(self.p_mean_row @ np.ones(self.n_p))
        p0 = self.prs.interp(prob.p_eq)
        p0 = p0 - fe.integral(self.prs, p0) / self.mesh.area
        self.p_init = p0
        self.p_mean_target = float(self.p_mean_row @ p0)

        pin = np.array([self.p_pin])  # problems.py:208-222
        self.div_bc = fe.bc_zero(self.div, rows=pin, cols=self.u_bc)
        self.div_t_bc = fe.bc_zero(self.div.T.tocsr(), rows=self.u_bc)
        self.mixed_ja_bc = fe.bc_zero((self.mixed_ja / self.mu0).tocsr(), cols=self.a_bc)
        self.mass_u_dt_bc = fe.bc_zero((self.mass_u / dt).tocsr(), rows=self.u_bc, cols=self.u_bc)
        self.mass_a_dt_bc = fe.bc_zero((self.mass_a / dt).tocsr(), rows=self.a_bc, cols=self.a_bc)
        self.mass_a_bc = fe.bc_identity(self.mass_a, self.a_bc)
        self.mass_a_coupling = fe.bc_zero(self.mass_a, rows=self.a_bc, cols=self.a_bc)
        self.stiff_a_bc0 = fe.bc_zero(self.stiff_a, rows=self.a_bc, cols=self.a_bc)
        self.stiff_p_pinned = fe.bc_identity(self.stiff_p, pin)

        self.lu_mass_j = LU(self.mass_j)  # problems.py:225-228
        self.lu_mass_a = LU(self.mass_a_bc)
        self.lu_mass_p = LU(self.mass_p)
        self.lu_stiff_p = LU(self.stiff_p_pinned)

    def clamp_u(self, u):
        u = u.copy()
        u[self.u_bc] = self.u_bc_vals
        return u

    def clamp_a(self, a):
        a = a.copy()
        a[self.a_bc] = self.a_bc_vals
        return a

    def field(self, vec, k, name):
        lo = k * self.slab + self.off[name]
        n = {"u": self.n_u, "p": self.n_p, "j": self.n_j, "A": self.n_a}[name]
        return vec[lo:lo + n]

    def fields(self, vec):
        """(nt, n) views of the four fields of a flat space-time vector."""
        v = np.asarray(vec).reshape(-1, self.slab)
        o = self.off
        return (v[:, :self.n_u], v[:, o["p"]:o["j"]],
                v[:, o["j"]:o["A"]], v[:, o["A"]:])

    def join(self, u, p, j, a):
        return np.concatenate([u, p, j, a], axis=1).ravel()


def make_disc(prob: ProblemSpec, n: int, dt: float, nt: int) -> Disc:
    """n cells along x (square cells), nt slabs of width dt."""
    x0, x1, y0, y1 = prob.domain
    return Disc(prob, n, int(round(n * (y1 - y0) / (x1 - x0))), dt, nt)


def make_disc_dx(prob: ProblemSpec, dx: float, dt: float, t_final: float) -> Disc:
    """Reference-style constructor (problems.py:150-166): dx, dt, T."""
    x0, x1, y0, y1 = prob.domain
    return Disc(prob, int(round((x1 - x0) / dx)), int(round((y1 - y0) / dx)), dt,
                int(round(t_final / dt)))


@dataclass
class State:
    vec: np.ndarray
    ic_u: np.ndarray
    ic_a: np.ndarray

    def copy(self):
        return State(self.vec.copy(), self.ic_u.copy(), self.ic_a.copy())


def initial_state(d: Disc, nt: int | None = None) -> State:
    """Equilibrium-projection guess, reference problems.py:263-287."""
    nt = d.nt if nt is None else nt
    pr = d.prob
    a_guess = d.pot.interp(pr.a_eq)
    a_ic = d.pot.interp(lambda x, y: pr.a_eq(x, y) + pr.a_pert(x, y))
    j_guess = d.lu_mass_j.solve(d.current_flux - (d.mixed_ja @ a_guess) / d.mu0)
    slab = np.concatenate([np.zeros(d.n_u), d.p_init, j_guess, a_guess])
    return State(np.tile(slab, nt), np.zeros(d.n_u), a_ic)


def _galerkin(d: Disc, u, p, j, a, u_prev, a_prev):
    """reference spacetime.py:42-62."""
    adv, _, _ = fe.momentum_advection(d.vel, u)
    lor, _, _ = fe.lorentz(d.vel, d.cur, d.pot, j, a)
    r_u = (d.mass_u @ (u - u_prev) / d.dt + d.mu * (d.stiff_u @ u) + d.div.T @ p + adv + lor)
    r_p = d.div @ u
    r_j = d.mass_j @ j + (d.mixed_ja @ a) / d.mu0 - d.current_flux
    adva, _, _ = fe.potential_advection(d.pot, d.vel, u, a)
    r_a = (d.mass_a @ (a - a_prev) / d.dt + (d.eta / d.mu0) * (d.stiff_a @ a) + adva + d.e_load)
    return r_u, r_p, r_j, r_a


def residual(state: State, d: Disc) -> np.ndarray:
    """reference spacetime.py:65-85."""
    nt = len(state.vec) // d.slab
    out = np.zeros_like(state.vec)
    up, ap = state.ic_u, state.ic_a
    for k in range(nt):
        ur, pr_, jr, ar = (d.field(state.vec, k, f) for f in "u p j A".split())
        u, a = d.clamp_u(ur), d.clamp_a(ar)
        r_u, r_p, r_j, r_a = _galerkin(d, u, pr_.copy(), jr.copy(), a, up, ap)
        r_u[d.u_bc] = ur[d.u_bc] - d.u_bc_vals
        r_p[d.p_pin] = d.p_mean_row @ pr_ - d.p_mean_target
        r_a[d.a_bc] = ar[d.a_bc] - d.a_bc_vals
        base = k * d.slab
        out[base:base + d.slab] = np.concatenate([r_u, r_p, r_j, r_a])
        up, ap = u, a
    return out


@dataclass
class Blocks:
    f_u: sp.csr_matrix
    z_j: sp.csr_matrix
    z_a: sp.csr_matrix
    y: sp.csr_matrix
    f_a: sp.csr_matrix


def linearize(d: Disc, u, j, a) -> Blocks:
    """reference spacetime.py:99-112 (state already clamped)."""
    _, tr, re = fe.momentum_advection(d.vel, u)
    f_u = d.mass_u / d.dt + d.mu * d.stiff_u + (tr + re).tocsr()
    _, z_j, z_a = fe.lorentz(d.vel, d.cur, d.pot, j, a)
    _, lin_a, lin_u = fe.potential_advection(d.pot, d.vel, u, a)
    f_a = d.mass_a / d.dt + (d.eta / d.mu0) * d.stiff_a + lin_a
    return Blocks(fe.bc_identity(f_u.tocsr(), d.u_bc), fe.bc_zero(z_j, rows=d.u_bc),
                  fe.bc_zero(z_a, rows=d.u_bc, cols=d.a_bc),
                  fe.bc_zero(lin_u, rows=d.a_bc, cols=d.u_bc), fe.bc_identity(f_a.tocsr(), d.a_bc))


class Jacobian:
    """Per-slab blocks + shared couplings; matvec of reference
    spacetime.py:131-153."""

    def __init__(self, d: Disc, slabs):
        self.d, self.slabs, self.nt = d, slabs, len(slabs)
        self.size = self.nt * d.slab

    def apply(self, v):
        d = self.d
        u, p, j, a = d.fields(v)
        ou, op, oj, oa = [], [], [], []
        for k, b in enumerate(self.slabs):
            xu = b.f_u @ u[k] + d.div_t_bc @ p[k] + b.z_j @ j[k] + b.z_a @ a[k]
            xp = d.div_bc @ u[k]
            xp[d.p_pin] += d.p_mean_row @ p[k]
            xj = d.mass_j @ j[k] + d.mixed_ja_bc @ a[k]
            xa = b.y @ u[k] + b.f_a @ a[k]
            if k > 0:
                xu = xu - d.mass_u_dt_bc @ u[k - 1]
                xa = xa - d.mass_a_dt_bc @ a[k - 1]
            ou.append(xu), op.append(xp), oj.append(xj), oa.append(xa)
        return d.join(np.array(ou), np.array(op), np.array(oj), np.array(oa))

    def abs_apply(self, v):
        """|J| |v| -- the rounding scale of each output entry (test helper)."""
        d = self.d
        u, p, j, a = d.fields(np.abs(v))
        A = abs
        ou, op, oj, oa = [], [], [], []
        for k, b in enumerate(self.slabs):
            xu = A(b.f_u) @ u[k] + A(d.div_t_bc) @ p[k] + A(b.z_j) @ j[k] + A(b.z_a) @ a[k]
            xp = A(d.div_bc) @ u[k]
            xp[d.p_pin] += np.abs(d.p_mean_row) @ p[k]
            xj = A(d.mass_j) @ j[k] + A(d.mixed_ja_bc) @ a[k]
            xa = A(b.y) @ u[k] + A(b.f_a) @ a[k]
            if k > 0:
                xu = xu + A(d.mass_u_dt_bc) @ u[k - 1]
                xa = xa + A(d.mass_a_dt_bc) @ a[k - 1]
            ou.append(xu), op.append(xp), oj.append(xj), oa.append(xa)
        return d.join(np.array(ou), np.array(op), np.array(oj), np.array(oa))


def jacobian(state: State, d: Disc) -> Jacobian:
    """reference spacetime.py:167-175."""
    nt = len(state.vec) // d.slab
    slabs = []
    for k in range(nt):
        u = d.clamp_u(d.field(state.vec, k, "u"))
        a = d.clamp_a(d.field(state.vec, k, "A"))
        slabs.append(linearize(d, u, d.field(state.vec, k, "j").copy(), a))
    return Jacobian(d, slabs)


def alfven(d: Disc, state: State):
    """reference precond.py:46-57 on clamped A of each slab."""
    nt = len(state.vec) // d.slab
    out = np.empty(nt)
    for k in range(nt):
        g = fe.mean_grad(d.pot, d.clamp_a(d.field(state.vec, k, "A")))
        out[k] = float(g @ g) / d.mu0
    return out
