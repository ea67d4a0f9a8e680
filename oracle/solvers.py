"""Space-time block preconditioner P_T, MGS GMRES and the Newton driver
(TEST INFRASTRUCTURE ONLY -- CPU restatement of reference ``precond.py``,
``linalg.py:99-209`` and ``solver.py:87-122``)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import fe
from .model import LU, Disc, Jacobian, State, alfven, jacobian, residual


class Precond:
    """Per-slab factors at one linearisation point, TRIANGULAR variant
    (reference precond.py:67-106, 122-301)."""

    def __init__(self, jac: Jacobian, d: Disc, state: State):
        self.d, self.jac, self.nt = d, jac, jac.nt
        self.lu_f_u = [LU(b.f_u) for b in jac.slabs]
        self.f_p = []
        for k in range(self.nt):
            u = d.clamp_u(d.field(state.vec, k, "u"))
            w_p = fe.pcd_advection(d.prs, d.vel, u)
            self.f_p.append((d.mass_p / d.dt + w_p + d.mu * d.stiff_p).tocsr())
        self.lu_f_p = [LU(m) for m in self.f_p]
        self.stiff_p_zrow = fe.bc_zero(d.stiff_p, rows=np.array([d.p_pin]))
        self.alfven = alfven(d, state)
        dinv = sp.diags(1.0 / d.mass_a_bc.diagonal()).tocsr()
        self.c_a = [(b.f_a @ dinv @ b.f_a + s * d.stiff_a_bc0).tocsr()
                    for b, s in zip(jac.slabs, self.alfven)]
        self.lu_c_a = [LU(m) for m in self.c_a]
        mc = d.mass_a_coupling
        self.c_a_sub1 = [((-1.0 / d.dt) * (mc @ dinv @ jac.slabs[k].f_a
                                          + jac.slabs[k + 1].f_a @ dinv @ mc)).tocsr()
                         for k in range(self.nt - 1)]
        self.c_a_sub2 = ((1.0 / d.dt**2) * (mc @ dinv @ mc)).tocsr()
        self._lu_f_a = None

    def lu_f_a(self, k):
        if self._lu_f_a is None:
            self._lu_f_a = [LU(b.f_a) for b in self.jac.slabs]
        return self._lu_f_a[k]

    # sequential sweeps and bidiagonal applies (precond.py:122-205)
    def solve_velocity(self, r):
        r = r.reshape(self.nt, -1)
        x = np.empty_like(r)
        for k in range(self.nt):
            rhs = r[k] if k == 0 else r[k] + self.d.mass_u_dt_bc @ x[k - 1]
            x[k] = self.lu_f_u[k].solve(rhs)
        return x.ravel()

    def apply_velocity(self, v):
        v = v.reshape(self.nt, -1)
        out = np.empty_like(v)
        for k in range(self.nt):
            out[k] = self.jac.slabs[k].f_u @ v[k]
            if k:
                out[k] -= self.d.mass_u_dt_bc @ v[k - 1]
        return out.ravel()

    def apply_pressure_cd(self, v):
        cpl = self.d.mass_p / self.d.dt
        v = v.reshape(self.nt, -1)
        out = np.empty_like(v)
        for k in range(self.nt):
            out[k] = self.f_p[k] @ v[k]
            if k:
                out[k] -= cpl @ v[k - 1]
        return out.ravel()

    def solve_pressure_cd(self, r):
        cpl = self.d.mass_p / self.d.dt
        r = r.reshape(self.nt, -1)
        x = np.empty_like(r)
        for k in range(self.nt):
            x[k] = self.lu_f_p[k].solve(r[k] if k == 0 else r[k] + cpl @ x[k - 1])
        return x.ravel()

    def apply_potential(self, v):
        v = v.reshape(self.nt, -1)
        out = np.empty_like(v)
        for k in range(self.nt):
            out[k] = self.jac.slabs[k].f_a @ v[k]
            if k:
                out[k] -= self.d.mass_a_dt_bc @ v[k - 1]
        return out.ravel()

    def solve_potential(self, r):
        r = r.reshape(self.nt, -1)
        x = np.empty_like(r)
        for k in range(self.nt):
            x[k] = self.lu_f_a(k).solve(r[k] if k == 0 else r[k] + self.d.mass_a_dt_bc @ x[k - 1])
        return x.ravel()

    def apply_wave(self, v):
        v = v.reshape(self.nt, -1)
        out = np.empty_like(v)
        for k in range(self.nt):
            out[k] = self.c_a[k] @ v[k]
            if k >= 1:
                out[k] += self.c_a_sub1[k - 1] @ v[k - 1]
            if k >= 2:
                out[k] += self.c_a_sub2 @ v[k - 2]
        return out.ravel()

    def solve_wave(self, r):
        r = r.reshape(self.nt, -1)
        x = np.empty_like(r)
        for k in range(self.nt):
            rhs = r[k].copy()
            if k >= 1:
                rhs -= self.c_a_sub1[k - 1] @ x[k - 1]
            if k >= 2:
                rhs -= self.c_a_sub2 @ x[k - 2]
            x[k] = self.lu_c_a[k].solve(rhs)
        return x.ravel()

    # Schur complements (precond.py:209-250)
    def pressure_schur_inverse(self, r):
        d = self.d
        r = r.reshape(self.nt, -1)
        r_pin = r[:, d.p_pin].copy()
        rh = r.copy()
        rh[:, d.p_pin] = 0.0
        y = np.vstack([d.lu_stiff_p.solve(x) for x in rh])
        z = self.apply_pressure_cd(y.ravel()).reshape(self.nt, -1)
        x = -np.vstack([d.lu_mass_p.solve(v) for v in z])
        alpha = (r_pin - x @ d.p_mean_row) / d.p_mean_mass
        return (x + alpha[:, None]).ravel()

    def pressure_schur_apply(self, x):
        d = self.d
        x = x.reshape(self.nt, -1)
        y = np.vstack([d.mass_p @ v for v in x])
        z = self.solve_pressure_cd(y.ravel()).reshape(self.nt, -1)
        out = -np.vstack([self.stiff_p_zrow @ v for v in z])
        out[:, d.p_pin] = x @ d.p_mean_row
        return out.ravel()

    def magnetic_schur_inverse(self, r):
        r = r.reshape(self.nt, -1)
        v = np.vstack([self.d.lu_mass_a.solve(x) for x in r])
        return self.solve_wave(self.apply_potential(v.ravel()))

    def magnetic_schur_apply(self, x):
        v = self.solve_potential(self.apply_wave(x)).reshape(self.nt, -1)
        return np.vstack([self.d.mass_a_bc @ w for w in v]).ravel()

    def apply_inverse(self, r):
        """TRIANGULAR P_T^{-1} r, reference precond.py:270-301."""
        d, sl, nt = self.d, self.jac.slabs, self.nt
        r_u, r_p, r_j, r_a = (f.copy() for f in d.fields(r))
        x_a = self.magnetic_schur_inverse(r_a.ravel()).reshape(nt, -1)
        x_j = np.vstack([d.lu_mass_j.solve(r_j[k] - d.mixed_ja_bc @ x_a[k]) for k in range(nt)])
        t_u = np.vstack([r_u[k] - sl[k].z_j @ x_j[k] - sl[k].z_a @ x_a[k] for k in range(nt)])
        x_p = self.pressure_schur_inverse(r_p.ravel()).reshape(nt, -1)
        rhs = t_u - np.vstack([d.div_t_bc @ x_p[k] for k in range(nt)])
        x_u = self.solve_velocity(rhs.ravel()).reshape(nt, -1)
        return d.join(x_u, x_p, x_j, x_a)

    def apply_forward(self, x):
        """TRIANGULAR P_T x (round-trip checks), reference precond.py:303-321."""
        d, sl, nt = self.d, self.jac.slabs, self.nt
        x_u, x_p, x_j, x_a = d.fields(x)
        coup = np.vstack([sl[k].z_j @ x_j[k] + sl[k].z_a @ x_a[k] for k in range(nt)])
        o_j = np.vstack([d.mass_j @ x_j[k] + d.mixed_ja_bc @ x_a[k] for k in range(nt)])
        o_a = self.magnetic_schur_apply(x_a.ravel()).reshape(nt, -1)
        o_u = self.apply_velocity(x_u.ravel()).reshape(nt, -1) + coup
        o_u += np.vstack([d.div_t_bc @ x_p[k] for k in range(nt)])
        o_p = self.pressure_schur_apply(x_p.ravel()).reshape(nt, -1)
        return d.join(o_u, o_p, o_j, o_a)


class Breakdown(Exception):
    pass


@dataclass
class GmresOut:
    x: np.ndarray
    iterations: int
    residuals: list = field(default_factory=list)
    converged: bool = True
    true_residual: float = 0.0


def gmres_mgs(apply_a, apply_pinv, b, rel_tol=1e-2, abs_tol=1e-14, max_iters=200, restart=None,
              max_total=None):
    """Right-preconditioned restarted GMRES with MGS + Givens, x0 = 0
    (reference linalg.py:122-209).  ``max_total`` stops the Arnoldi loop
    early for bounded CPU timing samples (not a reference feature)."""
    n = len(b)
    if not np.all(np.isfinite(b)):
        raise Breakdown("rhs")
    x = np.zeros(n)
    r = b.copy()
    beta = float(np.linalg.norm(r))
    res = [beta]
    tol = max(rel_tol * beta, abs_tol)
    if beta <= tol:
        return GmresOut(x, 0, res, True, beta)
    m_restart = restart or max_iters
    total, conv = 0, False
    cap = max_iters if max_total is None else min(max_iters, max_total)
    while total < cap and not conv:
        m = min(m_restart, cap - total)
        # column basis, as the reference stores it (restart + 1 columns: a capped timing
        # sample keeps the reference's column stride)
        V = np.zeros((n, max(m, min(m_restart, max_iters)) + 1))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        V[:, 0] = r / beta
        g[0] = beta
        last = -1
        for j in range(m):
            w = np.array(apply_a(apply_pinv(V[:, j])), dtype=float)
            if not np.all(np.isfinite(w)):
                raise Breakdown("arnoldi")
            for i in range(j + 1):
                H[i, j] = V[:, i] @ w
                w -= H[i, j] * V[:, i]
            H[j + 1, j] = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            last = j
            res.append(abs(float(g[j + 1])))
            if res[-1] <= tol:
                conv = True
                break
            if den == 0.0:
                break
            nw = np.linalg.norm(w)
            if nw > 0:
                V[:, j + 1] = w / nw
        if last >= 0:
            y = np.zeros(last + 1)
            for i in range(last, -1, -1):
                y[i] = (g[i] - H[i, i + 1:last + 1] @ y[i + 1:last + 1]) / H[i, i]
            x = x + apply_pinv(V[:, :last + 1] @ y)
        if conv or total >= cap:
            break
        r = b - apply_a(x)
        beta = float(np.linalg.norm(r))
        if beta <= tol:
            conv = True
            break
    return GmresOut(x, total, res, conv, float(np.linalg.norm(b - apply_a(x))))


@dataclass
class NewtonOut:
    newton_iters: int = 0
    gmres_iters: list = field(default_factory=list)
    residual_norms: list = field(default_factory=list)
    converged: bool = False


def newton_solve(state: State, d: Disc, rel_tol=1e-6, max_newton=25, one_step=False,
                 gmres_kw=None, hook=None):
    """Plain Newton with GMRES(P_T) inner solves (reference solver.py:87-104);
    the stop is relative, abs_tol = rel_tol*||r0||."""
    gkw = dict(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50)
    gkw.update(gmres_kw or {})
    out = NewtonOut()
    abs_tol = None
    for it in range(max_newton + 1):
        r = residual(state, d)
        rn = float(np.linalg.norm(r))
        out.residual_norms.append(rn)
        if abs_tol is None:
            abs_tol = rel_tol * rn
        if rn <= abs_tol or (one_step and out.newton_iters == 1):
            out.converged = rn <= abs_tol
            return out
        if out.newton_iters >= max_newton:
            return out
        jac = jacobian(state, d)
        pc = Precond(jac, d, state)
        res = gmres_mgs(jac.apply, pc.apply_inverse, -r, **gkw)
        if hook is not None:
            hook(it, r, jac, pc, res)
        state.vec += res.x
        out.newton_iters += 1
        out.gmres_iters.append(res.iterations)
    return out
