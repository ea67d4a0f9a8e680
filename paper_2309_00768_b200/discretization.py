"""Discretisation: host setup + the device handle (drop-in for reference
``problems.Discretization``, ``discretize`` and ``initial_state``,
problems.py:141-287).

All state-independent data is built once on the host (scipy) and uploaded to
the native handle, which owns the device tables, the fixed CSR patterns and
the nested-dissection symbolic factorisations, and factors the constant
blocks M_j, M_A^bc, M_p, K_p^pin on the device (problems.py:225-228).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib, fem
from .errors import ConfigurationError
from .linalg import BlockVector, FieldLayout, as_device
from .patterns import SlabPattern, csr_arrays, product_plan
from .problems import ProblemSpec, constrained_dofs, flux_terms


def _cell_count(length, dx):
    n = length / dx
    if round(n) < 1 or abs(n - round(n)) > 1e-9 * max(1.0, abs(n)):
        raise ConfigurationError(f"extent {length} is not an integer multiple of dx={dx}")
    return int(round(n))


class Discretization:
    """A problem on one space-time grid, resident on the GPU."""

    def __init__(self, problem: ProblemSpec, dx: float, dt: float, t_final: float, leaf=None):
        if dt <= 0 or t_final <= 0:
            raise ConfigurationError("dt and T must be positive")
        nst = t_final / dt
        if abs(nst - round(nst)) > 1e-9 or round(nst) < 1:
            raise ConfigurationError(f"T={t_final} is not an integer multiple of dt={dt}")
        kv = getattr(problem, "vel_degree", 3)  # a reference ProblemSpec: P3/P2
        if kv not in (2, 3):
            raise ConfigurationError("velocity degree must be 2 or 3")
        self.problem, self.dt, self.t_final = problem, dt, t_final
        self.n_steps = int(round(nst))
        x0, x1, y0, y1 = problem.domain
        self.mesh = fem.Mesh(x0, x1, y0, y1, _cell_count(x1 - x0, dx), _cell_count(y1 - y0, dx))
        self.vel = fem.Space(self.mesh, kv, 2)
        self.prs = fem.Space(self.mesh, kv - 1)
        self.cur = fem.Space(self.mesh, 1)
        self.pot = self.cur
        self.layout = FieldLayout(self.vel.ndof, self.prs.ndof, self.cur.ndof, self.pot.ndof)
        self.mu, self.eta, self.mu0 = problem.mu, problem.eta, problem.mu0
        m = self.mesh
        self.tensors = T = fem.element_tensors(kv, kv - 1, m.hx, m.hy)

        ops = fem.constant_operators(self.vel, self.prs, self.cur, T)
        self.mass_u, self.stiff_u = ops["mass_u"], ops["stiff_u"]
        self.mass_p, self.stiff_p = ops["mass_p"], ops["stiff_p"]
        self.mass_j = self.mass_a = ops["mass_1"]
        self.stiff_a = ops["stiff_1"]
        self.mixed_ja = ops["stiff_1"]
        self.div = ops["div"]
        self.e_load = fem.load_vector(self.pot, problem.e_eq)
        flux = np.zeros(self.cur.ndof)
        fterms = flux_terms(problem)
        for side in fem.SIDES:
            if side in fterms:
                flux = flux + fem.edge_load_vector(self.cur, side, fterms[side])
        self.current_flux = flux / problem.mu0

        # constrained DOFs from the problem's BCSpec (reference problems.py:179-180)
        self.u_bc_idx, self.u_bc_vals = constrained_dofs(self.vel, problem, "u")
        self.a_bc_idx, self.a_bc_vals = constrained_dofs(self.pot, problem, "A")

        self.p_pin = 0
        mvec = fem.load_vector(self.prs, lambda x, y: 1.0 + 0.0 * x)
        self.p_mean_row = mvec / np.linalg.norm(mvec)
        self.p_mean_mass = float(self.p_mean_row @ np.ones(self.prs.ndof))
        p0 = self.prs.interp(problem.p_eq)
        p0 = p0 - fem.mean_integral(self.prs, p0, T["MP"]) / m.area
        self._p_init = p0
        self.p_mean_target = float(self.p_mean_row @ p0)

        pin = np.array([self.p_pin])
        bz, bi = fem.bc_zero, fem.bc_identity
        self.div_bc = bz(self.div, rows=pin, cols=self.u_bc_idx)
        self.div_t_bc = bz(self.div.T.tocsr(), rows=self.u_bc_idx)
        self.mixed_ja_bc = bz((self.mixed_ja / self.mu0).tocsr(), cols=self.a_bc_idx)
        self.mass_u_dt_bc = bz((self.mass_u / dt).tocsr(), rows=self.u_bc_idx, cols=self.u_bc_idx)
        self.mass_a_dt_bc = bz((self.mass_a / dt).tocsr(), rows=self.a_bc_idx, cols=self.a_bc_idx)
        self.mass_a_bc = bi(self.mass_a, self.a_bc_idx)
        self.mass_a_coupling = bz(self.mass_a, rows=self.a_bc_idx, cols=self.a_bc_idx)
        self.stiff_a_bc0 = bz(self.stiff_a, rows=self.a_bc_idx, cols=self.a_bc_idx)
        self.stiff_p_pinned = bi(self.stiff_p, pin)
        self.stiff_p_zrow = bz(self.stiff_p, rows=pin)

        self.pattern = SlabPattern(self.vel, self.prs, self.cur,
                                   (self.layout.n_u, self.layout.n_p, self.layout.n_j, self.layout.n_a),
                                   self.u_bc_idx, self.a_bc_idx)
        self.leaf = leaf or {}
        self._bound_nt = self.n_steps
        self._handle = None
        self._build_handle()

    # -- native handle -------------------------------------------------------------
    def _build_handle(self):
        lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(lib.stmhd_disc_create(ctypes.byref(h)))
        self._handle = h
        self._keep = []
        L = self.layout
        P = self.pattern
        o_p, o_j, o_a = P.offsets
        ints = dict(nt=self.n_steps, n_u=L.n_u, n_p=L.n_p, n_j=L.n_j, n_a=L.n_a,
                    nv=self.vel.nloc, npl=self.prs.nloc, ne=self.mesh.ne, nnv=self.vel.n_nodes,
                    nnp=self.prs.n_nodes, nn1=self.cur.n_nodes, p_pin=self.p_pin,
                    nnz_js=P.nnz, nnz_fp=P.fp_nnz,
                    leaf_fu=self.leaf.get("fu", 32), leaf_ca=self.leaf.get("ca", 32),
                    leaf_c=self.leaf.get("const", 32))
        for k, v in ints.items():
            _lib.check(lib.stmhd_disc_set_int(h, k.encode(), int(v)))
        reals = dict(dt=self.dt, mu=self.mu, eta=self.eta, mu0=self.mu0,
                     p_mean_target=self.p_mean_target, p_mean_mass=self.p_mean_mass,
                     area=self.mesh.area, elem_area=0.5 * self.mesh.hx * self.mesh.hy)
        for k, v in reals.items():
            _lib.check(lib.stmhd_disc_set_real(h, k.encode(), float(v)))

        def up(key, arr):
            arr = np.ascontiguousarray(arr)
            if arr.dtype.kind in "iu":
                arr = np.ascontiguousarray(arr, dtype=np.int32)
                es = 4
            else:
                arr = np.ascontiguousarray(arr, dtype=np.float64)
                es = 8
            _lib.check(lib.stmhd_disc_upload(h, key.encode(), _lib.ptr(arr), arr.size, es))

        T = self.tensors
        blob = np.concatenate([T[k].ravel() for k in ("MV", "KV", "TV", "MX", "G1", "M1", "K1",
                                                      "MP", "KP", "TP", "BD")])
        up("tensors", blob)
        up("elem_v", self.vel.elem)
        up("elem_p", self.prs.elem)
        up("elem_1", self.cur.elem)
        for name, sp_ in (("v", self.vel), ("p", self.prs), ("1", self.cur)):
            ptr, code = sp_.node_elements()
            up(f"ne_{name}_ptr", ptr)
            up(f"ne_{name}", code)
        ubm = np.zeros(L.n_u, np.int32)
        ubm[self.u_bc_idx] = 1
        ubv = np.zeros(L.n_u)
        ubv[self.u_bc_idx] = self.u_bc_vals
        abm = np.zeros(L.n_a, np.int32)
        abm[self.a_bc_idx] = 1
        abv = np.zeros(L.n_a)
        abv[self.a_bc_idx] = self.a_bc_vals
        up("u_bc_mask", ubm), up("u_bc_val", ubv), up("a_bc_mask", abm), up("a_bc_val", abv)
        up("p_mean_row", self.p_mean_row), up("flux", self.current_flux), up("e_load", self.e_load)
        # merged per-slab pattern + contributions
        up("js_rowptr", P.rowptr), up("js_col", P.col), up("js_kind", P.kind)
        up("js_cptr", P.cptr.astype(np.int32)), up("js_contrib", P.contrib)
        up("js_seg0", P.seg0_end), up("js_seg1", P.seg1_end)
        up("fp_rowptr", P.fp_rowptr), up("fp_col", P.fp_col)
        up("fp_cptr", P.fp_cptr.astype(np.int32)), up("fp_contrib", P.fp_contrib)
        # merged shared CSR for J.apply: columns relative to the slab start
        # (negative = previous slab)
        nz = sp.csr_matrix((L.n_p, L.n_p))
        cur = sp.bmat([
            [sp.csr_matrix((L.n_u, L.n_u)), self.div_t_bc, sp.csr_matrix((L.n_u, L.n_j)), sp.csr_matrix((L.n_u, L.n_a))],
            [self.div_bc, nz, sp.csr_matrix((L.n_p, L.n_j)), sp.csr_matrix((L.n_p, L.n_a))],
            [sp.csr_matrix((L.n_j, L.n_u)), sp.csr_matrix((L.n_j, L.n_p)), self.mass_j, self.mixed_ja_bc],
            [sp.csr_matrix((L.n_a, L.n_u)), sp.csr_matrix((L.n_a, L.n_p)), sp.csr_matrix((L.n_a, L.n_j)),
             sp.csr_matrix((L.n_a, L.n_a))]]).tocsr()
        prev = sp.bmat([
            [-self.mass_u_dt_bc, None, None, None],
            [None, sp.csr_matrix((L.n_p, L.n_p)), None, None],
            [None, None, sp.csr_matrix((L.n_j, L.n_j)), None],
            [None, None, None, -self.mass_a_dt_bc]]).tocsr()
        big = sp.hstack([prev, cur]).tocsr()
        rp, ci, va = csr_arrays(big)
        up("jc_rowptr", rp), up("jc_col", ci.astype(np.int64) - L.slab_size), up("jc_val", va)
        self.jc_nnz = len(ci)
        # element-matrix patch plan of the Jacobian assembly (P2/P1)
        from .asm_patches import build_patch_plan, build_residual_plan

        ps = os.environ.get("STMHD_PATCH", "6x5").split("x")  # cells per patch (r01 sweep: 6x5 best)
        pp = build_patch_plan(self, int(ps[0]), int(ps[1]))
        if pp is not None:
            up("pa_desc", pp["desc"]), up("pa_slots", pp["slots"]), up("pa_out", pp["out"])
            up("pa_codes", pp["codes"]), up("pa_w", pp["w"])
            for k, v in (("pa_npatch", pp["npatch"]), ("pa_max_slots", pp["max_slots"])):
                _lib.check(lib.stmhd_disc_set_int(h, k.encode(), int(v)))
        rs = os.environ.get("STMHD_RPATCH", "16x8").split("x")  # residual patch cells (r01 sweep: 16x8 best)
        rp_ = build_residual_plan(self, int(rs[0]), int(rs[1]))
        if rp_ is not None:
            up("pr_desc", rp_["desc"]), up("pr_slots", rp_["slots"]), up("pr_out", rp_["out"])
            up("pr_codes", rp_["codes"]), up("pr_add", rp_["add"])
            for k, v in (("pr_npatch", rp_["npatch"]), ("pr_max_slots", rp_["max_slots"])):
                _lib.check(lib.stmhd_disc_set_int(h, k.encode(), int(v)))
        # preconditioner CSRs (field-local coordinates)
        for key, mat in (("mu_dt", self.mass_u_dt_bc), ("ma_dt", self.mass_a_dt_bc),
                         ("mp_dt", (self.mass_p / self.dt).tocsr()), ("divt", self.div_t_bc),
                         ("div", self.div_bc), ("mixja", self.mixed_ja_bc), ("mj", self.mass_j),
                         ("mabc", self.mass_a_bc), ("mp", self.mass_p), ("kpz", self.stiff_p_zrow)):
            rp, ci, va = csr_arrays(mat)
            up(key + "_rowptr", rp), up(key + "_col", ci), up(key + "_val", va)
        dinv = 1.0 / self.mass_a_bc.diagonal()
        c_sub2 = ((1.0 / self.dt**2) * (self.mass_a_coupling @ sp.diags(dinv) @ self.mass_a_coupling)).tocsr()
        rp, ci, va = csr_arrays(c_sub2, drop_zeros=False)
        up("sub2_rowptr", rp), up("sub2_col", ci), up("sub2_val", va)
        self.c_a_sub2 = c_sub2
        # blocks of the merged pattern used by the factorisations
        fu_rp, fu_col, fu_map = P.block(0, L.n_u, 0, 0, L.n_u)
        fa_rp, fa_col, fa_map = P.block(o_a, o_a + L.n_a, 1, o_a, o_a + L.n_a)
        up("fu_rowptr", fu_rp), up("fu_col", fu_col), up("fu_map", fu_map)
        up("fa_rowptr", fa_rp), up("fa_col", fa_col), up("fa_map", fa_map)
        self._fa_block = (fa_rp, fa_col, fa_map)
        gi_v = np.tile(self.vel.gi, 2)
        gj_v = np.tile(self.vel.gj, 2)
        up("fu_gx", gi_v), up("fu_gy", gj_v)
        up("p1_gx", self.cur.gi), up("p1_gy", self.cur.gj)
        up("prs_gx", self.prs.gi), up("prs_gy", self.prs.gj)
        # C_A = f_a D^-1 f_a + s K_bc0 (precond.py:91-96): entry-centric product plan
        F = sp.csr_matrix((np.arange(len(fa_col), dtype=np.float64) + 1, fa_col, fa_rp),
                          shape=(L.n_a, L.n_a))
        pl = product_plan(F, F)
        ca = sp.csr_matrix((np.ones(len(pl["col"])), pl["col"], pl["rowptr"]), shape=(L.n_a, L.n_a))
        kb = self.stiff_a_bc0.tocsr()
        kval = np.asarray(kb[ca.nonzero()]).ravel() if ca.nnz else np.zeros(0)
        # ca.nonzero() is row-major sorted like pl
        up("ca_rowptr", pl["rowptr"]), up("ca_col", pl["col"]), up("ca_pptr", pl["pptr"])
        up("ca_a", fa_map[pl["a"]]), up("ca_b", fa_map[pl["b"]]), up("ca_w", dinv[pl["l"]])
        up("ca_k", kval)
        self._ca_pattern = (pl["rowptr"], pl["col"])
        # sub1_k = -(1/dt)(Mc D^-1 f_a,k + f_a,k+1 D^-1 Mc)  (precond.py:100-104)
        Mc = sp.csr_matrix(self.mass_a_coupling)
        Mc.sort_indices()
        p1 = product_plan(Mc, F)
        p2 = product_plan(F, Mc)
        rows1 = np.repeat(np.arange(L.n_a), np.diff(p1["rowptr"]))
        rows2 = np.repeat(np.arange(L.n_a), np.diff(p2["rowptr"]))
        e1 = np.repeat(np.arange(len(p1["col"])), np.diff(p1["pptr"]))
        e2 = np.repeat(np.arange(len(p2["col"])), np.diff(p2["pptr"]))
        r_all = np.concatenate([rows1[e1], rows2[e2]])
        c_all = np.concatenate([p1["col"][e1], p2["col"][e2]])
        coef = np.concatenate([-Mc.data[p1["a"]] * dinv[p1["l"]] / self.dt,
                               -dinv[p2["l"]] * Mc.data[p2["b"]] / self.dt])
        idx = np.concatenate([fa_map[p1["b"]], fa_map[p2["a"]]])
        which = np.concatenate([np.zeros(len(e1), np.int32), np.ones(len(e2), np.int32)])
        order = np.lexsort((which, c_all, r_all))
        r_all, c_all, coef, idx, which = (x[order] for x in (r_all, c_all, coef, idx, which))
        key = r_all.astype(np.int64) * L.n_a + c_all
        ukey, start, cnt = np.unique(key, return_index=True, return_counts=True)
        s1_rp = np.zeros(L.n_a + 1, np.int64)
        np.add.at(s1_rp, ukey // L.n_a + 1, 1)
        up("s1_rowptr", np.cumsum(s1_rp)), up("s1_col", ukey % L.n_a)
        up("s1_pptr", np.concatenate([[0], np.cumsum(cnt)])), up("s1_coef", coef)
        up("s1_idx", idx), up("s1_which", which)
        self._s1_pattern = (np.cumsum(s1_rp).astype(np.int32), (ukey % L.n_a).astype(np.int32))
        # constant factorisations (problems.py:225-228)
        for key, mat, space in (("lu_mj", self.mass_j, self.cur), ("lu_ma", self.mass_a_bc, self.cur),
                                ("lu_mp", self.mass_p, self.prs), ("lu_kp", self.stiff_p_pinned, self.prs)):
            rp, ci, va = csr_arrays(mat, drop_zeros=False)
            up(key + "_rowptr", rp), up(key + "_col", ci), up(key + "_val", va)
        _lib.check(lib.stmhd_disc_finalize(h, _lib.stream_ptr()))
        torch.cuda.synchronize()

    def __del__(self):
        try:
            if self._handle:
                _lib.load().stmhd_disc_destroy(self._handle)
        except Exception:
            pass

    @property
    def handle(self):
        return self._handle

    def device_bytes(self) -> int:
        return int(_lib.load().stmhd_disc_device_bytes(self._handle))

    # -- reference helpers -------------------------------------------------------------
    def clamp(self, u=None, p=None, j=None, a=None):
        """Copies with constrained entries set to BC values (problems.py:230-247)."""
        out = []
        if u is not None:
            u = as_device(u).clone()
            u[torch.as_tensor(self.u_bc_idx, device=u.device)] = torch.as_tensor(self.u_bc_vals, device=u.device)
            out.append(u)
        if p is not None:
            out.append(as_device(p).clone())
        if j is not None:
            out.append(as_device(j).clone())
        if a is not None:
            a = as_device(a).clone()
            a[torch.as_tensor(self.a_bc_idx, device=a.device)] = torch.as_tensor(self.a_bc_vals, device=a.device)
            out.append(a)
        return out if len(out) > 1 else out[0]

    def project_zero_mean(self, p_coef):
        p = as_device(p_coef)
        w = torch.as_tensor(self.tensors["MP"].sum(axis=1), device=p.device)
        mean = float((p[torch.as_tensor(self.prs.elem, device=p.device)] @ w).sum()) / self.mesh.area
        return p - mean

    def solve_current_init(self, a_coef):
        """j with M_j j = flux - K_jA a / mu0 (problems.py:253-256)."""
        from .linalg import LUFactor

        if not hasattr(self, "_lu_mj"):
            self._lu_mj = LUFactor(self.mass_j, coords=(self.cur.gi, self.cur.gj))
        a = np.asarray(a_coef.cpu() if isinstance(a_coef, torch.Tensor) else a_coef)
        rhs = self.current_flux - (self.mixed_ja @ a) / self.mu0
        return self._lu_mj.solve(as_device(rhs))


def discretize(problem: ProblemSpec, dx: float, dt: float, t_final: float, **kw) -> Discretization:
    return Discretization(problem, dx, dt, t_final, **kw)


def discretize_config(name: str, **kw) -> Discretization:
    """A BASELINE.json configuration by name (C1, C2, C3, C4_64, ...)."""
    from .problems import config_problem

    prob, n, dt, nt, _ = config_problem(name)
    x0, x1, _, _ = prob.domain
    return Discretization(prob, (x1 - x0) / n, dt, nt * dt, **kw)


def initial_state(disc: Discretization, n_steps: int | None = None):
    """Equilibrium-projection initial guess (reference problems.py:263-287):
    u = 0, zero-mean equilibrium pressure, unperturbed potential and the
    consistent current on every slab; the perturbed potential as IC."""
    from .spacetime import SpaceTimeState

    n = disc.n_steps if n_steps is None else n_steps
    prob = disc.problem
    a_guess = disc.pot.interp(prob.a_eq)
    a_ic = disc.pot.interp(lambda x, y: prob.a_eq(x, y) + prob.a_perturbation(x, y))
    j_guess = disc.solve_current_init(a_guess)
    L = disc.layout
    slab = torch.cat([torch.zeros(L.n_u, dtype=torch.float64, device="cuda"), as_device(disc._p_init),
                      as_device(j_guess), as_device(a_guess)])
    vec = BlockVector(L, n, slab.repeat(n))
    return SpaceTimeState(vec, torch.zeros(L.n_u, dtype=torch.float64, device="cuda"), as_device(a_ic))
