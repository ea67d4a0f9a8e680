"""Generate golden fixtures from the UNMODIFIED reference package ``stmhd``.

Run in the build container only (the reference is not present on the GPU
box):  ``python tests/golden/make_golden.py``.  It imports
/root/reference/pkg/src/stmhd read-only and writes small ``.npz`` files next
to this script.  BASELINE.json configurations go through the SURVEY.md 0.1
adapter:

* velocity/pressure degrees swapped from P3/P2 to P2/P1 by rebinding
  ``stmhd.problems.FESpace`` while the ``Discretization`` is built,
* domain [-1,1]^2 via a hand-built ``ProblemSpec`` with BASELINE closures,
* A Dirichlet on top *and* bottom; the bottom edge flux is added to
  ``disc.current_flux`` (the attribute is read at spacetime.py:54 and
  problems.py:256),
* GMRES(restart 50) to rel 1e-8 (abs 1e-300).

Cases (file -> content):
  ref_island.npz   reference built-in island, dx=0.5, dt=0.5, T=1 (P3/P2)
  ref_tearing.npz  reference built-in tearing, dx=0.25, dt=0.5, T=1 (P3/P2)
  bl_island4.npz   BASELINE island physics, 4x4 mesh, dt=0.1, Nt=3 (P2/P1)
  bl_tearing4.npz  BASELINE tearing physics, 4x4 mesh, dt=0.02, Nt=2 (P2/P1)
  bl_c1.npz        BASELINE config 1 (16x16, Nt=8): vectors + GMRES count
  c5_tiny.npz      configuration-5 scalar operator at 8x8, Nt=4
"""

from __future__ import annotations

import contextlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import stmhd  # noqa: E402
from stmhd import fem, problems  # noqa: E402
from stmhd.fem import BCSpec, dirichlet, natural, slip  # noqa: E402
from stmhd.mesh import Side  # noqa: E402
from stmhd.precond import SpaceTimePreconditioner  # noqa: E402
from stmhd.spacetime import assemble_jacobian, residual  # noqa: E402

from paper_2309_00768_b200.c5 import c5_velocity_fields  # noqa: E402  (input generator)


@contextlib.contextmanager
def p2p1():
    orig = problems.FESpace

    def swapped(mesh, degree, components=1):
        return orig(mesh, {3: 2, 2: 1, 1: 1}[degree], components=components)

    problems.FESpace = swapped
    try:
        yield
    finally:
        problems.FESpace = orig


def baseline_spec(kind, visc):
    mu0 = 1.0
    if kind == "island":
        beta, tp = 0.2, 2.0 * np.pi

        def sheet(x, y):
            return np.cosh(tp * y) + beta * np.cos(tp * x)

        a_eq = lambda x, y: np.log(sheet(x, y)) / tp  # noqa: E731
        e_eq = lambda x, y: (visc / mu0) * tp * (1 - beta**2) / sheet(x, y) ** 2  # noqa: E731
        p_eq = lambda x, y: (1 - beta**2) / (2 * mu0 * sheet(x, y) ** 2)  # noqa: E731
        dady = lambda x, y: np.sinh(tp * y) / sheet(x, y)  # noqa: E731
        pert = lambda x, y: 1e-3 * np.cos(0.5 * np.pi * x) * np.cos(0.5 * np.pi * y)  # noqa: E731
    else:
        lam = 0.5
        a_eq = lambda x, y: lam * np.log(np.cosh(y / lam)) + 0 * x  # noqa: E731
        e_eq = lambda x, y: (visc / mu0) / lam * np.cosh(y / lam) ** -2 + 0 * x  # noqa: E731
        p_eq = lambda x, y: np.cosh(y / lam) ** -2 / (2 * mu0) + 0 * x  # noqa: E731
        dady = lambda x, y: np.tanh(y / lam) + 0 * x  # noqa: E731
        pert = lambda x, y: 1e-3 * np.cos(np.pi * x) * np.cos(0.5 * np.pi * y)  # noqa: E731
    sym = {s: slip() for s in Side}
    a_cond = {s: natural() for s in Side}
    a_cond[Side.TOP] = dirichlet(a_eq)
    a_cond[Side.BOTTOM] = dirichlet(a_eq)
    bcs = BCSpec(conditions={"u": sym, "p": {s: natural() for s in Side},
                             "j": {s: natural() for s in Side}, "A": a_cond})
    spec = problems.ProblemSpec(name=kind, domain=(-1.0, 1.0, -1.0, 1.0), mu=visc, eta=visc,
                                mu0=mu0, eps=1e-3, a_eq=a_eq, e_eq=e_eq, p_eq=p_eq,
                                a_perturbation=pert, a_eq_normal_flux_top=dady, bcs=bcs)
    return spec, dady


def baseline_disc(kind, visc, n, dt, nt):
    spec, dady = baseline_spec(kind, visc)
    with p2p1():
        disc = problems.Discretization(spec, 2.0 / n, dt, nt * dt)
    disc.current_flux = disc.current_flux + fem.assemble_edge_load(
        disc.cur, Side.BOTTOM, lambda x, y: -dady(x, y)) / spec.mu0
    assert disc.n_steps == nt
    return disc


def csr_dump(prefix, m, out):
    m = m.tocsr()
    out[prefix + "_data"] = m.data
    out[prefix + "_indices"] = m.indices.astype(np.int32)
    out[prefix + "_indptr"] = m.indptr.astype(np.int32)
    out[prefix + "_shape"] = np.array(m.shape)


def full_case(disc, seed, out, blocks=True, solve=True, gmres_cfg=None):
    """Residual, J.v, P^-1 v, per-slab blocks, preconditioner pieces, and a
    small Newton-step GMRES solve at a perturbed state."""
    rng = np.random.default_rng(seed)
    st0 = stmhd.initial_state(disc)
    out["state0"] = st0.vec.data.copy()
    out["ic_u"], out["ic_a"] = st0.ic_u, st0.ic_a
    out["r0"] = residual(st0, disc).data
    st = st0.copy()
    st.vec.data += 1e-3 * rng.standard_normal(st.vec.data.size)
    out["state"] = st.vec.data.copy()
    out["r"] = residual(st, disc).data
    jac = assemble_jacobian(st, disc)
    prec = SpaceTimePreconditioner(jac, disc, st)
    v = rng.standard_normal(jac.size)
    out["v"] = v
    out["Jv"] = jac.apply(v)
    out["Pv"] = prec.apply_inverse(v)
    out["PFv"] = prec.apply_forward(v)
    out["alfven"] = prec.alfven
    if blocks:
        for k, b in enumerate(jac.slabs):
            for name in ("f_u", "z_j", "z_a", "y", "f_a"):
                csr_dump(f"s{k}_{name}", getattr(b, name), out)
            csr_dump(f"s{k}_f_p", prec.f_p[k], out)
            csr_dump(f"s{k}_c_a", prec.c_a[k], out)
        for k, m in enumerate(prec.c_a_sub1):
            csr_dump(f"sub1_{k}", m, out)
        csr_dump("sub2", prec.c_a_sub2, out)
        for name in ("div_bc", "div_t_bc", "mixed_ja_bc", "mass_u_dt_bc", "mass_a_dt_bc",
                     "mass_a_bc", "mass_j", "mass_p", "stiff_p_pinned", "stiff_a_bc0",
                     "mass_u", "stiff_u"):
            csr_dump(name, getattr(disc, name), out)
        nt = jac.n_steps
        n_u, n_p, n_a = disc.layout.n_u, disc.layout.n_p, disc.layout.n_a
        out["sv_u"] = prec.solve_velocity(v[: nt * n_u].copy())
        out["sw_a"] = prec.solve_wave(v[: nt * n_a].copy())
        out["psi_p"] = prec.pressure_schur_inverse(v[: nt * n_p].copy())
        out["msi_a"] = prec.magnetic_schur_inverse(v[: nt * n_a].copy())
    for name in ("u_bc_idx", "u_bc_vals", "a_bc_idx", "a_bc_vals", "p_mean_row", "e_load",
                 "current_flux"):
        out[name] = np.asarray(getattr(disc, name))
    out["p_mean_target"] = disc.p_mean_target
    out["p_mean_mass"] = disc.p_mean_mass
    out["layout"] = np.array([disc.layout.n_u, disc.layout.n_p, disc.layout.n_j, disc.layout.n_a,
                              jac.n_steps])
    if solve:
        cfg = gmres_cfg or stmhd.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000,
                                             restart=50)
        jac0 = assemble_jacobian(st0, disc)
        prec0 = SpaceTimePreconditioner(jac0, disc, st0)
        t0 = time.perf_counter()
        res = stmhd.gmres(jac0.apply, prec0.apply_inverse, -out["r0"], config=cfg)
        out["gmres_time"] = time.perf_counter() - t0
        out["gmres_iters"] = res.iterations
        out["gmres_residuals"] = np.array(res.residuals)
        out["gmres_x"] = res.x
        out["gmres_true"] = res.true_residual
        st1 = st0.copy()
        st1.vec.data += res.x
        out["r1"] = residual(st1, disc).data


def c5_case(out, n=8, nt=4, seed=0):
    """Configuration 5 scalar operator built from reference fem
    functions: F_k = M/dt + 1e-3 K + W(u_k), Dirichlet rows top/bottom."""
    dt, eps = 1e-2, 1e-3
    mesh = stmhd.build_rect_mesh(-1.0, 1.0, -1.0, 1.0, 2.0 / n)
    p1 = fem.FESpace(mesh, 1)
    v1 = fem.FESpace(mesh, 1, components=2)
    bc = np.unique(np.concatenate([p1.boundary_nodes[Side.TOP], p1.boundary_nodes[Side.BOTTOM]]))
    m, k = fem.assemble_mass(p1), fem.assemble_stiffness(p1)
    ufields = c5_velocity_fields(p1.node_coords, nt, seed)
    out["ufields"] = ufields
    out["bc"] = bc
    rng = np.random.default_rng(1)
    x = rng.standard_normal((nt, p1.dof_count))
    out["x"] = x
    coup = fem.bc_zero((m / dt).tocsr(), rows=bc, cols=bc)
    fs, lus = [], []
    for kk in range(nt):
        u = np.concatenate([ufields[kk, :, 0], ufields[kk, :, 1]])
        _, lin_a, _ = fem.assemble_advection_A(p1, v1, u, np.zeros(p1.dof_count))
        f = fem.bc_identity((m / dt + eps * k + lin_a).tocsr(), bc)
        fs.append(f)
        csr_dump(f"F{kk}", f, out)
        lus.append(stmhd.LUFactor(f))
    csr_dump("coupling", coup, out)
    y = np.stack([fs[kk] @ x[kk] - (coup @ x[kk - 1] if kk else 0.0) for kk in range(nt)])
    out["Fx"] = y
    s = np.empty_like(x)
    for kk in range(nt):
        s[kk] = lus[kk].solve(x[kk] + (coup @ s[kk - 1] if kk else 0.0))
    out["Finv_x"] = s


def main():
    cases = {}
    prob = stmhd.by_name("island_coalescence")
    cases["ref_island"] = (stmhd.discretize(prob, 0.5, 0.5, 1.0), 5)
    prob = stmhd.by_name("tearing_mode")
    cases["ref_tearing"] = (stmhd.discretize(prob, 0.25, 0.5, 1.0), 6)
    cases["bl_island4"] = (baseline_disc("island", 1e-2, 4, 0.1, 3), 7)
    cases["bl_tearing4"] = (baseline_disc("tearing", 1e-3, 4, 0.02, 2), 8)
    for name, (disc, seed) in cases.items():
        out = {}
        full_case(disc, seed, out)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, "gmres", out["gmres_iters"], "slab", disc.layout.slab_size)
    # config 1 at full size: vectors only
    disc = baseline_disc("island", 1e-2, 16, 0.1, 8)
    out = {}
    full_case(disc, 0, out, blocks=False)
    out.pop("PFv")
    np.savez_compressed(os.path.join(HERE, "bl_c1.npz"), **out)
    print("bl_c1 gmres", out["gmres_iters"], "r0", np.linalg.norm(out["r0"]),
          "r1/r0", np.linalg.norm(out["r1"]) / np.linalg.norm(out["r0"]))
    out = {}
    c5_case(out)
    np.savez_compressed(os.path.join(HERE, "c5_tiny.npz"), **out)
    print("c5 ok")


if __name__ == "__main__":
    main()
