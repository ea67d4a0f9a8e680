"""GPU parity of the drop-in operators against the reference's golden vectors
and the CPU oracle.

Tolerances (north star): assembled values and matvecs per entry
|gpu - ref| <= 1e-12 * max(|ref|, floor) with floor = max |row| (cancelling
entries) for matrices and the |J||v| rounding scale for matvecs; P_T^{-1} r
relative L2 <= 1e-10; FGMRES iteration count within +-1; solution relative
L2 <= 1e-8.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import csr_from

pytestmark = pytest.mark.gpu

TOL_ENTRY = 1e-12


@pytest.fixture(scope="module")
def p():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as pkg

    return pkg


def _disc(p, name):
    if name == "ref_island":
        return p.discretize(p.by_name("island_coalescence"), 0.5, 0.5, 1.0)
    if name == "ref_tearing":
        return p.discretize(p.by_name("tearing_mode"), 0.25, 0.5, 1.0)
    if name == "bl_island4":
        return p.discretize(p.baseline_island(1e-2), 0.5, 0.1, 0.3)
    if name == "bl_tearing4":
        return p.discretize(p.baseline_tearing(1e-3), 0.5, 0.02, 0.04)
    if name == "bl_c1":
        return p.discretize_config("C1")
    raise KeyError(name)


def _oracle_disc(name):
    from oracle import configs, model

    if name == "ref_island":
        return model.make_disc_dx(configs.reference_problem("island_coalescence"), 0.5, 0.5, 1.0)
    if name == "ref_tearing":
        return model.make_disc_dx(configs.reference_problem("tearing_mode"), 0.25, 0.5, 1.0)
    if name == "bl_island4":
        return model.make_disc(configs.baseline_problem("island", 1e-2), 4, 0.1, 3)
    if name == "bl_tearing4":
        return model.make_disc(configs.baseline_problem("tearing", 1e-3), 4, 0.02, 2)
    if name == "bl_c1":
        return model.make_disc(configs.baseline_problem("island", 1e-2), 16, 0.1, 8)


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def entry_ok(mine, ref, scale):
    """Per-entry check |mine-ref| <= TOL*max(|ref|, scale); returns worst ratio."""
    err = np.abs(mine - ref)
    den = np.maximum(np.abs(ref), scale)
    den = np.where(den == 0, 1e-300, den)
    return float(np.max(err / den)) if err.size else 0.0


def matrix_ok(mine: sp.csr_matrix, ref: sp.csr_matrix):
    """Union-pattern per-entry check with a 1e-12*max|row| floor."""
    diff = (sp.csr_matrix(mine) - sp.csr_matrix(ref)).tocsr()
    rowmax = np.asarray(abs(ref).max(axis=1).todense()).ravel()
    rowmax = np.maximum(rowmax, np.asarray(abs(mine).max(axis=1).todense()).ravel())
    worst = 0.0
    diff = diff.tocoo()
    refd = sp.csr_matrix(ref)
    for r, c, v in zip(diff.row, diff.col, diff.data):
        den = max(abs(refd[r, c]), rowmax[r])
        if den > 0:
            worst = max(worst, abs(v) / den)
    return worst


CASES = ["ref_island", "ref_tearing", "bl_island4", "bl_tearing4"]


@pytest.fixture(scope="module", params=CASES)
def case(request, p, golden):
    import torch

    g = golden(request.param)
    d = _disc(p, request.param)
    st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["state"]),
                          torch.as_tensor(g["ic_u"], device="cuda"), torch.as_tensor(g["ic_a"], device="cuda"))
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    return request.param, g, d, st, jac, pc


def test_disc_data(case):
    _, g, d, *_ = case
    np.testing.assert_array_equal(d.u_bc_idx, g["u_bc_idx"])
    np.testing.assert_array_equal(d.a_bc_idx, g["a_bc_idx"])
    assert np.max(np.abs(d.a_bc_vals - g["a_bc_vals"])) < 1e-15
    for name, mine in (("p_mean_row", d.p_mean_row), ("e_load", d.e_load), ("current_flux", d.current_flux)):
        assert np.max(np.abs(mine - g[name])) <= 1e-14 * max(1.0, np.max(np.abs(g[name]))), name


def test_initial_state(case, p):
    _, g, d, *_ = case
    st0 = p.initial_state(d)
    assert np.max(np.abs(st0.vec.data.cpu().numpy() - g["state0"])) < 1e-13 * np.max(np.abs(g["state0"]))
    assert np.max(np.abs(st0.ic_a.cpu().numpy() - g["ic_a"])) < 1e-15


def test_residual(case, p):
    name, g, d, st, *_ = case
    import torch

    for key, vec in (("r0", g["state0"]), ("r", g["state"])):
        s = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, vec), torch.as_tensor(g["ic_u"], device="cuda"),
                             torch.as_tensor(g["ic_a"], device="cuda"))
        mine = p.residual(s, d).data.cpu().numpy()
        ref = g[key]
        # per entry <= 1e-12 of the rounding scale of the entry's terms: |J||x| bounds the
        # state-dependent element terms (linear and quadratic), |r(0)| the constant ones
        # (loads, fluxes, BC values, initial condition), |r| the result itself
        from oracle import model

        od = _oracle_disc(name)
        ojac = model.jacobian(model.State(np.asarray(vec).copy(), g["ic_u"], g["ic_a"]), od)
        z = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, np.zeros_like(vec)),
                             torch.as_tensor(g["ic_u"], device="cuda"), torch.as_tensor(g["ic_a"], device="cuda"))
        const = np.abs(p.residual(z, d).data.cpu().numpy())
        scale = ojac.abs_apply(np.asarray(vec)) + const + np.abs(ref)
        w = np.abs(mine - ref) / np.maximum(scale, 1e-300)
        assert float(w.max()) <= TOL_ENTRY, (name, key, float(w.max()))


def test_jacobian_blocks(case):
    name, g, d, st, jac, pc = case
    for k, b in enumerate(jac.slabs):
        for blk in ("f_u", "z_j", "z_a", "y", "f_a"):
            w = matrix_ok(getattr(b, blk), csr_from(g, f"s{k}_{blk}"))
            assert w <= TOL_ENTRY, (name, k, blk, w)
        assert matrix_ok(pc.f_p[k], csr_from(g, f"s{k}_f_p")) <= TOL_ENTRY
        assert matrix_ok(pc.c_a[k], csr_from(g, f"s{k}_c_a")) <= TOL_ENTRY
    for k, m in enumerate(pc.c_a_sub1):
        assert matrix_ok(m, csr_from(g, f"sub1_{k}")) <= TOL_ENTRY
    np.testing.assert_allclose(pc.alfven, g["alfven"], rtol=1e-12, atol=1e-15)


def test_jacobian_apply(case):
    name, g, d, st, jac, pc = case
    from oracle import model

    od = _oracle_disc(name)
    ost = model.State(g["state"].copy(), g["ic_u"], g["ic_a"])
    scale = model.jacobian(ost, od).abs_apply(g["v"])
    mine = jac.apply(g["v"]).cpu().numpy()
    assert entry_ok(mine, g["Jv"], scale) <= TOL_ENTRY


def test_preconditioner_apply(case):
    name, g, d, st, jac, pc = case
    v = g["v"]
    nt, L = d.n_steps, d.layout
    assert relerr(pc.apply_inverse(v).cpu().numpy(), g["Pv"]) < 1e-10
    assert relerr(pc.apply_forward(v).cpu().numpy(), g["PFv"]) < 1e-10
    assert relerr(pc.solve_velocity(v[: nt * L.n_u]).cpu().numpy(), g["sv_u"]) < 1e-10
    assert relerr(pc.solve_wave(v[: nt * L.n_a]).cpu().numpy(), g["sw_a"]) < 1e-10
    assert relerr(pc.pressure_schur_inverse(v[: nt * L.n_p]).cpu().numpy(), g["psi_p"]) < 1e-10
    assert relerr(pc.magnetic_schur_inverse(v[: nt * L.n_a]).cpu().numpy(), g["msi_a"]) < 1e-10


def test_gmres_newton_step(case, p):
    name, g, d, *_ = case
    st0 = p.initial_state(d)
    jac = p.assemble_jacobian(st0, d)
    pc = p.SpaceTimePreconditioner(jac, d, st0)
    r0 = p.residual(st0, d).data
    cfg = p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50)
    res = p.gmres(jac.apply, pc.apply_inverse, -r0, config=cfg)
    assert abs(res.iterations - int(g["gmres_iters"])) <= 1, (name, res.iterations, int(g["gmres_iters"]))
    assert relerr(res.x.cpu().numpy(), g["gmres_x"]) < 1e-8


def test_config1(p, golden):
    """BASELINE config 1 (16x16, Nt=8): r0, J.v, P^-1 v and one Newton step
    with 92 +- 1 FGMRES iterations."""
    import torch

    g = golden("bl_c1")
    d = _disc(p, "bl_c1")
    st0 = p.initial_state(d)
    assert np.max(np.abs(st0.vec.data.cpu().numpy() - g["state0"])) < 1e-13 * np.max(np.abs(g["state0"]))
    r0 = p.residual(st0, d).data.cpu().numpy()
    assert abs(np.linalg.norm(r0) - np.linalg.norm(g["r0"])) < 1e-12 * np.linalg.norm(g["r0"])
    st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["state"]), torch.as_tensor(g["ic_u"], device="cuda"),
                          torch.as_tensor(g["ic_a"], device="cuda"))
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    assert relerr(jac.apply(g["v"]).cpu().numpy(), g["Jv"]) < 1e-13
    assert relerr(pc.apply_inverse(g["v"]).cpu().numpy(), g["Pv"]) < 1e-10
    cfg = p.NewtonConfig(abs_tol=1e-300, max_iters=1,
                         gmres=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=100000, restart=50))
    state, stats = p.solve_all_at_once(d, cfg)
    assert stats.newton_iters == 1
    assert abs(stats.gmres_iters[0] - 92) <= 1, stats.gmres_iters
    x = state.vec.data.cpu().numpy() - g["state0"]
    assert relerr(x, g["gmres_x"]) < 1e-8
    assert abs(stats.residual_norms[1] / stats.residual_norms[0] - 1.0303688174095965e-2) < 1e-6


def test_pipelined_apply_deterministic_and_matches_sequential(p, golden):
    """The TRIANGULAR P_T^{-1} runs its three sweeps in one pipelined launch (per-slab
    release/acquire flags between clusters).  Repeated applications must be bitwise
    identical (no race in the handshake), and equal the sequential composition of the
    individual operators to rounding: x_A = S_A^{-1} r_A, x_p = S_p^{-1} r_p, and the
    velocity block checked through the forward operator, P (P^{-1} v) = v."""
    import torch

    g = golden("bl_c1")
    d = _disc(p, "bl_c1")
    st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["state"]), torch.as_tensor(g["ic_u"], device="cuda"),
                          torch.as_tensor(g["ic_a"], device="cuda"))
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    v = torch.as_tensor(g["v"], device="cuda")
    outs = [pc.apply_inverse(v).clone() for _ in range(6)]
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    L, nt = d.layout, d.n_steps
    o = outs[0].view(nt, -1)
    vv = v.view(nt, -1)
    o_p, o_j, o_a = L.n_u, L.n_u + L.n_p, L.n_u + L.n_p + L.n_j
    x_a = pc.magnetic_schur_inverse(vv[:, o_a:].reshape(-1)).view(nt, -1)
    assert relerr(o[:, o_a:].cpu().numpy(), x_a.cpu().numpy()) < 1e-12
    x_p = pc.pressure_schur_inverse(vv[:, o_p:o_j].reshape(-1)).view(nt, -1)
    assert relerr(o[:, o_p:o_j].cpu().numpy(), x_p.cpu().numpy()) < 1e-12
    assert relerr(pc.apply_forward(outs[0]).cpu().numpy(), g["v"]) < 1e-10


@pytest.mark.parametrize("case_name,prob,dx", [("variants_island", "island_coalescence", 0.5),
                                                ("variants_tearing", "tearing_mode", 0.25)])
@pytest.mark.parametrize("variant", ["triangular", "simplified", "full"])
def test_variants_match_reference_and_round_trip(p, golden, case_name, prob, dx, variant):
    """All three P_T variants, inverse and forward application, against the
    reference (golden vectors) and the round trips of reference
    tests/test_precond.py:187-196."""
    import torch

    g = golden(case_name)
    d = p.discretize(p.by_name(prob), dx, 0.5, 1.0)
    st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["state"]), torch.as_tensor(g["ic_u"], device="cuda"),
                          torch.as_tensor(g["ic_a"], device="cuda"))
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st, variant)
    x = g["x"]
    assert relerr(pc.apply_inverse(x).cpu().numpy(), g[f"inv_{variant}"]) < 1e-10
    assert relerr(pc.apply_forward(x).cpu().numpy(), g[f"fwd_{variant}"]) < 1e-10
    rng = np.random.default_rng(5)
    for _ in range(3):
        y = rng.standard_normal(jac.size)
        assert relerr(pc.apply_inverse(pc.apply_forward(y)).cpu().numpy(), y) <= 1e-9
        assert relerr(pc.apply_forward(pc.apply_inverse(y)).cpu().numpy(), y) <= 1e-9
