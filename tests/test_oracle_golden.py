"""Pin the CPU oracle (``oracle/``) to golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py``).  CPU only."""

import numpy as np
import pytest

import oracle
from oracle import configs, model, solvers
from conftest import csr_from

CASES = {
    "ref_island": lambda: model.make_disc_dx(configs.reference_problem("island_coalescence"),
                                             0.5, 0.5, 1.0),
    "ref_tearing": lambda: model.make_disc_dx(configs.reference_problem("tearing_mode"),
                                              0.25, 0.5, 1.0),
    "bl_island4": lambda: model.make_disc(configs.baseline_problem("island", 1e-2), 4, 0.1, 3),
    "bl_tearing4": lambda: model.make_disc(configs.baseline_problem("tearing", 1e-3), 4, 0.02, 2),
}


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=list(CASES))
def case(request, golden):
    g = golden(request.param)
    d = CASES[request.param]()
    st = model.State(g["state"].copy(), g["ic_u"].copy(), g["ic_a"].copy())
    jac = model.jacobian(st, d)
    pc = solvers.Precond(jac, d, st)
    return request.param, g, d, st, jac, pc


def test_discretisation_data(case):
    _, g, d, *_ = case
    assert list(g["layout"][:4]) == [d.n_u, d.n_p, d.n_j, d.n_a]
    np.testing.assert_array_equal(g["u_bc_idx"], d.u_bc)
    np.testing.assert_array_equal(g["a_bc_idx"], d.a_bc)
    np.testing.assert_allclose(d.a_bc_vals, g["a_bc_vals"], rtol=0, atol=1e-15)
    for name, mine in (("p_mean_row", d.p_mean_row), ("e_load", d.e_load),
                       ("current_flux", d.current_flux)):
        assert np.max(np.abs(mine - g[name])) <= 1e-14 * max(1.0, np.max(np.abs(g[name])))
    assert abs(d.p_mean_target - float(g["p_mean_target"])) < 1e-14


def test_initial_state_and_residuals(case):
    _, g, d, st, *_ = case
    st0 = model.initial_state(d)
    assert np.max(np.abs(st0.vec - g["state0"])) < 1e-13
    r0 = model.residual(model.State(g["state0"], g["ic_u"], g["ic_a"]), d)
    r = model.residual(st, d)
    for mine, ref in ((r0, g["r0"]), (r, g["r"])):
        assert np.max(np.abs(mine - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_jacobian_blocks(case):
    _, g, d, st, jac, pc = case
    for k, b in enumerate(jac.slabs):
        for name in ("f_u", "z_j", "z_a", "y", "f_a"):
            ref = csr_from(g, f"s{k}_{name}")
            diff = abs(getattr(b, name) - ref).max()
            assert diff <= 1e-12 * max(abs(ref).max(), 1e-300), (k, name, diff)
        for name, mine in (("f_p", pc.f_p[k]), ("c_a", pc.c_a[k])):
            ref = csr_from(g, f"s{k}_{name}")
            assert abs(mine - ref).max() <= 1e-12 * abs(ref).max(), (k, name)
    for k, m in enumerate(pc.c_a_sub1):
        ref = csr_from(g, f"sub1_{k}")
        assert abs(m - ref).max() <= 1e-12 * max(abs(ref).max(), 1e-300)
    np.testing.assert_allclose(pc.alfven, g["alfven"], rtol=1e-12, atol=1e-14)


def test_operators_and_preconditioner(case):
    _, g, d, st, jac, pc = case
    v = g["v"]
    assert relerr(jac.apply(v), g["Jv"]) < 1e-13
    assert relerr(pc.apply_inverse(v), g["Pv"]) < 1e-10
    assert relerr(pc.apply_forward(v), g["PFv"]) < 1e-10
    nt = jac.nt
    assert relerr(pc.solve_velocity(v[: nt * d.n_u].copy()), g["sv_u"]) < 1e-10
    assert relerr(pc.solve_wave(v[: nt * d.n_a].copy()), g["sw_a"]) < 1e-10
    assert relerr(pc.pressure_schur_inverse(v[: nt * d.n_p].copy()), g["psi_p"]) < 1e-10
    assert relerr(pc.magnetic_schur_inverse(v[: nt * d.n_a].copy()), g["msi_a"]) < 1e-10


def test_gmres_newton_step(case):
    _, g, d, *_ = case
    st0 = model.State(g["state0"].copy(), g["ic_u"], g["ic_a"])
    jac = model.jacobian(st0, d)
    pc = solvers.Precond(jac, d, st0)
    res = solvers.gmres_mgs(jac.apply, pc.apply_inverse, -g["r0"], rel_tol=1e-8, abs_tol=1e-300,
                            max_iters=100000, restart=50)
    assert res.iterations == int(g["gmres_iters"])
    assert relerr(res.x, g["gmres_x"]) < 1e-8


def test_config1_vectors(golden):
    """BASELINE config 1 at full size: r0, J.v, P^-1 v, 92 GMRES iterations."""
    g = golden("bl_c1")
    d = model.make_disc(configs.baseline_problem("island", 1e-2), 16, 0.1, 8)
    st0 = model.initial_state(d)
    assert np.max(np.abs(st0.vec - g["state0"])) < 1e-13
    r0 = model.residual(st0, d)
    assert abs(np.linalg.norm(r0) - 5.1396e-2) < 1e-5
    assert np.max(np.abs(r0 - g["r0"])) < 1e-13
    st = model.State(g["state"].copy(), g["ic_u"], g["ic_a"])
    jac = model.jacobian(st, d)
    pc = solvers.Precond(jac, d, st)
    assert relerr(jac.apply(g["v"]), g["Jv"]) < 1e-13
    assert relerr(pc.apply_inverse(g["v"]), g["Pv"]) < 1e-10
    assert int(g["gmres_iters"]) == 92


def test_config1_newton_step_iterations(golden):
    g = golden("bl_c1")
    d = model.make_disc(configs.baseline_problem("island", 1e-2), 16, 0.1, 8)
    st0 = model.initial_state(d)
    out = solvers.newton_solve(st0, d, one_step=True)
    assert out.gmres_iters == [92]
    assert relerr(st0.vec - g["state0"], g["gmres_x"]) < 1e-8


def test_c5_operator(golden):
    from oracle.c5 import C5
    from paper_2309_00768_b200.c5 import c5_velocity_fields

    g = golden("c5_tiny")
    op = C5(8, 4, g["ufields"])
    np.testing.assert_array_equal(op.bc, g["bc"])
    np.testing.assert_allclose(c5_velocity_fields(op.p1.coords, 4, 0), g["ufields"], rtol=0,
                               atol=1e-15)
    for k in range(4):
        ref = csr_from(g, f"F{k}")
        assert abs(op.F[k] - ref).max() <= 1e-12 * abs(ref).max()
    assert relerr(op.apply(g["x"]), g["Fx"]) < 1e-14
    assert relerr(op.solve(g["x"]), g["Finv_x"]) < 1e-12
