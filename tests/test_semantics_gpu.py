"""Reference test semantics on the device path (through the C-ABI kernels):
FGMRES contract (reference tests/test_linalg.py:78-149 -> linalg.py:122-209),
Jacobian against central differences, linearity and causality
(tests/test_spacetime.py:79-93,129-145 -> spacetime.py:131-153) and bitwise
reproducible solves (tests/test_solver.py:42-47).  The operators here are the
device drop-ins; dense test matrices are applied with torch on the GPU, the
Krylov arithmetic (CGS2 dots/updates/normalisation/combination) is ours."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(7)


@pytest.fixture(scope="module")
def p():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p

    return p


def _mat(a):
    import torch

    t = torch.as_tensor(a, dtype=torch.float64, device="cuda")
    return lambda v: t @ v


def _np(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def test_gmres_identity_converges_immediately(p):
    b = RNG.standard_normal(30)
    res = p.gmres(lambda v: v, None, b, config=p.GmresConfig(rel_tol=1e-12))
    assert res.converged and res.iterations <= 1
    assert res.true_residual <= 1e-12 * np.linalg.norm(b)


def test_gmres_finite_termination(p):
    n = 12
    a = RNG.standard_normal((n, n)) + n * np.eye(n)
    b = RNG.standard_normal(n)
    res = p.gmres(_mat(a), None, b, config=p.GmresConfig(rel_tol=1e-14, abs_tol=1e-30, max_iters=n))
    assert res.converged and res.iterations <= n
    assert np.linalg.norm(a @ _np(res.x) - b) <= 1e-10 * np.linalg.norm(b)


def test_gmres_exact_preconditioner_one_iteration(p):
    n = 25
    a = RNG.standard_normal((n, n)) + n * np.eye(n)
    b = RNG.standard_normal(n)
    res = p.gmres(_mat(a), _mat(np.linalg.inv(a)), b, config=p.GmresConfig(rel_tol=1e-10))
    assert res.converged and res.iterations == 1


def test_gmres_monotone_history_and_true_residual(p):
    n = 40
    a = RNG.standard_normal((n, n)) + 8 * np.eye(n)
    b = RNG.standard_normal(n)
    cfg = p.GmresConfig(rel_tol=1e-8, abs_tol=1e-30, max_iters=100)
    res = p.gmres(_mat(a), None, b, config=cfg)
    hist = res.residuals
    assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1))
    assert res.true_residual <= max(cfg.rel_tol * hist[0], cfg.abs_tol) * (1 + 1e-6)


def test_gmres_restarted_still_converges(p):
    n = 40
    a = RNG.standard_normal((n, n)) + 10 * np.eye(n)
    b = RNG.standard_normal(n)
    res = p.gmres(_mat(a), None, b, config=p.GmresConfig(rel_tol=1e-8, max_iters=200, restart=7))
    assert res.converged
    assert np.linalg.norm(a @ _np(res.x) - b) <= 1e-7 * np.linalg.norm(b)


def test_gmres_zero_rhs(p):
    res = p.gmres(lambda v: 2 * v, None, np.zeros(5))
    assert res.converged and res.iterations == 0 and np.all(_np(res.x) == 0)


def test_gmres_max_iters_nonconvergence(p):
    n = 30
    a = RNG.standard_normal((n, n)) + 6 * np.eye(n)
    b = RNG.standard_normal(n)
    res = p.gmres(_mat(a), None, b, config=p.GmresConfig(rel_tol=1e-13, abs_tol=1e-30, max_iters=3))
    assert not res.converged and res.iterations == 3
    assert np.all(np.isfinite(_np(res.x)))


def test_gmres_breakdown_on_nonfinite(p):
    with pytest.raises(p.BreakdownError):
        p.gmres(lambda v: v * float("nan"), None, np.ones(4))


def test_gmres_config_validation(p):
    with pytest.raises(ValueError):
        p.GmresConfig(rel_tol=0.0)
    with pytest.raises(ValueError):
        p.GmresConfig(max_iters=0)


@pytest.mark.parametrize("problem", ["tearing_mode", "island_coalescence"])
def test_jacobian_matches_central_differences(p, problem):
    prob = p.by_name(problem)
    dx = 0.5 if problem == "island_coalescence" else 0.25
    disc = p.discretize(prob, dx, 0.5, 1.0)
    state = p.initial_state(disc)
    jac = p.assemble_jacobian(state, disc)
    v = RNG.standard_normal(jac.size)
    eps = 1e-6
    plus, minus = state.copy(), state.copy()
    import torch

    vt = torch.as_tensor(v, dtype=torch.float64, device="cuda")
    plus.vec.data += eps * vt
    minus.vec.data -= eps * vt
    fd = (_np(p.residual(plus, disc).data) - _np(p.residual(minus, disc).data)) / (2 * eps)
    jv = _np(jac.apply(v))
    assert np.linalg.norm(fd - jv) <= 1e-6 * np.linalg.norm(jv)


@pytest.fixture(scope="module")
def small(p):
    disc = p.discretize(p.by_name("island_coalescence"), 0.5, 0.5, 1.0)
    state = p.initial_state(disc)
    return disc, state, p.assemble_jacobian(state, disc)


def test_apply_linearity_and_zero(p, small):
    _, _, jac = small
    assert np.all(_np(jac.apply(np.zeros(jac.size))) == 0.0)
    v, w = RNG.standard_normal((2, jac.size))
    a, b = 0.37, -1.21
    lhs = _np(jac.apply(a * v + b * w))
    rhs = a * _np(jac.apply(v)) + b * _np(jac.apply(w))
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_apply_causality(p, small):
    disc, _, jac = small
    s = disc.layout.slab_size
    v = np.zeros(jac.size)
    v[s:] = RNG.standard_normal(s * (jac.n_steps - 1))
    assert np.all(_np(jac.apply(v))[:s] == 0.0)


def test_preconditioner_causality(p, small):
    """P_T^{-1} is block lower triangular in time: slab-0 output depends on slab 0 only."""
    disc, state, jac = small
    pc = p.SpaceTimePreconditioner(jac, disc, state)
    s = disc.layout.slab_size
    v = np.zeros(jac.size)
    v[s:] = RNG.standard_normal(s * (jac.n_steps - 1))
    assert np.all(_np(pc.apply_inverse(v))[:s] == 0.0)


def test_solve_bitwise_reproducible(p):
    disc = p.discretize(p.by_name("island_coalescence"), 0.5, 0.25, 0.5)
    s1, st1 = p.solve_all_at_once(disc)
    s2, st2 = p.solve_all_at_once(disc)
    assert st1.newton_iters == st2.newton_iters
    assert st1.gmres_iters == st2.gmres_iters
    assert np.array_equal(_np(s1.vec.data), _np(s2.vec.data))


# -- preconditioner pieces (reference tests/test_precond.py:39-48,139-154) ------------


def test_alfven_scaling_tearing_equilibrium_analytic_device(p):
    """The device Alfven kernel (assembly pass) on the Harris sheet: the mean field is
    exactly (2/5) log cosh(5/2) in every slab (reference precond.py:46-57,89-90)."""
    import torch

    prob = p.by_name("tearing_mode")
    disc = p.discretize(prob, 0.25, 0.5, 1.0)
    state = p.initial_state(disc)
    a = torch.as_tensor(disc.pot.interp(prob.a_eq), dtype=torch.float64, device="cuda")
    state.vec.fields("A")[:] = a
    jac = p.assemble_jacobian(state, disc)
    s = p.SpaceTimePreconditioner(jac, disc, state).alfven
    b_norm = 0.4 * np.log(np.cosh(2.5))
    assert np.all(np.abs(np.sqrt(s * prob.mu0) - b_norm) < 1e-8)
    assert np.all(np.abs(s - b_norm**2 / prob.mu0) < 1e-10)


@pytest.fixture(scope="module")
def small_pc(p, small):
    disc, state, jac = small
    return disc, p.SpaceTimePreconditioner(jac, disc, state)


@pytest.mark.parametrize("pair,field,tol", [
    (("pressure_schur_inverse", "pressure_schur_apply"), "n_p", 1e-10),
    (("magnetic_schur_inverse", "magnetic_schur_apply"), "n_a", 1e-9),
    (("solve_velocity", "apply_velocity"), "n_u", 1e-10),
    (("solve_wave", "apply_wave"), "n_a", 1e-10),
])
def test_sub_operator_round_trips(p, small_pc, pair, field, tol):
    disc, pc = small_pc
    inv, fwd = getattr(pc, pair[0]), getattr(pc, pair[1])
    n = getattr(disc.layout, field) * pc.n_steps
    for _ in range(3):
        x = RNG.standard_normal(n)
        y = _np(inv(fwd(x)))
        assert np.linalg.norm(y - x) <= tol * np.linalg.norm(x)


def test_singular_velocity_block_raises_preconditioner_error(p, small):
    """A zero-pivot F_u factorisation surfaces as PreconditionerError('F_u')
    (reference precond.py:108-113; status STMHD_SINGULAR through the C-ABI)."""
    disc, state, _ = small
    jac = p.assemble_jacobian(state, disc)
    jac.values.zero_()
    with pytest.raises(p.PreconditionerError) as err:
        p.SpaceTimePreconditioner(jac, disc, state)
    assert err.value.block == "F_u"
