"""Reference-shaped problem intake: a ProblemSpec carrying its own ``bcs: BCSpec``
and ``a_eq_normal_flux_top`` (reference problems.py:25-63, fem.py:478-568) goes
through ``discretize`` unchanged.

CPU: the boundary data (constrained DOFs and values, the current-equation flux)
of a custom problem -- lid-driven Dirichlet velocity on the top, Dirichlet
potential on the top and left -- equals the reference's (``tests/golden/ref_bcs.npz``,
``make_golden_bcs.py``); the reference's own ProblemSpec object is accepted when
the reference is importable (build container); BCSpec validation errors.
GPU: residual, J.v, P_T^-1 v and the first FGMRES solve of that problem against the
reference's vectors.
"""

import os
import sys

import numpy as np
import pytest


def lid_problem(p):
    """The make_golden_bcs.py problem written with this package's mirror classes."""
    ref = p.by_name("island_coalescence", mu=0.1, eta=0.1)
    lid = (lambda x, y: 0.05 * np.sin(np.pi * x) + 0.0 * y, lambda x, y: 0.0 * x)
    S = p.Side
    bcs = p.BCSpec(conditions={
        "u": {S.LEFT: p.slip(), S.RIGHT: p.slip(), S.BOTTOM: p.slip(), S.TOP: p.dirichlet(lid)},
        "p": {s: p.natural() for s in S},
        "j": {s: p.natural() for s in S},
        "A": {S.LEFT: p.dirichlet(ref.a_eq), S.RIGHT: p.natural(), S.BOTTOM: p.natural(),
              S.TOP: p.dirichlet(ref.a_eq)},
    })
    return p.ProblemSpec(name="island_lid", domain=ref.domain, mu=ref.mu, eta=ref.eta, mu0=ref.mu0,
                         eps=ref.eps, a_eq=ref.a_eq, e_eq=ref.e_eq, p_eq=ref.p_eq,
                         a_perturbation=ref.a_perturbation,
                         a_eq_normal_flux_top=ref.a_eq_normal_flux_top, bcs=bcs)


def host_boundary_data(problem):
    from paper_2309_00768_b200 import fem, problems

    m = fem.Mesh(*problem.domain, 4, 4)
    vel, p1 = fem.Space(m, 3, 2), fem.Space(m, 1)
    ui, uv = problems.constrained_dofs(vel, problem, "u")
    ai, av = problems.constrained_dofs(p1, problem, "A")
    flux = np.zeros(p1.ndof)
    for side, f in problems.flux_terms(problem).items():
        flux += fem.edge_load_vector(p1, side, f)
    return ui, uv, ai, av, flux / problem.mu0


def test_custom_bcspec_boundary_data_matches_reference(golden):
    import paper_2309_00768_b200 as p

    g = golden("ref_bcs")
    ui, uv, ai, av, flux = host_boundary_data(lid_problem(p))
    np.testing.assert_array_equal(ui, g["u_bc_idx"])
    np.testing.assert_allclose(uv, g["u_bc_vals"], rtol=0, atol=1e-15)
    assert np.max(np.abs(uv)) > 0.01  # the lid values are really there
    np.testing.assert_array_equal(ai, g["a_bc_idx"])
    np.testing.assert_allclose(av, g["a_bc_vals"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(flux, g["current_flux"], rtol=1e-13, atol=1e-15)


def test_builtins_are_reference_shaped():
    """The built-in records carry a BCSpec and the top flux, like the reference's,
    and resolve to the same boundary data as the legacy adapter fields."""
    import paper_2309_00768_b200 as p
    from paper_2309_00768_b200 import fem, problems

    for prob in (p.by_name("island_coalescence"), p.by_name("tearing_mode"), p.baseline_island(),
                 p.baseline_tearing()):
        assert isinstance(prob.bcs, p.BCSpec) and callable(prob.a_eq_normal_flux_top)
        m = fem.Mesh(*prob.domain, 4, 4)
        vel, p1 = fem.Space(m, prob.vel_degree, 2), fem.Space(m, 1)
        ui, uv = problems.constrained_dofs(vel, prob, "u")
        np.testing.assert_array_equal(ui, fem.slip_dofs(vel))
        assert not np.any(uv)
        ai, av = problems.constrained_dofs(p1, prob, "A")
        li, lv = fem.dirichlet_dofs(p1, prob.a_dirichlet, prob.a_eq)
        np.testing.assert_array_equal(ai, li)
        np.testing.assert_array_equal(av, lv)


def test_bcspec_validation_errors():
    import paper_2309_00768_b200 as p

    full = {s: p.natural() for s in p.Side}
    with pytest.raises(p.ConfigurationError, match="unknown field"):
        p.BCSpec(conditions={}).for_field("q")
    with pytest.raises(p.ConfigurationError, match="no boundary conditions given for field 'A'"):
        p.BCSpec(conditions={"u": full}).for_field("A")
    part = dict(full)
    del part[p.Side.TOP]
    with pytest.raises(p.ConfigurationError, match="missing condition on top"):
        p.BCSpec(conditions={"A": part}).for_field("A")
    with pytest.raises(p.ConfigurationError, match="unknown boundary tag"):
        p.BCSpec(conditions={"A": {**full, "diag": p.natural()}}).for_field("A")


def test_reference_problem_object_accepted(golden):
    """The reference's own ProblemSpec (its Side/BCKind enums) resolves to the same
    boundary data (build container only: /root/reference is not on the GPU box)."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference package not present")
    sys.path.insert(0, src)
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    try:
        from make_golden_bcs import lid_problem as ref_lid_problem
    finally:
        sys.path.remove(src)
    g = golden("ref_bcs")
    ui, uv, ai, av, flux = host_boundary_data(ref_lid_problem())
    np.testing.assert_array_equal(ui, g["u_bc_idx"])
    np.testing.assert_allclose(uv, g["u_bc_vals"], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(ai, g["a_bc_idx"])
    np.testing.assert_allclose(flux, g["current_flux"], rtol=1e-13, atol=1e-15)


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.gpu
def test_custom_bcspec_on_device_matches_reference(golden):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p

    g = golden("ref_bcs")
    d = p.discretize(lid_problem(p), 0.25, 0.5, 1.0)
    np.testing.assert_array_equal(d.u_bc_idx, g["u_bc_idx"])
    st0 = p.initial_state(d)
    np.testing.assert_allclose(st0.vec.data.cpu().numpy(), g["state0"], rtol=0, atol=1e-12)
    st = p.SpaceTimeState(p.BlockVector(d.layout, d.n_steps, g["x"]),
                          torch.as_tensor(g["ic_u"], device="cuda"), torch.as_tensor(g["ic_a"], device="cuda"))
    r = p.residual(st, d).data.cpu().numpy()
    assert np.max(np.abs(r - g["r"])) <= 1e-12 * max(1.0, np.max(np.abs(g["r"])))
    jac = p.assemble_jacobian(st, d)
    pc = p.SpaceTimePreconditioner(jac, d, st)
    assert relerr(jac.apply(g["v"]).cpu().numpy(), g["Jv"]) < 1e-13
    assert relerr(pc.apply_inverse(g["v"]).cpu().numpy(), g["Pv"]) < 1e-10
    # first Newton step's FGMRES solve from the initial state
    r0 = p.residual(st0, d).data
    assert relerr(r0.cpu().numpy(), g["r0"]) < 1e-12
    j0 = p.assemble_jacobian(st0, d)
    pc0 = p.SpaceTimePreconditioner(j0, d, st0)
    res = p.gmres(j0.apply, pc0.apply_inverse, -r0,
                  config=p.GmresConfig(rel_tol=1e-8, abs_tol=1e-300, max_iters=1000, restart=50))
    assert abs(res.iterations - int(g["gmres_iters"])) <= 1, (res.iterations, int(g["gmres_iters"]))
    assert relerr(res.x.cpu().numpy(), g["gmres_x"]) <= 1e-8
