"""Sequential time stepping and the single-step preconditioner,
against golden values from the reference itself (tests/golden/make_golden_seq.py)
-- mirrors reference tests/test_solver.py and test_precond.py:210-226."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def p():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as pkg

    return pkg


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.gpu
def test_sequential_matches_reference(p, golden):
    g = golden("seq_tearing")
    disc = p.discretize(p.by_name("tearing_mode"), 0.25, 0.5, 1.0)
    seq_state, seq = p.solve_sequential(disc)
    assert seq.per_step_newton == g["seq_newton"].tolist()
    ptr = g["seq_gmres_ptr"]
    for k, its in enumerate(seq.per_step_gmres):
        ref = g["seq_gmres"][ptr[k]:ptr[k + 1]].tolist()
        assert len(its) == len(ref) and all(abs(a - b) <= 1 for a, b in zip(its, ref)), (k, its, ref)
    assert relerr(seq_state.vec.data.cpu().numpy(), g["seq_x"]) < 1e-8
    st_state, st = p.solve_all_at_once(disc)
    assert st.newton_iters == int(g["st_newton"])
    assert relerr(st_state.vec.data.cpu().numpy(), g["st_x"]) < 1e-8
    # solutions agree across drivers (reference test_solutions_agree_across_drivers)
    d = np.linalg.norm(st_state.vec.data.cpu().numpy() - seq_state.vec.data.cpu().numpy())
    assert d <= 1e-6 * np.linalg.norm(st_state.vec.data.cpu().numpy())
    nr, gr = p.compute_overhead_ratios(st, seq)
    assert abs(nr - g["ratios"][0]) < 1e-12 and abs(gr - g["ratios"][1]) < 0.15
    assert 0.95 <= nr <= 2.5 and 0.95 <= gr <= 3.0
    # the sequential solution meets the space-time tolerance
    assert p.residual(seq_state, disc).norm() <= 1e-10


@pytest.mark.gpu
def test_single_step_sequential_equals_all_at_once(p):
    """One slab: both drivers run the identical Newton iteration -> bitwise equal."""
    disc = p.discretize(p.by_name("island_coalescence"), 0.5, 1.0, 1.0)
    st_state, st = p.solve_all_at_once(disc)
    seq_state, seq = p.solve_sequential(disc)
    assert st.converged and seq.converged
    assert np.array_equal(st_state.vec.data.cpu().numpy(), seq_state.vec.data.cpu().numpy())
    assert st.newton_iters == seq.newton_iters and st.gmres_iters == seq.gmres_iters


@pytest.mark.gpu
def test_frozen_step_accounting_matches_reference(p, golden):
    g = golden("seq_frozen")
    disc = p.discretize(p.by_name("island_coalescence", eps=0.0), 0.5, 0.25, 1.0)
    _, seq = p.solve_sequential(disc)
    ref = g["seq_newton"].tolist()
    assert len(seq.per_step_newton) == len(ref)
    assert all(abs(a - b) <= 1 for a, b in zip(seq.per_step_newton, ref)), (seq.per_step_newton, ref)
    assert seq.frozen_steps == [k + 1 for k, n in enumerate(seq.per_step_newton) if n == 0]
    assert seq.effective_steps == disc.n_steps - len(seq.frozen_steps)


@pytest.mark.gpu
def test_sequential_nonconvergence_raises(p):
    disc = p.discretize(p.by_name("island_coalescence"), 0.5, 0.5, 1.0)
    with pytest.raises(p.ConvergenceError) as err:
        p.solve_sequential(disc, p.NewtonConfig(abs_tol=1e-13, max_iters=1))
    assert err.value.step == 1


@pytest.mark.gpu
def test_single_step_preconditioner(p, golden):
    import torch

    g = golden("seq_single")
    disc = p.discretize(p.by_name("island_coalescence"), 0.5, 0.5, 1.0)
    st = p.SpaceTimeState(p.BlockVector(disc.layout, disc.n_steps, g["state"]),
                          torch.as_tensor(g["ic_u"], device="cuda"), torch.as_tensor(g["ic_a"], device="cuda"))
    jac = p.assemble_jacobian(st, disc)
    pc = p.SpaceTimePreconditioner(jac, disc, st)
    for k in range(disc.n_steps):
        x = g[f"x{k}"]
        assert relerr(pc.apply_single_step_inverse(k, x).cpu().numpy(), g[f"inv{k}"]) < 1e-10
        assert relerr(pc.apply_single_step(k, x).cpu().numpy(), g[f"fwd{k}"]) < 1e-10
        rt = pc.apply_single_step_inverse(k, pc.apply_single_step(k, x)).cpu().numpy()
        assert relerr(rt, x) < 1e-9
    # the reference's single-step operator ignores the variant (precond.py:344-387 never
    # reads self.variant), so the same golden vectors hold for SIMPLIFIED and FULL
    for var in (p.Variant.SIMPLIFIED, p.Variant.FULL):
        pcv = p.SpaceTimePreconditioner(jac, disc, st, variant=var)
        for k in range(disc.n_steps):
            x = g[f"x{k}"]
            assert relerr(pcv.apply_single_step_inverse(k, x).cpu().numpy(), g[f"inv{k}"]) < 1e-10, var
            assert relerr(pcv.apply_single_step(k, x).cpu().numpy(), g[f"fwd{k}"]) < 1e-10, var
        # ...while the space-time apply still uses the variant (differs from TRIANGULAR)
        xs = np.concatenate([g[f"x{k}"] for k in range(disc.n_steps)])
        assert relerr(pcv.apply_inverse(xs).cpu().numpy(), pc.apply_inverse(xs).cpu().numpy()) > 1e-8
    # one slab: the space-time and single-step applications coincide
    d1 = p.discretize(p.by_name("island_coalescence"), 0.5, 1.0, 1.0)
    s1 = p.initial_state(d1)
    j1 = p.assemble_jacobian(s1, d1)
    pc1 = p.SpaceTimePreconditioner(j1, d1, s1)
    x = np.random.default_rng(3).standard_normal(d1.layout.slab_size)
    a, b = pc1.apply_inverse(x).cpu().numpy(), pc1.apply_single_step_inverse(0, x).cpu().numpy()
    assert relerr(b, a) <= 1e-12
    fa, fb = pc1.apply_forward(x).cpu().numpy(), pc1.apply_single_step(0, x).cpu().numpy()
    assert relerr(fb, fa) <= 1e-12
