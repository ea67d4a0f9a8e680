"""GPU sparse LU (nested-dissection supernodal) vs SuperLU / dense solves.
Mirrors the reference LU tests (reference tests/test_linalg.py:14-50) plus
batched FE matrices from the oracle."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(7)


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p

    return p


def test_lu_identity(pkg):
    lu = pkg.LUFactor(sp.eye(6).tocsr())
    b = RNG.standard_normal(6)
    assert np.allclose(lu.solve(b), b, atol=1e-15)


def test_lu_two_by_two(pkg):
    lu = pkg.LUFactor(sp.csr_matrix(np.array([[2.0, 1.0], [1.0, 3.0]])))
    assert np.allclose(lu.solve(np.array([3.0, 4.0])), [1.0, 1.0], atol=1e-14)


def test_lu_needs_pivoting(pkg):
    lu = pkg.LUFactor(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]])))
    assert np.allclose(lu.solve(np.array([3.0, 4.0])), [4.0, 3.0], atol=1e-15)


def test_lu_random_spd_residual(pkg):
    a = RNG.standard_normal((50, 50))
    a = a @ a.T + 50 * np.eye(50)
    lu = pkg.LUFactor(sp.csr_matrix(a))
    b = RNG.standard_normal(50)
    x = lu.solve(b)
    assert np.linalg.norm(a @ x - b) <= 1e-10 * np.linalg.norm(b)


def test_lu_random_sparse_graph_bisection(pkg):
    n = 400
    a = sp.random(n, n, density=0.01, random_state=3).tocsr() + sp.eye(n) * 4.0
    lu = pkg.LUFactor(a, leaf=16)
    b = RNG.standard_normal(n)
    x = lu.solve(b)
    assert np.linalg.norm(a @ x - b) <= 1e-12 * np.linalg.norm(b)


def test_lu_singular_raises(pkg):
    with pytest.raises(pkg.SingularMatrixError):
        pkg.LUFactor(sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 4.0]]))).solve(np.ones(2))


@pytest.mark.parametrize("n,leaf", [(8, 16), (16, 32), (16, 64), (32, 64)])
def test_lu_fe_velocity_block_batched(pkg, n, leaf):
    """Per-slab F_u blocks of the BASELINE island problem factored as one batch
    with grid-coordinate nested dissection."""
    import torch
    from oracle import configs, model
    from paper_2309_00768_b200.linalg import _LUHandle

    d = model.make_disc(configs.baseline_problem("island", 1e-2), n, 0.1, 3)
    st = model.initial_state(d)
    st.vec += 1e-3 * RNG.standard_normal(st.vec.size)
    jac = model.jacobian(st, d)
    mats = [b.f_u for b in jac.slabs]
    pat = sum(abs(m) for m in mats).tocsr()
    pat.sort_indices()
    vals = []
    for m in mats:
        mm = (m + 0 * pat).tocsr()  # same pattern
        mm = mm + sp.csr_matrix((np.zeros(pat.nnz), pat.indices, pat.indptr), shape=pat.shape)
        mm.sort_indices()
        assert np.array_equal(mm.indices, pat.indices)
        vals.append(mm.data)
    vals = torch.as_tensor(np.stack(vals), device="cuda")
    gx = np.tile(d.vel.coords[:, 0] * 0 + np.arange(d.vel.n_nodes) % (2 * n + 1), 2)
    gy = np.tile(np.arange(d.vel.n_nodes) // (2 * n + 1), 2)
    h = _LUHandle(pat, 3, gx, gy, leaf)
    h.factor(vals, pat.nnz)
    rhs = RNG.standard_normal((3, pat.shape[0]))
    x = torch.empty((3, pat.shape[0]), dtype=torch.float64, device="cuda")
    h.solve(torch.as_tensor(rhs, device="cuda"), x, 3, pat.shape[0], pat.shape[0])
    x = x.cpu().numpy()
    for k in range(3):
        ref = spla.spsolve(mats[k].tocsc(), rhs[k])
        assert np.linalg.norm(x[k] - ref) <= 1e-11 * np.linalg.norm(ref), k
    info = h.info()
    assert info["levels"] >= 1


def _fe_velocity_batch(n, nslab=3):
    """Per-slab F_u blocks (oracle assembly) on one pattern + grid coordinates."""
    from oracle import configs, model

    d = model.make_disc(configs.baseline_problem("island", 1e-2), n, 0.1, nslab)
    st = model.initial_state(d)
    st.vec += 1e-3 * np.random.default_rng(11).standard_normal(st.vec.size)
    jac = model.jacobian(st, d)
    mats = [b.f_u for b in jac.slabs]
    pat = sum(abs(m) for m in mats).tocsr()
    pat.sort_indices()
    vals = []
    for m in mats:
        mm = m.tocsr() + sp.csr_matrix((np.zeros(pat.nnz), pat.indices, pat.indptr), shape=pat.shape)
        mm.sort_indices()
        assert np.array_equal(mm.indices, pat.indices)
        vals.append(mm.data)
    gx = np.tile(np.arange(d.vel.n_nodes) % (2 * n + 1), 2)
    gy = np.tile(np.arange(d.vel.n_nodes) // (2 * n + 1), 2)
    return mats, pat, np.stack(vals), gx, gy


def test_lu_amalgamated_tree(pkg, monkeypatch):
    """Elimination tree with amalgamated separators (nd_analyze merge mask, the default
    of the 32^2+ velocity blocks; STMHD_LU_MERGE_MASK for stmhd_lu handles): supernodes
    with four children through the factorisation, the per-matrix solves and the shared
    factor multi-right-hand-side solve, against SuperLU; fewer tree levels than the plain
    tree and the same solution to rounding."""
    import torch
    from paper_2309_00768_b200.linalg import _LUHandle

    n = 32  # n_u = 8450: the size from which the discretisation merges by default
    mats, pat, vals, gx, gy = _fe_velocity_batch(n)
    N = pat.shape[0]
    rhs = RNG.standard_normal((3, N))
    sols, levels = {}, {}
    for mask in ("0", "336"):
        monkeypatch.setenv("STMHD_LU_MERGE_MASK", mask)
        h = _LUHandle(pat, 3, gx, gy, 32)
        h.factor(torch.as_tensor(vals, device="cuda"), pat.nnz)
        x = torch.empty((3, N), dtype=torch.float64, device="cuda")
        h.solve(torch.as_tensor(rhs, device="cuda"), x, 3, N, N)
        sols[mask] = x.cpu().numpy()
        levels[mask] = h.info()["levels"]
    assert levels["336"] <= levels["0"] - 2, levels
    for k in range(3):
        ref = spla.spsolve(mats[k].tocsc(), rhs[k])
        for mask in sols:
            assert np.linalg.norm(sols[mask][k] - ref) <= 1e-11 * np.linalg.norm(ref), (mask, k)
        assert np.linalg.norm(sols["336"][k] - sols["0"][k]) <= 1e-13 * np.linalg.norm(ref)
    # one shared factor, many right-hand sides (the multi-right-hand-side CTA kernel)
    monkeypatch.setenv("STMHD_LU_MERGE_MASK", "336")
    h1 = _LUHandle(pat, 1, gx, gy, 32)
    h1.factor(torch.as_tensor(vals[:1], device="cuda"), pat.nnz)
    nr = 320  # >= 2 x SMs: four right-hand sides per CTA; its first 16 alone: one per CTA
    rhs2 = RNG.standard_normal((nr, N))
    x2 = torch.empty((nr, N), dtype=torch.float64, device="cuda")
    h1.solve(torch.as_tensor(rhs2, device="cuda"), x2, nr, N, N)
    x2 = x2.cpu().numpy()
    lu0 = spla.splu(mats[0].tocsc())
    for k in (0, 1, 77, nr - 1):
        ref = lu0.solve(rhs2[k])
        assert np.linalg.norm(x2[k] - ref) <= 1e-11 * np.linalg.norm(ref), k
    x3 = torch.empty((16, N), dtype=torch.float64, device="cuda")
    h1.solve(torch.as_tensor(rhs2[:16], device="cuda"), x3, 16, N, N)
    assert np.array_equal(x3.cpu().numpy(), x2[:16])  # same per-right-hand-side arithmetic


def test_lu_shared_factor_many_rhs(pkg):
    """Shared factor, >= 2 x SMs right-hand sides (nd_solve_cta_multi_kernel: four
    right-hand sides per CTA share every factor load -- the constant-operator pre-steps of
    P_T^-1 at 512 slabs): against SuperLU, and bitwise equal to the one-CTA-per-
    right-hand-side kernel (same arithmetic per item and right-hand side)."""
    import torch
    from paper_2309_00768_b200.linalg import _LUHandle

    mats, pat, vals, gx, gy = _fe_velocity_batch(16, nslab=1)
    N = pat.shape[0]
    h = _LUHandle(pat, 1, gx, gy, 32)
    h.factor(torch.as_tensor(vals[:1], device="cuda"), pat.nnz)
    nr = 333
    rhs = RNG.standard_normal((nr, N))
    x = torch.empty((nr, N), dtype=torch.float64, device="cuda")
    h.solve(torch.as_tensor(rhs, device="cuda"), x, nr, N, N)
    x = x.cpu().numpy()
    lu0 = spla.splu(mats[0].tocsc())
    for k in (0, 3, 170, nr - 1):
        ref = lu0.solve(rhs[k])
        assert np.linalg.norm(x[k] - ref) <= 1e-11 * np.linalg.norm(ref), k
    x1 = torch.empty((20, N), dtype=torch.float64, device="cuda")
    h.solve(torch.as_tensor(rhs[-20:], device="cuda"), x1, 20, N, N)
    assert np.array_equal(x1.cpu().numpy(), x[-20:])
