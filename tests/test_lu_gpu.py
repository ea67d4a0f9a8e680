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
