"""Device assembly of the state-independent operators (csrc/constops.cu)
against the unmodified reference's matrices (tests/golden/ref_*.npz, made by
tests/golden/make_golden.py) and against the oracle at a BASELINE mesh size.
Reference: fem.py:211-271 (assemble_*), problems.py:185-228."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _close(a, b, tol=1e-12):
    a, b = sp.csr_matrix(a), sp.csr_matrix(b)
    assert a.shape == b.shape
    d = abs(a - b)
    scale = abs(b).max()
    assert (d.max() if d.nnz else 0.0) <= tol * scale, (d.max(), scale)


@pytest.mark.parametrize("name", ["ref_island", "ref_tearing", "bl_island4", "bl_tearing4"])
def test_constant_operators_match_reference(name, golden):
    """Every state-independent matrix the reference's Discretization holds
    (problems.py:185-228; P3/P2 for ref_*, P2/P1 for bl_*), device-assembled."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p
    from conftest import csr_from
    from test_parity_gpu import _disc

    g = golden(name)
    d = _disc(p, name)
    checked = 0
    for key in ("div_bc", "div_t_bc", "mixed_ja_bc", "mass_u_dt_bc", "mass_a_dt_bc", "mass_a_bc", "mass_j",
                "mass_p", "stiff_p_pinned", "stiff_a_bc0", "mass_u", "stiff_u"):
        if key + "_data" in g:
            _close(getattr(d, key), csr_from(g, key))
            checked += 1
    assert checked >= 10


def test_device_assembly_is_what_the_handle_uses():
    """The operators come from the native kernels: the launch counter moves and the
    pattern keeps structural zeros like the reference's COO->CSR sum."""
    from paper_2309_00768_b200 import _lib, fem

    lib = _lib.load()
    m = fem.Mesh(-1, 1, -1, 1, 8, 8)
    vel, prs = fem.Space(m, 2, 2), fem.Space(m, 1)
    T = fem.element_tensors(2, 1, m.hx, m.hy)
    n0 = lib.stmhd_launch_count()
    ops = fem.constant_operators(vel, prs, prs, T)
    assert lib.stmhd_launch_count() - n0 >= 3 * 8  # count + scan + fill per assembled block
    k = ops["stiff_1"]
    assert k.nnz == sp.csr_matrix(abs(ops["mass_1"]) > 0).nnz  # same pattern, zeros kept
    assert abs(k @ np.ones(k.shape[0])).max() <= 1e-13 * abs(k).max()  # constants in the kernel
    mu = ops["mass_u"]
    assert abs((mu @ np.ones(mu.shape[0])).sum() - 2 * m.area) <= 1e-12 * m.area


def test_constant_operators_match_oracle_at_64():
    from oracle import configs, model
    from paper_2309_00768_b200 import fem

    od = model.make_disc(configs.baseline_problem("island", 1e-2), 64, 0.1, 1)
    m = fem.Mesh(-1, 1, -1, 1, 64, 64)
    T = fem.element_tensors(2, 1, m.hx, m.hy)
    ops = fem.constant_operators(fem.Space(m, 2, 2), fem.Space(m, 1), fem.Space(m, 1), T)
    for name, ref in (("mass_u", od.mass_u), ("stiff_u", od.stiff_u), ("mass_p", od.mass_p),
                      ("stiff_p", od.stiff_p), ("mass_1", od.mass_j), ("stiff_1", od.stiff_a), ("div", od.div)):
        _close(ops[name], ref)
