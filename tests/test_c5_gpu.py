"""Configuration-5 scalar advection-diffusion block on the device:
assembly, block-bidiagonal SpMV and the sequential exact inverse against the
reference's golden vectors (c5_tiny) and the CPU oracle (oracle/c5.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5mod():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_00768_b200 import c5

    return c5


def relerr(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_c5_matches_reference_golden(c5mod, golden):
    from conftest import csr_from

    g = golden("c5_tiny")
    nt = g["ufields"].shape[0]
    op = c5mod.C5Operator(8, nt, ufields=g["ufields"])
    for k in range(nt):
        ref = csr_from(g, f"F{k}")
        mine = op.matrix(k)
        assert abs(mine - ref).max() <= 1e-12 * abs(ref).max()
    x = g["x"]
    assert relerr(op.apply(x).cpu().numpy().reshape(nt, -1), g["Fx"]) < 1e-13
    assert relerr(op.solve(x).cpu().numpy().reshape(nt, -1), g["Finv_x"]) < 1e-10


def test_c5_matches_oracle_and_round_trips(c5mod):
    from oracle.c5 import C5

    n, nt = 16, 12
    u = c5mod.c5_velocity_fields(c5mod.c5_host_tables(n)["p1"].coords, nt, seed=3)
    op = c5mod.C5Operator(n, nt, ufields=u)
    ref = C5(n, nt, u)
    x = np.random.default_rng(4).standard_normal(nt * op.n)
    assert relerr(op.apply(x).cpu().numpy(), ref.apply(x).ravel()) < 1e-13
    s = op.solve(x).cpu().numpy()
    assert relerr(s, ref.solve(x).ravel()) < 1e-10
    assert relerr(op.apply(s).cpu().numpy(), x) < 1e-10  # F (F^{-1} x) = x


def test_c5_device_velocity_fields_match_host_generator(c5mod):
    coords = c5mod.c5_host_tables(24)["p1"].coords
    host = c5mod.c5_velocity_fields(coords, 5, seed=7)
    dev = c5mod.c5_velocity_fields_device(coords, 5, seed=7).cpu().numpy()
    assert np.max(np.abs(dev - host)) < 1e-13
    assert np.allclose(np.sqrt((dev ** 2).sum(-1)).max(axis=1), 1.0, atol=1e-14)
