"""Amalgamated elimination tree of the velocity factor (DESIGN 4.4b; nd_analyze merge
mask, default for n_u >= 8000) on meshes the BASELINE fixtures do not cover: an elongated
P3/P2 mesh (unbalanced coordinate dissection) and a 40^2 P2/P1 mesh (tree depths that are
not the 32^2 / 64^2 ones).  The merged and the plain tree factor the same matrices, so
P_T^-1 v agrees to rounding; P_T (P_T^-1 v) = v checks each on its own.
Reference operators: precond.py:270-340 (apply_inverse / apply_forward)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(p, name):
    if name == "tearing_p3_96x16":
        return p.tearing_mode(), 1.0 / 32, 0.05, 0.15  # [0,3] x [0,1/2], P3/P2: n_u = 28,322
    return p.baseline_island(1e-2), 2.0 / 40, 0.05, 0.15  # 40^2 P2/P1: n_u = 13,122


@pytest.mark.parametrize("name", ["tearing_p3_96x16", "island_p2_40"])
def test_merged_tree_matches_plain_tree(name, monkeypatch):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2309_00768_b200 as p

    prob, dx, dt, T = _case(p, name)
    out = {}
    for mask in ("0", None):  # plain tree, then the default (depths 4, 6, 8)
        if mask is None:
            monkeypatch.delenv("STMHD_ND_MERGE_MASK", raising=False)
        else:
            monkeypatch.setenv("STMHD_ND_MERGE_MASK", mask)
        d = p.discretize(prob, dx, dt, T)
        assert d.layout.n_u >= 8000
        st = p.initial_state(d)
        g = torch.Generator(device="cuda").manual_seed(5)
        st.vec.data += 1e-3 * torch.randn(st.vec.data.shape, dtype=torch.float64, device="cuda", generator=g)
        jac = p.assemble_jacobian(st, d)
        pc = p.SpaceTimePreconditioner(jac, d, st)
        v = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=g)
        x = pc.apply_inverse(v)
        back = pc.apply_forward(x)
        rt = float(torch.linalg.vector_norm(back - v) / torch.linalg.vector_norm(v))
        assert rt <= 1e-10, (name, mask, rt)
        xu = pc.solve_velocity(v[: d.n_steps * d.layout.n_u].clone())
        out[mask] = (x.cpu().numpy(), xu.cpu().numpy(), pc.pivot_ratio)
    (x0, u0, pr0), (x1, u1, pr1) = out["0"], out[None]
    assert np.linalg.norm(x1 - x0) <= 1e-11 * np.linalg.norm(x0)
    assert np.linalg.norm(u1 - u0) <= 1e-11 * np.linalg.norm(u0)
    assert min(pr1.values()) >= 0.1 * min(pr0.values())  # the restricted pivoting is as good
