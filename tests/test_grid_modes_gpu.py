"""Grid-mode sweeps (one CTA per SM / grid-family pipelined launch with software
barriers, nd_sweep.cu) give the same P_T^{-1} and C5 inverse as the cluster mode:
a child process forces the grid modes (STMHD_SWEEP_GRID=1, STMHD_PC_GRID=1) and its
results are compared with this process's cluster-mode results."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2309_00768_b200 as p
from paper_2309_00768_b200 import c5
d = p.discretize_config("C1")
st = p.initial_state(d)
st.vec.data += 1e-3 * torch.randn(st.vec.data.shape, dtype=torch.float64, device="cuda",
                                  generator=torch.Generator(device="cuda").manual_seed(0))
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
r = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
z = pc.apply_inverse(r)
n, nt = 16, 6
u = c5.c5_velocity_fields(c5.c5_host_tables(n)["p1"].coords, nt, seed=3)
op = c5.C5Operator(n, nt, ufields=u)
x = np.random.default_rng(4).standard_normal(nt * op.n)
s = op.solve(x)
np.savez(sys.argv[2], z=z.cpu().numpy(), s=s.cpu().numpy())
"""


def _run(tmp_path, env_extra, name):
    env = dict(os.environ, **env_extra)
    out = str(tmp_path / name)
    subprocess.run([sys.executable, "-c", CHILD, ROOT, out], env=env, check=True, timeout=600)
    return np.load(out)


def test_grid_modes_match_cluster_mode(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run(tmp_path, {"STMHD_SWEEP_GRID": "0", "STMHD_PC_GRID": "0"}, "cluster.npz")
    b = _run(tmp_path, {"STMHD_SWEEP_GRID": "1", "STMHD_PC_GRID": "1"}, "grid.npz")
    for k in ("z", "s"):
        err = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(a[k])
        assert err < 1e-10, (k, err)


@pytest.mark.parametrize("opt", [
    {"STMHD_SWEEP_DENSE_R": "1"},   # dense top as plain K rows (one row per ring item)
    {"STMHD_SWEEP_DENSE_R": "8"},   # row groups of 8
    {"STMHD_SWEEP_L2PF": "1"},      # extra L2 prefetch cluster next to the stages
    {"STMHD_SWEEP_LDGSTS": "1"},    # warp-wide cp.async item ring instead of cp.async.bulk
    {"STMHD_TOPK_NC": "1"},         # dense-top K built with 32 identity columns per item
])
def test_sweep_options_match_default(tmp_path, opt):
    """The sweep's optional layouts and item paths (nd_sweep.cu, off by default) give
    the same P_T^{-1} (pipelined three-stage launch) and C5 inverse (single stage)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    a = _run(tmp_path, {}, "default.npz")
    b = _run(tmp_path, opt, "opt.npz")
    for k in ("z", "s"):
        err = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(a[k])
        assert err < 1e-12, (k, opt, err)


CHILD_MERGED = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2309_00768_b200 as p
d = p.discretize(p.baseline_island(1e-2), 2.0 / 32, 0.05, 0.3)   # 32^2 P2/P1, 6 slabs: n_u = 8450 (merged tree)
st = p.initial_state(d)
st.vec.data += 1e-3 * torch.randn(st.vec.data.shape, dtype=torch.float64, device="cuda",
                                  generator=torch.Generator(device="cuda").manual_seed(0))
jac = p.assemble_jacobian(st, d)
pc = p.SpaceTimePreconditioner(jac, d, st)
r = torch.randn(jac.size, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
z = pc.apply_inverse(r)
u = pc.solve_velocity(r[: d.n_steps * d.layout.n_u].clone())
np.savez(sys.argv[2], z=z.cpu().numpy(), s=u.cpu().numpy())
"""


@pytest.mark.parametrize("opt", [
    {"STMHD_SWEEP_GRID": "0", "STMHD_PC_GRID": "0"},  # 16-CTA clusters: the amalgamated separators are subtree roots
    {"STMHD_SWEEP_GRID": "0", "STMHD_PC_GRID": "0", "STMHD_SWEEP_SMEM_TABLES": "0"},  # ... on the table-in-ring path
    {"STMHD_SWEEP_DENSE_TOP": "0"},                   # every top level a tree level (wide top-level tasks)
    {"STMHD_ND_MERGE_MASK": "0"},                     # the plain tree
])
def test_amalgamated_tree_launch_modes_match_default(tmp_path, opt):
    """The amalgamated velocity tree (four-child supernodes, DESIGN 4.4b) through every
    sweep path: CTA-local subtrees with resident tables and with tables in the ring,
    top-level tasks with and without the dense top, against the default grid-family
    launch, and the default against the plain tree."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")

    def run(env_extra, name):
        env = dict(os.environ, **env_extra)
        out = str(tmp_path / name)
        subprocess.run([sys.executable, "-c", CHILD_MERGED, ROOT, out], env=env, check=True, timeout=600)
        return np.load(out)

    a = run({}, "default.npz")
    b = run(opt, "opt.npz")
    for k in ("z", "s"):
        err = np.linalg.norm(a[k] - b[k]) / np.linalg.norm(a[k])
        assert err < 1e-12, (k, opt, err)
