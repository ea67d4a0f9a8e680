"""CPU-only tests: the C-ABI library loads and exports every symbol of
include/stmhd_b200.h, the host-side nested-dissection analysis, the element
tensors / constant operators / fixed patterns against the oracle, and the
problem definitions.  No compute is launched on a device."""

import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "stmhd_b200.h")).read()
    return sorted(set(re.findall(r"\b(stmhd_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2309_00768_b200 import _lib

    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding declares every header symbol
    assert set(syms) <= set(_lib.EXPORTS), set(syms) - set(_lib.EXPORTS)
    assert lib.stmhd_abi_version() == _lib.ABI_VERSION == 3


def _plan_info(mat, gx, gy, leaf):
    from paper_2309_00768_b200 import _lib

    lib = _lib.load()
    mat = sp.csr_matrix(mat)
    mat.sort_indices()
    rp = np.ascontiguousarray(mat.indptr, dtype=np.int32)
    ci = np.ascontiguousarray(mat.indices, dtype=np.int32)
    gx = None if gx is None else np.ascontiguousarray(gx, dtype=np.int32)
    gy = None if gy is None else np.ascontiguousarray(gy, dtype=np.int32)
    out = np.zeros(8, dtype=np.int64)
    _lib.check(lib.stmhd_nd_plan_info(mat.shape[0], _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(gx), _lib.ptr(gy),
                                      leaf, _lib.ptr(out)))
    return dict(zip("factor sn levels maxf symnnz front cbv items".split(), out.tolist()))


@pytest.mark.parametrize("n", [8, 16, 32])
def test_nested_dissection_plan_grid(n):
    """Coordinate bisection on the P2 velocity block: the supernodal fill stays
    below the reference's SuperLU (COLAMD) fill and the tree
    depth grows logarithmically."""
    from paper_2309_00768_b200 import fem

    m = fem.Mesh(-1, 1, -1, 1, n, n)
    vel = fem.Space(m, 2, 2)
    e = vel.elem
    r = np.repeat(e[:, :, None], 6, 2).ravel()
    c = np.repeat(e[:, None, :], 6, 1).ravel()
    A = sp.coo_matrix((np.ones(len(r)), (r, c)), shape=(vel.n_nodes,) * 2).tocsr()
    fu = sp.bmat([[A, A], [A, A]]).tocsr()
    info = _plan_info(fu, np.tile(vel.gi, 2), np.tile(vel.gj, 2), 32)
    superlu_fill = {8: None, 16: 188572, 32: 1421718}[n]
    if superlu_fill:  # same order as SuperLU/COLAMD, below it once the grid is large
        assert info["symnnz"] < (1.0 if n >= 32 else 1.25) * superlu_fill
    assert info["levels"] <= 2 * int(np.log2(n)) + 4
    assert info["maxf"] <= 2 * (2 * n + 1) * 3


def test_nested_dissection_plan_graph_bisection():
    rng = np.random.default_rng(3)
    a = sp.random(300, 300, density=0.02, random_state=3).tocsr() + sp.eye(300)
    info = _plan_info(a + a.T, None, None, 16)
    assert info["sn"] >= 3 and info["factor"] > 0


def test_element_tensors_match_oracle_operators():
    from oracle import configs, model
    from paper_2309_00768_b200 import fem

    d = model.make_disc(configs.baseline_problem("island", 1e-2), 4, 0.1, 3)
    T = fem.element_tensors(2, 1, 0.5, 0.5)
    m = fem.Mesh(-1, 1, -1, 1, 4, 4)
    from conftest import host_assemble as coo

    vel, prs, p1 = fem.Space(m, 2, 2), fem.Space(m, 1), fem.Space(m, 1)
    ops = {"mass_u": fem.blockdiag2(coo(vel, vel, [T["MV"], T["MV"]])),
           "stiff_u": fem.blockdiag2(coo(vel, vel, T["KV"])),
           "mass_p": coo(prs, prs, [T["MP"], T["MP"]]), "stiff_p": coo(prs, prs, T["KP"]),
           "mass_1": coo(p1, p1, [T["M1"], T["M1"]]), "stiff_1": coo(p1, p1, T["K1"]),
           "div": sum(coo(prs, vel, T["BD"][:, :, :, c], coff=c * vel.n_nodes, shape=(prs.ndof, vel.ndof))
                      for c in range(2))}
    for name, ref in (("mass_u", d.mass_u), ("stiff_u", d.stiff_u), ("mass_p", d.mass_p),
                      ("stiff_p", d.stiff_p), ("mass_1", d.mass_j), ("stiff_1", d.stiff_a), ("div", d.div)):
        assert abs(ops[name] - ref).max() <= 1e-14 * abs(ref).max(), name
    # transport tensor against quadrature: int phi_i phi_m d_c phi_j on the lower element
    from oracle import fe

    pts, w = fe.duffy_rule(6)
    tab, g = fe.ref_basis(2, pts)
    inv = np.linalg.inv(np.array([[0.5, 0.5], [0.0, 0.5]]))
    gp = np.einsum("iqr,rd->iqd", g, inv)
    ref = np.einsum("iq,mq,jqc,q->imjc", tab, tab, gp, w) * 0.25
    assert np.max(np.abs(T["TV"][0] - ref)) < 1e-13 * np.max(np.abs(ref))  # quadrature rounding


def test_slab_pattern_covers_reference_blocks(golden):
    """The fixed union pattern contains every structurally nonzero entry of the
    reference's per-slab blocks (BC rows/cols removed as bc_identity/bc_zero do)."""
    from conftest import csr_from
    from paper_2309_00768_b200 import fem, patterns, problems

    prob = problems.baseline_island(1e-2)
    m = fem.Mesh(-1, 1, -1, 1, 4, 4)
    vel, prs, p1 = fem.Space(m, 2, 2), fem.Space(m, 1), fem.Space(m, 1)
    ubc = fem.slip_dofs(vel)
    abc, _ = fem.dirichlet_dofs(p1, prob.a_dirichlet, prob.a_eq)
    lay = (vel.ndof, prs.ndof, p1.ndof, p1.ndof)
    P = patterns.SlabPattern(vel, prs, p1, lay, ubc, abc)
    g = golden("bl_island4")
    o_p, o_j, o_a = P.offsets
    ones = np.ones(P.nnz)
    blocks = {
        "f_u": P.to_csr(ones, 0, lay[0], 0, 0, lay[0]),
        "z_j": P.to_csr(ones, 0, lay[0], 1, o_j, o_j + lay[2]),
        "z_a": P.to_csr(ones, 0, lay[0], 2, o_a, o_a + lay[3]),
        "y": P.to_csr(ones, o_a, o_a + lay[3], 0, 0, lay[0]),
        "f_a": P.to_csr(ones, o_a, o_a + lay[3], 1, o_a, o_a + lay[3]),
    }
    for name, pat in blocks.items():
        ref = csr_from(g, f"s0_{name}")
        ref.eliminate_zeros()
        missing = (abs(ref) > 0).astype(int) - (abs(ref) > 0).multiply(pat > 0).astype(int)
        assert missing.nnz == 0, name


def test_problem_definitions():
    from paper_2309_00768_b200 import problems

    isl = problems.baseline_island()
    # A_eq(0,0) = ln(1.2)/(2 pi) (reference test_problems.py known answer, beta=0.2)
    assert abs(isl.a_eq(0.0, 0.0) - np.log(1.2) / (2 * np.pi)) < 1e-15
    assert abs(isl.e_eq(0.0, 0.0) - 1e-2 * 2 * np.pi * 0.96 / 1.44) < 1e-15
    tm = problems.baseline_tearing()
    assert abs(tm.a_eq(0.3, 1.0) - 0.5 * np.log(np.cosh(2.0))) < 1e-15
    assert problems.CONFIGS["C2"]["nt"] == 64 and problems.CONFIGS["C3"]["n"] == 64
    with pytest.raises(Exception):
        problems.by_name("nope")


def test_c5_velocity_fields_divergence_free_and_normalised():
    from paper_2309_00768_b200.c5 import c5_velocity_fields

    n = 16
    xs = np.linspace(-1, 1, n + 1)
    X, Y = np.meshgrid(xs, xs, indexing="xy")
    coords = np.column_stack([X.ravel(), Y.ravel()])
    u = c5_velocity_fields(coords, 3, 0)
    assert u.shape == (3, (n + 1) ** 2, 2)
    np.testing.assert_allclose(np.sqrt((u ** 2).sum(-1)).max(axis=1), 1.0, rtol=1e-14)


def test_overhead_ratio_arithmetic_and_errors():
    """reference tests/test_solver.py:76-106 (pure host logic)."""
    from paper_2309_00768_b200 import ConfigurationError, SolveStats, compute_overhead_ratios

    st = SolveStats(mode="spacetime", newton_iters=6, gmres_iters=[2] * 6)
    seq = SolveStats(mode="sequential", newton_iters=6, gmres_iters=[2] * 6, per_step_newton=[3, 3],
                     per_step_gmres=[[2, 1, 1], [1, 1, 2]])
    nr, gr = compute_overhead_ratios(st, seq)
    assert nr == pytest.approx(2.0) and gr == pytest.approx(3.0)
    assert seq.effective_steps == 2 and seq.avg_newton_per_step == 3 and seq.avg_gmres_per_step == 4
    st = SolveStats(mode="spacetime", newton_iters=4, gmres_iters=[3, 3, 3, 3])
    seq = SolveStats(mode="sequential", newton_iters=4, gmres_iters=[3] * 4, per_step_newton=[4],
                     per_step_gmres=[[3, 3, 3, 3]])
    assert compute_overhead_ratios(st, seq) == (1.0, 1.0)
    frozen = SolveStats(mode="sequential", per_step_newton=[0, 0], per_step_gmres=[[], []])
    with pytest.raises(ConfigurationError):
        compute_overhead_ratios(st, frozen)
    with pytest.raises(ConfigurationError):
        compute_overhead_ratios(seq, st)


def test_c5_host_tables_match_reference(golden, monkeypatch):
    """The configuration-5 tables the device assembly consumes, contracted on the host
    in numpy, reproduce the reference's F_k (golden, make_golden.py c5_case) and its
    coupling bc_zero(M/dt) -- pattern exactly, values to 1e-12."""
    from conftest import csr_from, host_assemble
    from paper_2309_00768_b200 import fem
    from paper_2309_00768_b200.c5 import c5_host_tables

    g = golden("c5_tiny")
    monkeypatch.setattr(fem, "_assemble", host_assemble)  # no GPU here (device path: test_c5_gpu.py)
    h = c5_host_tables(8)
    nn = h["p1"].n_nodes
    el = h["p1"].elem
    mloc = h["mloc"].reshape(3, 3)
    grad = h["grad"].reshape(2, 3, 2)
    for k in range(g["ufields"].shape[0]):
        u = g["ufields"][k]
        vals = h["base"].copy()
        for e in range(h["nnz"]):
            for j in range(h["cptr"][e], h["cptr"][e + 1]):
                elem, i, jj, o = h["cinfo"][j]
                s = mloc[i] @ u[el[elem]]  # sum_m M[i][m] u[node_m][c]
                vals[e] += grad[o, jj] @ s
        mine = sp.csr_matrix((vals, h["col"], h["rowptr"]), shape=(nn, nn))
        ref = csr_from(g, f"F{k}")
        np.testing.assert_array_equal(mine.indptr, ref.indptr)
        np.testing.assert_array_equal(mine.indices, ref.indices)
        assert np.max(np.abs(mine.data - ref.data)) <= 1e-12 * np.max(np.abs(ref.data))
    ref_c = csr_from(g, "coupling")
    assert abs(h["coupling"] - ref_c).max() <= 1e-12 * abs(ref_c).max()
    np.testing.assert_array_equal(np.sort(h["bc"]), np.sort(g["bc"]))
