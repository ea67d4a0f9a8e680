"""CPU check of the element-matrix patch plan (asm_patches.py): a numpy emulation
of values_patch_kernel (phase A element matrices, phase B 16-bit gathers) equals the
entry-centric contribution sums that values_kernel evaluates (reference
linearize_slab, spacetime.py:99-112; F_p precond.py:80-84), on every entry of the
merged pattern and of F_p."""

import numpy as np
import pytest


def _disc(n):
    import paper_2309_00768_b200.discretization as D

    from paper_2309_00768_b200 import fem
    from conftest import host_assemble

    orig, orig_asm = D.Discretization._build_handle, fem._assemble
    D.Discretization._build_handle = lambda self: None
    fem._assemble = host_assemble  # no GPU here: host stand-in for the device constant assembly
    try:
        from paper_2309_00768_b200 import problems

        d = D.Discretization(problems.baseline_island(1e-2), 2.0 / n, 0.1, 0.2)
    finally:
        D.Discretization._build_handle = orig
        fem._assemble = orig_asm
    return d


def _element_matrices(d, s):
    """ESZ doubles per element, layout of asm_patches (phase A)."""
    T = d.tensors
    L = d.layout
    o_j, o_a = L.n_u + L.n_p, L.n_u + L.n_p + L.n_j
    ev, e1 = d.vel.elem, d.cur.elem
    o = np.arange(len(ev)) & 1
    u = np.stack([s[ev], s[d.vel.n_nodes + ev]], axis=1)  # (ne, 2, 6)
    av, jv = s[o_a + e1], s[o_j + e1]
    TV, KV, G1, K1, KP, TP = (T[k][o] for k in ("TV", "KV", "G1", "K1", "KP", "TP"))
    MV, MX, M1, MP = T["MV"], T["MX"], T["M1"], T["MP"]
    idt, mu, ceta = 1.0 / d.dt, d.mu, d.eta / d.mu0
    E = np.zeros((len(ev), 270))
    tr = np.einsum("ecm,eimjc->eij", u, TV)
    for dd in range(2):
        for c in range(2):
            re = np.einsum("em,eijm->eij", u[:, dd], TV[..., c])
            blk = re + (MV * idt + mu * KV + tr if dd == c else 0.0)
            E[:, (dd * 2 + c) * 36:(dd * 2 + c + 1) * 36] = blk.reshape(-1, 36)
    ga = np.einsum("en,end->ed", av, G1)
    jm = np.einsum("en,in->ei", jv, MX)
    E[:, 144:180] = np.einsum("ed,ij->edij", ga, MX).reshape(-1, 36)
    E[:, 180:216] = np.einsum("ei,ejd->edij", jm, G1).reshape(-1, 36)
    E[:, 216:252] = np.einsum("ec,ji->ecij", ga, MX).reshape(-1, 36)
    mxy = np.einsum("ecl,li->eci", u, MX)
    E[:, 252:261] = (M1 * idt + ceta * K1 + np.einsum("eci,ejc->eij", mxy, G1)).reshape(-1, 9)
    E[:, 261:270] = (MP * idt + np.einsum("ecl,eiljc->eij", u, TP) + mu * KP).reshape(-1, 9)
    return E


@pytest.mark.parametrize("n", [4, 10])
def test_patch_plan_reproduces_entry_sums(n):
    from paper_2309_00768_b200.asm_patches import CW, ESZ, MAXC, NONE, ROUND, build_patch_plan

    d = _disc(n)
    P = d.pattern
    pp = build_patch_plan(d)
    rng = np.random.default_rng(0)
    s = rng.standard_normal(d.layout.slab_size)
    E = _element_matrices(d, s)
    # entry-centric reference: sum of element-matrix entries over each entry's contributions
    def entry_sums(cptr, contrib, kind):
        k = kind.astype(np.int64)
        kd, dd, cc = k & 15, (k >> 4) & 1, (k >> 5) & 1
        from paper_2309_00768_b200.asm_patches import _slot_offset

        cnt = np.diff(cptr)
        ent = np.repeat(np.arange(len(cnt)), cnt)
        e, il, jl = contrib >> 8, (contrib >> 4) & 15, contrib & 15
        off = _slot_offset(kd[ent], dd[ent], cc[ent], il, jl)
        v = np.zeros(len(cnt))
        np.add.at(v, ent, E[e, off])
        v[kd == 0] = 1.0
        return v
    js_ref = entry_sums(P.cptr, P.contrib.astype(np.int64), P.kind)
    fp_ref = entry_sums(P.fp_cptr, P.fp_contrib.astype(np.int64), np.full(P.fp_nnz, 6))
    # emulate the kernel through the tables
    codes = pp["codes"].view(np.uint16)
    js = np.full(P.nnz, np.nan)
    fp = np.full(P.fp_nnz, np.nan)
    for pt, (roff, nr, soff, nn) in enumerate(pp["desc"]):
        n0, n1 = nn & 0xFFFF, nn >> 16
        sl = pp["slots"][soff:soff + n0 + n1]
        assert np.all(sl[:n0] % 2 == 0) and np.all(sl[n0:] % 2 == 1)  # orientation groups
        Ep = E[sl].ravel()
        for i in range(nr * ROUND):
            w = int(pp["out"][roff * ROUND + i])
            if w < 0:
                continue
            base = (roff * ROUND + i) * CW
            v = 0.0
            if w & (1 << 29):
                v = 1.0
            else:
                for j in range(MAXC):
                    c = int(codes[base + j])
                    if c == NONE:
                        break
                    assert c < len(sl) * ESZ
                    v += Ep[c]
            idx = w & ((1 << 29) - 1)
            if w & (1 << 30):
                fp[idx] = v
            else:
                js[idx] = v
    assert not np.isnan(js).any() and not np.isnan(fp).any()  # every entry owned exactly once
    np.testing.assert_allclose(js, js_ref, rtol=1e-13, atol=1e-13 * np.abs(js_ref).max())
    np.testing.assert_allclose(fp, fp_ref, rtol=1e-13, atol=1e-13 * np.abs(fp_ref).max())


@pytest.mark.parametrize("n", [4, 10])
def test_residual_plan_bookkeeping(n):
    """Phase B of residual_patch_kernel through the tables equals the direct node ->
    element gather (Space.node_elements) for arbitrary element vectors: every row of
    the slab except the pressure pin row is written exactly once."""
    from paper_2309_00768_b200.asm_patches import CW, NONE, ROUND, RSZ, build_residual_plan

    d = _disc(n)
    L = d.layout
    o_p, o_j, o_a = L.n_u, L.n_u + L.n_p, L.n_u + L.n_p + L.n_j
    rp = build_residual_plan(d)
    rng = np.random.default_rng(1)
    E = rng.standard_normal((d.mesh.ne, RSZ))
    raw = rng.standard_normal(L.slab_size)
    # direct
    ref = np.full(L.slab_size, np.nan)
    bc = np.zeros(L.slab_size, bool)
    bc[d.u_bc_idx] = True
    bc[o_a + d.a_bc_idx] = True

    def gather(space, rows, base):
        ptr, code = space.node_elements()
        for node, r in enumerate(rows):
            cs = code[ptr[node]:ptr[node + 1]]
            ref[r] = E[cs >> 4, base + (cs & 15)].sum()
    nnv = d.vel.n_nodes
    for dd in range(2):
        gather(d.vel, dd * nnv + np.arange(nnv), dd * 6)
    gather(d.prs, o_p + np.arange(d.prs.n_nodes), 12)
    gather(d.cur, o_j + np.arange(d.cur.n_nodes), 15)
    gather(d.cur, o_a + np.arange(d.cur.n_nodes), 18)
    ref = np.where(bc, raw, ref) + rp["add"]
    ref[o_p + d.p_pin] = np.nan
    # through the tables
    codes = rp["codes"].view(np.uint16)
    got = np.full(L.slab_size, np.nan)
    for roff, nr, soff, nn in rp["desc"]:
        sl = rp["slots"][soff:soff + (nn & 0xFFFF) + (nn >> 16)]
        Ep = E[sl].ravel()
        for i in range(nr * ROUND):
            w = int(rp["out"][roff * ROUND + i])
            if w < 0:
                continue
            r = w & ((1 << 29) - 1)
            assert np.isnan(got[r])
            if w & (1 << 29):
                got[r] = raw[r] + rp["add"][r]
                continue
            cs = codes[(roff * ROUND + i) * CW:(roff * ROUND + i + 1) * CW]
            got[r] = Ep[cs[cs != NONE].astype(np.int64)].sum() + rp["add"][r]
    assert np.isnan(got[o_p + d.p_pin])
    m = ~np.isnan(ref)
    assert np.array_equal(m, ~np.isnan(got))
    np.testing.assert_allclose(got[m], ref[m], rtol=1e-13, atol=1e-13)


def test_element_linear_maps_reproduce_element_matrices():
    from paper_2309_00768_b200.asm_patches import element_linear_maps

    d = _disc(4)
    L = d.layout
    o_j, o_a = L.n_u + L.n_p, L.n_u + L.n_p + L.n_j
    s = np.random.default_rng(2).standard_normal(L.slab_size)
    E = _element_matrices(d, s)
    W, *_ = element_linear_maps(d.tensors, d.dt, d.mu, d.eta, d.mu0)
    ev, e1 = d.vel.elem, d.cur.elem
    S = np.concatenate([s[ev], s[d.vel.n_nodes + ev], np.ones((len(ev), 1)), s[o_a + e1], s[o_j + e1]], axis=1)
    got = np.einsum("eqt,et->eq", W[np.arange(len(ev)) & 1], S)
    np.testing.assert_allclose(got, E, rtol=1e-12, atol=1e-12 * np.abs(E).max())
