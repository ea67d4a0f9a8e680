"""Patch plan of the element-matrix Jacobian assembly (host, once per discretisation).

The device kernel `values_patch_kernel` (csrc/assembly.cu) assembles every slab's
Jacobian values (reference linearize_slab, spacetime.py:99-112, blocks of
fem.py:341-472) and F_p (precond.py:80-84) patch by patch: for a patch of cells it
first evaluates the element matrices of every element the patch's entries touch
(the patch plus a one-cell halo on its left and bottom) into shared memory, then
each owned CSR entry is the sum of its element contributions, read back as 16-bit
shared-memory offsets.  This module builds those tables from the merged pattern's
contribution lists (patterns.SlabPattern).

Ownership: a P2 node (gi, gj) belongs to cell (min(gi//2, nx-1), min(gj//2, ny-1)),
a P1 node (i, j) to cell (min(i, nx-1), min(j, ny-1)); an entry belongs to its
row's node; a cell to patch (ci//px, cj//py).

Element-matrix layout per slot (doubles, ESZ = 270):
  [0,144)   FU[d][c][il][jl]  (f_u, P2 x P2, 2x2 components)
  [144,180) ZJ[d][il][jl]     (z_j, P2 x P1)
  [180,216) ZA[d][il][jl]     (z_a, P2 x P1)
  [216,252) Y[c][il][jl]      (y,   P1 x P2)
  [252,261) FA[il][jl]        (f_a, P1 x P1)
  [261,270) FP[il][jl]        (F_p, P1 x P1)
"""

from __future__ import annotations

import numpy as np

from .patterns import K_BCDIAG, K_FA, K_FP, K_FU, K_Y, K_ZA, K_ZJ

ESZ = 270
ROUND = 256          # threads per CTA = entries per table round
MAXC = 6             # contribution codes per entry (P2: a vertex diagonal touches 6 elements)
CW = 8               # code slots per entry in the table (one 16-byte word)
NONE = 0xFFFF


def _slot_offset(kd, d, c, il, jl):
    off = np.zeros(len(kd), np.int64)
    m = kd == K_FU
    off[m] = (d[m] * 2 + c[m]) * 36 + il[m] * 6 + jl[m]
    m = kd == K_ZJ
    off[m] = 144 + d[m] * 18 + il[m] * 3 + jl[m]
    m = kd == K_ZA
    off[m] = 180 + d[m] * 18 + il[m] * 3 + jl[m]
    m = kd == K_Y
    off[m] = 216 + c[m] * 18 + il[m] * 6 + jl[m]
    m = kd == K_FA
    off[m] = 252 + il[m] * 3 + jl[m]
    m = kd == K_FP
    off[m] = 261 + il[m] * 3 + jl[m]
    return off


def build_patch_plan(disc, px: int = 6, py: int = 5):
    """Tables for values_patch_kernel, or None when the element pair is not P2/P1."""
    if disc.vel.nloc != 6 or disc.prs.nloc != 3:
        return None
    P, mesh = disc.pattern, disc.mesh
    nx, ny = mesh.nx, mesh.ny
    npx, npy = -(-nx // px), -(-ny // py)
    n_u = disc.layout.n_u
    o_a = P.offsets[2]
    nnv = disc.vel.n_nodes

    def patch_of_cell(ci, cj):
        return (cj // py) * npx + ci // px

    def owner_p2(node):
        return patch_of_cell(np.minimum(disc.vel.gi[node] // 2, nx - 1), np.minimum(disc.vel.gj[node] // 2, ny - 1))

    def owner_p1(space, node):
        return patch_of_cell(np.minimum(space.gi[node], nx - 1), np.minimum(space.gj[node], ny - 1))

    # ---- entries: merged js (CSR order) then F_p ----
    rows = P.rows
    js_owner = np.empty(P.nnz, np.int64)
    mu = rows < n_u
    js_owner[mu] = owner_p2(rows[mu] % nnv)
    ma = rows >= o_a
    js_owner[ma] = owner_p1(disc.cur, rows[ma] - o_a)
    assert np.all(mu | ma), "js entries only on u and A rows"
    kind = P.kind.astype(np.int64)
    kd, d, c = kind & 15, (kind >> 4) & 1, (kind >> 5) & 1
    fp_rows = np.repeat(np.arange(disc.prs.n_nodes), np.diff(P.fp_rowptr))
    fp_owner = owner_p1(disc.prs, fp_rows)

    n_js, n_fp = P.nnz, P.fp_nnz
    owner = np.concatenate([js_owner, fp_owner])
    ekd = np.concatenate([kd, np.full(n_fp, K_FP)])
    ed = np.concatenate([d, np.zeros(n_fp, np.int64)])
    ec = np.concatenate([c, np.zeros(n_fp, np.int64)])
    # output word: js index, or fp index | bit 30; BC diagonal: bit 29 (value 1)
    out = np.concatenate([np.arange(n_js), np.arange(n_fp) | (1 << 30)]).astype(np.int64)
    out[:n_js][kd == K_BCDIAG] |= 1 << 29
    ccnt = np.concatenate([np.diff(P.cptr), np.diff(P.fp_cptr)]).astype(np.int64)
    contrib = np.concatenate([P.contrib, P.fp_contrib]).astype(np.int64)
    assert ccnt.max() <= MAXC

    # ---- contributions -> (patch, element) slots ----
    ent_of = np.repeat(np.arange(len(owner)), ccnt)
    ce = contrib >> 8
    cil, cjl = (contrib >> 4) & 15, contrib & 15
    cpatch = owner[ent_of]
    npatch = npx * npy
    ne = mesh.ne
    # slots sorted by (patch, orientation, element)
    key = np.unique(cpatch * (2 * ne) + (ce & 1) * ne + ce)
    kp = key // (2 * ne)
    ko = (key % (2 * ne)) // ne
    kel = key % ne
    first = np.searchsorted(kp, np.arange(npatch + 1))
    slot_in_patch = np.arange(len(key)) - first[kp]
    n_o = np.zeros((npatch, 2), np.int64)
    np.add.at(n_o, (kp, ko), 1)
    nslots = n_o.sum(1)
    assert nslots.max() * ESZ < NONE, "patch too large for 16-bit slot offsets"
    cslot = slot_in_patch[np.searchsorted(key, cpatch * (2 * ne) + (ce & 1) * ne + ce)]
    code = cslot * ESZ + _slot_offset(ekd[ent_of], ed[ent_of], ec[ent_of], cil, cjl)

    # ---- per patch tables: entries in output order, rounds of ROUND ----
    order = np.lexsort((out & ((1 << 29) - 1), out >> 30, owner))  # by patch, js before fp, index
    cnt = np.bincount(owner, minlength=npatch)
    rounds = -(-cnt // ROUND)
    round_off = np.concatenate([[0], np.cumsum(rounds)])
    total = int(round_off[-1]) * ROUND
    pos_in_patch = np.arange(len(order)) - np.concatenate([[0], np.cumsum(cnt)])[owner[order]]
    tpos = round_off[owner[order]] * ROUND + pos_in_patch  # table position of entry order[i]
    t_out = np.full(total, -1, np.int64)
    t_out[tpos] = out[order]
    # codes: CW uint16 per table entry (one 16-byte word)
    t_code = np.full(total * CW, NONE, np.int64)
    pos_of_ent = np.empty(len(order), np.int64)
    pos_of_ent[order] = tpos
    start = np.concatenate([[0], np.cumsum(ccnt)[:-1]])
    rank = np.arange(len(ent_of)) - np.repeat(start, ccnt)  # contribution number within its entry
    p = pos_of_ent[ent_of]
    t_code[p * CW + rank] = code
    desc = np.stack([round_off[:-1], rounds, first[:-1], n_o[:, 0] | (n_o[:, 1] << 16)], axis=1)
    codes16 = t_code.astype(np.uint16)
    _, W1, _, _ = element_linear_maps(disc.tensors, disc.dt, disc.mu, disc.eta, disc.mu0)
    return dict(desc=desc.astype(np.int32), slots=kel.astype(np.int32), out=t_out.astype(np.int32),
                codes=codes16.view(np.int32), w=W1.ravel(),
                npatch=npatch, max_slots=int(nslots.max()), max_per_orient=int(n_o.max()))


# ---- phase A as a linear map: every element-matrix entry is affine in the element
# state (u: 12 values, A: 3, j: 3), so per orientation E[q] = sum_t W[q][t] s[t] with
# the discretisation constants (1/dt, mu, eta/mu0) folded into W.
NW1, NW2, NW3 = 162, 72, 36      # outputs of the u-, A- and j-driven groups
Q1 = np.r_[0:144, 252:270]       # FU, FA, FP  <- [u00..u05, u10..u15, 1] (13, padded to 14)
Q2 = np.r_[144:180, 216:252]     # ZJ, Y       <- [A0, A1, A2] (padded to 4)
Q3 = np.r_[180:216]              # ZA          <- [j0, j1, j2] (padded to 4)


def element_linear_maps(T, dt, mu, eta, mu0):
    """W1 (2, 162, 14), W2 (2, 72, 4), W3 (2, 36, 4) of values_patch_kernel."""
    idt, ceta = 1.0 / dt, eta / mu0
    W = np.zeros((2, ESZ, 19))   # inputs: u[c][m] at c*6+m, 1 at 12, A[n] at 13+n, j[n] at 16+n
    for o in range(2):
        TV, KV, G1, K1, KP, TP = (T[k][o] for k in ("TV", "KV", "G1", "K1", "KP", "TP"))
        MV, MX, M1, MP = T["MV"], T["MX"], T["M1"], T["MP"]
        for d in range(2):
            for c in range(2):
                for il in range(6):
                    for jl in range(6):
                        q = (d * 2 + c) * 36 + il * 6 + jl
                        if d == c:
                            W[o, q, 12] = MV[il, jl] * idt + mu * KV[il, jl]
                            for cc in range(2):
                                W[o, q, cc * 6:cc * 6 + 6] += TV[il, :, jl, cc]
                        W[o, q, d * 6:d * 6 + 6] += TV[il, jl, :, c]
        for d in range(2):
            for il in range(6):
                for jl in range(3):
                    W[o, 144 + d * 18 + il * 3 + jl, 13:16] = G1[:, d] * MX[il, jl]
                    W[o, 180 + d * 18 + il * 3 + jl, 16:19] = MX[il, :] * G1[jl, d]
        for c in range(2):
            for il in range(3):
                for jl in range(6):
                    W[o, 216 + c * 18 + il * 6 + jl, 13:16] = G1[:, c] * MX[jl, il]
        for il in range(3):
            for jl in range(3):
                q = 252 + il * 3 + jl
                W[o, q, 12] = M1[il, jl] * idt + ceta * K1[il, jl]
                for c in range(2):
                    W[o, q, c * 6:c * 6 + 6] = G1[jl, c] * MX[:, il]
                q = 261 + il * 3 + jl
                W[o, q, 12] = MP[il, jl] * idt + mu * KP[il, jl]
                for c in range(2):
                    W[o, q, c * 6:c * 6 + 6] = TP[il, :, jl, c]
    W1 = np.zeros((2, NW1, 14))
    W1[:, :, :13] = W[:, Q1, :13]
    W2 = np.zeros((2, NW2, 4))
    W2[:, :, :3] = W[:, Q2, 13:16]
    W3 = np.zeros((2, NW3, 4))
    W3[:, :, :3] = W[:, Q3, 16:19]
    return W, W1, W2, W3


# ---- residual (reference residual/_slab_galerkin, spacetime.py:42-85) ----
# Element residual vector per slot (RSZ doubles): RU[d][il] (12) | RP[ml] (3) |
# RJ[ml] (3) | RA[ml] (3).  A row is the sum of its node's element entries plus a
# per-row constant (j rows: -flux; A rows: e_load; Dirichlet rows: raw - bc_val with
# no element part).  The pressure pin row is written by pin_row_kernel.
RSZ = 21


def build_residual_plan(disc, px: int = 16, py: int = 8):
    if disc.vel.nloc != 6 or disc.prs.nloc != 3:
        return None
    mesh, L = disc.mesh, disc.layout
    nx, ny = mesh.nx, mesh.ny
    npx, npy = -(-nx // px), -(-ny // py)
    o_p, o_j, o_a = L.n_u, L.n_u + L.n_p, L.n_u + L.n_p + L.n_j
    nnv = disc.vel.n_nodes

    def patch_of(space, node, k):
        return ((np.minimum(space.gj[node] // k, ny - 1) // py) * npx + np.minimum(space.gi[node] // k, nx - 1) // px)

    add = np.zeros(L.slab_size)
    bc = np.zeros(L.slab_size, bool)
    ubc = np.zeros(L.n_u, bool)
    ubc[disc.u_bc_idx] = True
    abc = np.zeros(L.n_a, bool)
    abc[disc.a_bc_idx] = True
    add[disc.u_bc_idx] = -disc.u_bc_vals
    add[o_a + disc.a_bc_idx] = -disc.a_bc_vals
    bc[disc.u_bc_idx] = True
    bc[o_a + disc.a_bc_idx] = True
    add[o_j:o_a] = -disc.current_flux
    add[o_a:][~abc] = disc.e_load[~abc]
    # (rows, space, grid refinement, node, offset of the field in the element vector)
    specs = []
    for d in range(2):
        r = d * nnv + np.arange(nnv)
        specs.append((r, disc.vel, 2, np.arange(nnv), d * 6))  # RU[d][il]
    npn = disc.prs.n_nodes
    keep = np.arange(npn) != disc.p_pin
    specs.append((o_p + np.arange(npn)[keep], disc.prs, 1, np.arange(npn)[keep], 12))
    n1 = disc.cur.n_nodes
    specs.append((o_j + np.arange(n1), disc.cur, 1, np.arange(n1), 15))
    specs.append((o_a + np.arange(n1), disc.cur, 1, np.arange(n1), 18))
    ent_rows, ent_owner, ent_bc, con_ent, con_e, con_off = [], [], [], [], [], []
    nent = 0
    for r, space, k, node, off in specs:
        ptr, code = space.node_elements()
        own = patch_of(space, node, k)
        isbc = bc[r]
        cnt = np.where(isbc, 0, ptr[node + 1] - ptr[node])
        ent = nent + np.arange(len(r))
        idx = np.repeat(ptr[node], cnt) + (np.arange(cnt.sum()) - np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt))
        cc = code[idx].astype(np.int64)
        ent_rows.append(r), ent_owner.append(own), ent_bc.append(isbc)
        con_ent.append(np.repeat(ent, cnt)), con_e.append(cc >> 4), con_off.append(off + (cc & 15))
        nent += len(r)
    rows = np.concatenate(ent_rows)
    owner = np.concatenate(ent_owner)
    isbc = np.concatenate(ent_bc)
    ce = np.concatenate(con_e)
    cen = np.concatenate(con_ent)
    coff = np.concatenate(con_off)
    ccnt = np.bincount(cen, minlength=nent)
    assert ccnt.max() <= MAXC
    npatch = npx * npy
    ne = mesh.ne
    cpatch = owner[cen]
    key = np.unique(cpatch * (2 * ne) + (ce & 1) * ne + ce)
    kp = key // (2 * ne)
    ko = (key % (2 * ne)) // ne
    first = np.searchsorted(kp, np.arange(npatch + 1))
    slot_in_patch = np.arange(len(key)) - first[kp]
    n_o = np.zeros((npatch, 2), np.int64)
    np.add.at(n_o, (kp, ko), 1)
    assert n_o.sum(1).max() * RSZ < NONE
    # contributions sorted by entry (stable), then slot codes
    order_c = np.argsort(cen, kind="stable")
    cen, ce, coff, cpatch = cen[order_c], ce[order_c], coff[order_c], cpatch[order_c]
    code = slot_in_patch[np.searchsorted(key, cpatch * (2 * ne) + (ce & 1) * ne + ce)] * RSZ + coff
    start = np.concatenate([[0], np.cumsum(ccnt)[:-1]])
    rank = np.arange(len(cen)) - start[cen]
    order = np.lexsort((rows, owner))
    cnt = np.bincount(owner, minlength=npatch)
    rounds = -(-cnt // ROUND)
    round_off = np.concatenate([[0], np.cumsum(rounds)])
    total = int(round_off[-1]) * ROUND
    tpos = round_off[owner[order]] * ROUND + (np.arange(nent) - np.concatenate([[0], np.cumsum(cnt)])[owner[order]])
    t_out = np.full(total, -1, np.int64)
    t_out[tpos] = rows[order] | (isbc[order].astype(np.int64) << 29)
    pos_of = np.empty(nent, np.int64)
    pos_of[order] = tpos
    t_code = np.full(total * CW, NONE, np.int64)
    t_code[pos_of[cen] * CW + rank] = code
    desc = np.stack([round_off[:-1], rounds, first[:-1], n_o[:, 0] | (n_o[:, 1] << 16)], axis=1)
    return dict(desc=desc.astype(np.int32), slots=(key % ne).astype(np.int32), out=t_out.astype(np.int32),
                codes=t_code.astype(np.uint16).view(np.int32), add=add, npatch=npatch,
                max_slots=int(n_o.sum(1).max()))
