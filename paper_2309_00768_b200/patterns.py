"""Fixed sparsity patterns and gather plans for the device kernels (host, once).

The reference rebuilds every per-slab block with COO->CSR in each Newton step
(``fem.py:192-197``), so its patterns drift with the state (exact zeros are
dropped).  Here each block gets the *union* structural pattern once, with BC
rows/columns removed exactly as ``bc_identity``/``bc_zero`` remove them
(``fem.py:593-610``), and the kernels write values in place.

Merged per-slab CSR "JS" (rows = slab rows, cols = slab coordinates):
  u row  (d,i): [ f_u (c,j) | z_j (o_j+n) | z_a (o_a+n) ]   (BC row: [diag 1])
  A row  m    : [ y (c,n)   | f_a (o_a+n) ]                 (BC row: [diag 1])
  p, j rows   : empty
Every entry carries a kind code and the list of (element, local row, local
col) contributions that sum to its value (codes e*256 + il*16 + jl).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fem import Space

K_BCDIAG, K_FU, K_ZJ, K_ZA, K_Y, K_FA, K_FP = 0, 1, 2, 3, 4, 5, 6


class PairTable:
    """All element-local (row node, col node) couplings of two spaces with
    their (e, il, jl) contributions, sorted by (row, col, e)."""

    def __init__(self, R: Space, Cs: Space):
        ne, nr = R.elem.shape
        nc = Cs.elem.shape[1]
        rows = np.repeat(R.elem[:, :, None], nc, axis=2).ravel()
        cols = np.repeat(Cs.elem[:, None, :], nr, axis=1).ravel()
        e = np.repeat(np.arange(ne), nr * nc)
        il = np.tile(np.repeat(np.arange(nr), nc), ne)
        jl = np.tile(np.arange(nc), ne * nr)
        code = (e * 256 + il * 16 + jl).astype(np.int64)
        key = rows.astype(np.int64) * Cs.n_nodes + cols
        order = np.lexsort((code, key))
        key, self.code = key[order], code[order].astype(np.int32)
        self.ukey, self.start, self.count = np.unique(key, return_index=True, return_counts=True)
        self.row = (self.ukey // Cs.n_nodes).astype(np.int64)
        self.col = (self.ukey % Cs.n_nodes).astype(np.int64)
        self.ncol = Cs.n_nodes


def _gather_codes(tab: PairTable, pair_ids):
    """Concatenated contribution codes of the given pairs (+ per-entry counts)."""
    cnt = tab.count[pair_ids]
    starts = tab.start[pair_ids]
    total = int(cnt.sum())
    if total == 0:
        return np.zeros(0, np.int32), cnt
    rep = np.repeat(starts - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    idx = np.arange(total) + rep
    return tab.code[idx], cnt


class SlabPattern:
    """Merged per-slab CSR + F_p CSR with assembly contribution lists."""

    def __init__(self, vel: Space, prs: Space, p1: Space, layout, u_bc, a_bc):
        nnv = vel.n_nodes
        n_u, n_p, n_j, n_a = layout
        o_p, o_j, o_a = n_u, n_u + n_p, n_u + n_p + n_j
        self.slab = n_u + n_p + n_j + n_a
        ubc = np.zeros(n_u, bool)
        ubc[u_bc] = True
        abc = np.zeros(n_a, bool)
        abc[a_bc] = True
        vv, v1, one_v, oo, pp = (PairTable(vel, vel), PairTable(vel, p1), PairTable(p1, vel),
                                 PairTable(p1, p1), PairTable(prs, prs))
        ent = []  # (row, seg, col, kind, pair_table_id, pair)
        tabs = [vv, v1, one_v, oo]

        def add(rows, seg, cols, kind, tid, pairs):
            ent.append((np.asarray(rows, np.int64), np.full(len(rows), seg, np.int64),
                        np.asarray(cols, np.int64), np.asarray(kind, np.int64),
                        np.full(len(rows), tid, np.int64), np.asarray(pairs, np.int64)))

        pid_vv = np.arange(len(vv.ukey))
        for d in range(2):
            for c in range(2):
                r = d * nnv + vv.row
                cc = c * nnv + vv.col
                keep = ~ubc[r] & ~ubc[cc]
                add(r[keep], 0, cc[keep], np.full(keep.sum(), K_FU | d << 4 | c << 5), 0, pid_vv[keep])
        bcr = np.flatnonzero(ubc)
        add(bcr, 0, bcr, np.full(len(bcr), K_BCDIAG), -1, np.full(len(bcr), -1))
        pid_v1 = np.arange(len(v1.ukey))
        for d in range(2):
            r = d * nnv + v1.row
            keep = ~ubc[r]
            add(r[keep], 1, o_j + v1.col[keep], np.full(keep.sum(), K_ZJ | d << 4), 1, pid_v1[keep])
            keep = ~ubc[r] & ~abc[v1.col]
            add(r[keep], 2, o_a + v1.col[keep], np.full(keep.sum(), K_ZA | d << 4), 1, pid_v1[keep])
        pid_1v = np.arange(len(one_v.ukey))
        for c in range(2):
            cc = c * nnv + one_v.col
            keep = ~abc[one_v.row] & ~ubc[cc]
            add(o_a + one_v.row[keep], 0, cc[keep], np.full(keep.sum(), K_Y | c << 5), 2, pid_1v[keep])
        pid_oo = np.arange(len(oo.ukey))
        keep = ~abc[oo.row] & ~abc[oo.col]
        add(o_a + oo.row[keep], 1, o_a + oo.col[keep], np.full(keep.sum(), K_FA), 3, pid_oo[keep])
        bca = np.flatnonzero(abc)
        add(o_a + bca, 1, o_a + bca, np.full(len(bca), K_BCDIAG), -1, np.full(len(bca), -1))

        rows, seg, cols, kind, tid, pair = (np.concatenate(x) for x in zip(*ent))
        order = np.lexsort((cols, seg, rows))
        rows, seg, cols, kind, tid, pair = (x[order] for x in (rows, seg, cols, kind, tid, pair))
        self.nnz = len(rows)
        self.rowptr = np.zeros(self.slab + 1, np.int64)
        np.add.at(self.rowptr, rows + 1, 1)
        self.rowptr = np.cumsum(self.rowptr)
        self.col = cols.astype(np.int32)
        self.kind = kind.astype(np.int32)
        # contribution lists
        counts = np.zeros(self.nnz, np.int64)
        codes = []
        for t, tab in enumerate(tabs):
            m = tid == t
            cds, cnt = _gather_codes(tab, pair[m])
            counts[m] = cnt
            codes.append((np.flatnonzero(m), cds, cnt))
        self.cptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        contrib = np.zeros(self.cptr[-1], np.int32)
        for ent_idx, cds, cnt in codes:
            if len(ent_idx) == 0:
                continue
            dst = np.repeat(self.cptr[ent_idx], cnt) + (np.arange(len(cds)) - np.repeat(
                np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt))
            contrib[dst] = cds
        self.contrib = contrib
        # segment boundaries
        nrow = self.slab
        segcount = np.zeros((nrow, 3), np.int64)
        np.add.at(segcount, (rows, seg), 1)
        self.seg0_end = (self.rowptr[:-1] + segcount[:, 0]).astype(np.int32)
        self.seg1_end = (self.seg0_end + segcount[:, 1]).astype(np.int32)
        self.rowptr = self.rowptr.astype(np.int32)
        self.rows = rows
        self.offsets = (o_p, o_j, o_a)

        # F_p pattern (pressure space, no BCs; precond.py:80-84)
        self.fp_rowptr = np.zeros(prs.n_nodes + 1, np.int64)
        np.add.at(self.fp_rowptr, pp.row + 1, 1)
        self.fp_rowptr = np.cumsum(self.fp_rowptr).astype(np.int32)
        self.fp_col = pp.col.astype(np.int32)
        self.fp_nnz = len(pp.col)
        cds, cnt = _gather_codes(pp, np.arange(self.fp_nnz))
        self.fp_cptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        self.fp_contrib = cds

    def block(self, row_lo, row_hi, which, col_lo, col_hi):
        """(rowptr, col, value_map) of one sub-block: rows [row_lo,row_hi) of the
        merged CSR, segment `which` (0 or 1 boundary based), columns shifted by
        col_lo.  value_map indexes the slab value array."""
        starts = {0: self.rowptr[:-1], 1: self.seg0_end, 2: self.seg1_end}[which]
        ends = {0: self.seg0_end, 1: self.seg1_end, 2: self.rowptr[1:]}[which]
        s, e = starts[row_lo:row_hi].astype(np.int64), ends[row_lo:row_hi].astype(np.int64)
        cnt = e - s
        rp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
        vmap = (np.repeat(s, cnt) + np.arange(int(cnt.sum())) -
                np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)).astype(np.int32)
        col = self.col[vmap].astype(np.int64) - col_lo
        assert np.all((col >= 0) & (col < col_hi - col_lo))
        return rp, col.astype(np.int32), vmap

    def to_csr(self, values, row_lo, row_hi, which, col_lo, col_hi):
        rp, col, vmap = self.block(row_lo, row_hi, which, col_lo, col_hi)
        return sp.csr_matrix((np.asarray(values)[vmap], col, rp),
                             shape=(row_hi - row_lo, col_hi - col_lo))


def product_plan(A: sp.csr_matrix, B: sp.csr_matrix):
    """Structural product A*B as an entry-centric gather plan:
    for output entry t, pairs (a_idx, b_idx, l) with A[i,l] B[l,j]."""
    A, B = sp.csr_matrix(A), sp.csr_matrix(B)
    A.sort_indices(), B.sort_indices()
    # expand (i, l, a_idx) then (l, j, b_idx)
    ai = np.repeat(np.arange(A.shape[0]), np.diff(A.indptr))
    al = A.indices.astype(np.int64)
    aidx = np.arange(A.nnz)
    blen = np.diff(B.indptr)[al]
    tot = int(blen.sum())
    i = np.repeat(ai, blen)
    a_of = np.repeat(aidx, blen)
    l_of = np.repeat(al, blen)
    offs = np.arange(tot) - np.repeat(np.concatenate([[0], np.cumsum(blen)[:-1]]), blen)
    b_of = np.repeat(B.indptr[al], blen) + offs
    j = B.indices[b_of].astype(np.int64)
    key = i * B.shape[1] + j
    order = np.lexsort((l_of, key))
    key, a_of, b_of, l_of = key[order], a_of[order], b_of[order], l_of[order]
    ukey, start, cnt = np.unique(key, return_index=True, return_counts=True)
    rows = ukey // B.shape[1]
    cols = ukey % B.shape[1]
    rowptr = np.zeros(A.shape[0] + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    return dict(rowptr=np.cumsum(rowptr).astype(np.int32), col=cols.astype(np.int32),
                pptr=np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32),
                a=a_of.astype(np.int32), b=b_of.astype(np.int32), l=l_of.astype(np.int32))


def csr_arrays(m: sp.csr_matrix, drop_zeros=True):
    m = sp.csr_matrix(m, dtype=np.float64)
    if drop_zeros:
        m.eliminate_zeros()
    m.sort_indices()
    return (np.ascontiguousarray(m.indptr, dtype=np.int32), np.ascontiguousarray(m.indices, dtype=np.int32),
            np.ascontiguousarray(m.data, dtype=np.float64))
