// Space-time SpMV in a sliced-ELL layout (stspmv.cu).
//
//   y_k = alpha_a * A_k x_k + alpha_b * B x_{k + rel}
//
// A: one CSR pattern with per-slab values; B: optional CSR with values shared by
// every slab and columns relative to the start of slab k (negative columns reach into
// slab k-1 and are skipped for k = 0).  This is the space-time Jacobian
// (spacetime.py:131-153: per-slab f_u|z_j|z_a / y|f_a rows + the shared B^T, B, M_j,
// K_jA and -M/dt couplings) and the configuration-5 block-bidiagonal operator.
//
// Layout (SELL-32-sigma): rows are sorted by length inside windows of kStSigma rows
// and cut into slices of 32; a slice stores its entries column-major
// ([slice][j][lane]) padded to the slice's longest row, so thread = row and every
// load of values and columns is one coalesced 256-byte warp access.  The per-slab A
// values are relaid from CSR once per assembly (relayout); B is gathered at build.
#pragma once

#include <vector>

#include "common.cuh"

namespace stmhd {

constexpr int kStSigma = 128;

struct StSpmvPlan {
  int nrows = 0, nslices = 0, has_b = 0;
  int64_t nnz_a = 0, nnz_b = 0;
  int64_t sell_a = 0, sell_b = 0;  // padded entries per slab (A) / total (B)
  DevBuf slice;   // int4 per slice: {width A, width B, offset A / 32, offset B / 32}
  DevBuf rowmap;  // nslices*32: original row (-1: padding lane)
  DevBuf src_a;   // sell_a: CSR index of the A entry (-1: padding)
  DevBuf col_a;   // sell_a: column
  DevBuf col_b;   // sell_b: slab-relative column
  DevBuf val_b;   // sell_b: shared values (0 on padding)
  // rpA/colA: host CSR of A; rpB/colB/valB: host CSR of B (may be NULL); col_b_shift
  // is added to every B column (e.g. -n for a coupling to slab k-1 stored in [0, n)).
  void build(int nrows, const int *rpA, const int *colA, const int *rpB, const int *colB, const double *valB,
             int col_b_shift, cudaStream_t s);
  // sell[k*sell_a + e] = csr[k*val_stride + src_a[e]] (0 on padding), k < nt
  void relayout(int nt, const double *csr, int64_t val_stride, double *sell, cudaStream_t s) const;
  // y_k (k in [0, nt)) from the relaid values (slab stride sell_a)
  void apply(int nt, const double *sell, double alpha_a, double alpha_b, const double *x, int64_t xs, double *y,
             int64_t ys, cudaStream_t s) const;
};

}  // namespace stmhd
