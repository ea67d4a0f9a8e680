// Configuration-5 scalar advection-diffusion block (oracle/c5.py):
// per slab F_k = M/dt + eps K + W(u_k) on a P1 space (W: reference fem.py:430-462,
// lin_a with a P1 vector velocity), Dirichlet rows/columns -> identity, sub-diagonal -C with
// C = bc_zero(M/dt).  Device parts: entry-centric assembly of every slab's values in
// a fixed pattern, the block-bidiagonal batched SpMV, and the exact inverse by the
// cluster sweep over a batched LU (NDFactor::sweep).
#include <cstdint>

#include "capi_common.hpp"
#include "disc.hpp"
#include "nd.hpp"

namespace stmhd {

struct C5Args {
  int64_t nnz;
  const double *base;   // M/dt + eps K at the pattern entries (identity rows on BC rows)
  const int *cptr;      // nnz + 1: element contributions of each entry
  const int4 *cinfo;    // {element, local row, local col, orientation}
  const int *elem;      // 3 nodes per element
  const double *u;      // [slab][node][2]
  int64_t n_nodes;
  double m[3][3];       // P1 element mass (same on both orientations)
  double g[2][3][2];    // P1 basis gradients per orientation
  double *values;       // [slab][nnz]
};

// values[k][e] = base[e] + sum over the entry's element contributions of
//   int psi_i (u_k . grad psi_j) = sum_c g[o][j][c] sum_m M[i][m] u_k[node_m][c]
__global__ void c5_values_kernel(C5Args a) {
  const int k = blockIdx.y;
  const double *uk = a.u + (int64_t)k * a.n_nodes * 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.nnz; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = a.cptr[e]; j < a.cptr[e + 1]; ++j) {
      const int4 c = a.cinfo[j];
      const int *nd = a.elem + 3 * (int64_t)c.x;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double2 um = reinterpret_cast<const double2 *>(uk)[nd[m]];
        s0 = fma(a.m[c.y][m], um.x, s0);
        s1 = fma(a.m[c.y][m], um.y, s1);
      }
      acc = fma(a.g[c.w][c.z][0], s0, fma(a.g[c.w][c.z][1], s1, acc));
    }
    a.values[(int64_t)k * a.nnz + e] = a.base[e] + acc;
  }
}

}  // namespace stmhd

using namespace stmhd;

extern "C" {

int stmhd_c5_values(void *stream, int64_t nnz, int nt, const double *base, const int32_t *cptr,
                    const int32_t *cinfo, const int32_t *elem, const double *u, int64_t n_nodes,
                    const double *mloc9, const double *grad12, double *values) {
  CAPI_BEGIN
  require(nnz >= 0 && nt >= 1 && base && cptr && cinfo && elem && u && mloc9 && grad12 && values,
          "stmhd_c5_values: bad arguments");
  C5Args a{};
  a.nnz = nnz;
  a.base = base;
  a.cptr = cptr;
  a.cinfo = reinterpret_cast<const int4 *>(cinfo);
  a.elem = elem;
  a.u = u;
  a.n_nodes = n_nodes;
  for (int i = 0; i < 9; ++i) a.m[i / 3][i % 3] = mloc9[i];
  for (int i = 0; i < 12; ++i) a.g[i / 6][(i / 2) % 3][i % 2] = grad12[i];
  a.values = values;
  c5_values_kernel<<<dim3((unsigned)std::min<int64_t>(cdiv(std::max<int64_t>(nnz, 1), 256), 1024), nt), 256, 0,
                     (cudaStream_t)stream>>>(a);
  STMHD_LAUNCH_CHECK();
  CAPI_END
}

int stmhd_bidiag_spmv(void *stream, int64_t n, int nt, const int32_t *rowptr, const int32_t *col,
                      const double *vals, int64_t val_stride, const int32_t *c_rowptr, const int32_t *c_col,
                      const double *c_val, double c_coef, const double *x, double *y) {
  CAPI_BEGIN
  require(n >= 1 && nt >= 1 && rowptr && col && vals && x && y, "stmhd_bidiag_spmv: bad arguments");
  SpmvArgs a;
  a.nrows = (int)n;
  a.nslab = nt;
  a.y = y;
  a.y_stride = n;
  SpTerm f;
  f.beg = rowptr;
  f.col = col;
  f.val = vals;
  f.val_stride = val_stride;
  f.x = x;
  f.x_stride = n;
  a.t[0] = f;
  a.nterms = 1;
  if (c_rowptr) {
    SpTerm c;
    c.beg = c_rowptr;
    c.col = c_col;
    c.val = c_val;
    c.x = x;
    c.x_stride = n;
    c.lag = 1;
    c.alpha = c_coef;
    a.t[1] = c;
    a.nterms = 2;
  }
  spmv(a, (cudaStream_t)stream, 8);
  CAPI_END
}

}  // extern "C"
