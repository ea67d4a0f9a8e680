// K2 and the preconditioner's sparse applies: batched multi-term CSR SpMV.
//
//   y[k][r] = beta * z[k][r] + sum_t alpha_t sum_{e in row r of term t}
//                                 val_t[(k - shift_t)][e] * x_t[(k - lag_t)][col_t[e] - off_t]
//
// One launch covers every slab (grid.y) and every block row (grid.x); G lanes
// cooperate on a row (strided over its entries, shuffle-reduced) so the
// per-slab values stream with coalesced loads while column indices and the
// shared matrices stay L2 resident across slabs.  Covers the space-time
// Jacobian (spacetime.py:131-153: per-slab f_u|z_j|z_a and y|f_a rows + the
// shared coupling rows with the -M/dt sub-diagonal), and the bidiagonal /
// tridiagonal applies of the preconditioner (precond.py:133-192, 286-299).
#include "disc.hpp"

namespace stmhd {

template <int G>
__global__ void __launch_bounds__(256) spmv_kernel(SpmvArgs a) {
  const int lane = threadIdx.x % G;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int k = a.kbeg + blockIdx.y;
  const bool valid = r < a.nrows;  // keep the warp converged for the shuffles
  double acc = 0.0;
#pragma unroll
  for (int ti = 0; ti < 4; ++ti) {
    if (ti >= a.nterms || !valid) break;
    const SpTerm &t = a.t[ti];
    const int kx = k - t.lag;
    if (kx < 0) continue;
    const int b = t.beg[r];
    const int e = t.end ? t.end[r] : t.beg[r + 1];
    const double *v = t.val + (int64_t)(k - t.val_shift) * t.val_stride;
    const double *x = t.x + (int64_t)kx * t.x_stride - t.col_off;
    double s = 0.0;
    if (t.rel) {
      const int64_t base = (int64_t)kx * t.x_stride;
      for (int q = b + lane; q < e; q += G) {
        int c = t.col[q];
        if (base + c - t.col_off >= 0) s += v[q] * x[c];
      }
    } else {
      for (int q = b + lane; q < e; q += G) s += v[q] * x[t.col[q]];
    }
    acc += t.alpha * s;
  }
  acc = group_sum<G>(acc);
  if (lane == 0 && valid) {
    double out = acc;
    if (a.z) out += a.beta * a.z[(int64_t)k * a.z_stride + r];
    a.y[(int64_t)k * a.y_stride + r] = out;
  }
}

void spmv(const SpmvArgs &a, cudaStream_t s, int group) {
  if (a.nrows <= 0 || a.nslab <= 0) return;
  const int threads = 256;
  dim3 grid(cdiv((int64_t)a.nrows * group, threads), a.nslab);
  switch (group) {
    case 4: spmv_kernel<4><<<grid, threads, 0, s>>>(a); break;
    case 8: spmv_kernel<8><<<grid, threads, 0, s>>>(a); break;
    case 16: spmv_kernel<16><<<grid, threads, 0, s>>>(a); break;
    default: spmv_kernel<32><<<grid, threads, 0, s>>>(a); break;
  }
  STMHD_LAUNCH_CHECK();
}

__global__ void dense_row_kernel(const double *w, int n, const double *x, int64_t xs, double *y, int64_t ys,
                                 double alpha) {
  __shared__ double sh[32];
  const int k = blockIdx.x;
  const double *xv = x + (int64_t)k * xs;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += w[i] * xv[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) y[(int64_t)k * ys] += alpha * acc;
}

void dense_row(const double *w, int n, const double *x, int64_t xs, double *y, int64_t ys, int nslab,
               double alpha, cudaStream_t s) {
  dense_row_kernel<<<nslab, 256, 0, s>>>(w, n, x, xs, y, ys, alpha);
  STMHD_LAUNCH_CHECK();
}

}  // namespace stmhd
