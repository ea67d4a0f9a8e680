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

// A CTA covers `sb` consecutive slabs of its rows (grid.y = slab blocks), U of them
// interleaved per thread so U gathers are in flight per entry (a launch of nrows x
// nslab small CTAs, one slab per thread, was bound by the beg -> col -> x chain of
// L2 round trips).  Per slab the arithmetic is that of one group of G lanes
// (strided partial sums, then the butterfly), so results do not depend on U or sb.
template <int G, int U>
__global__ void __launch_bounds__(256) spmv_kernel(SpmvArgs a, int sb) {
  const int lane = threadIdx.x % G;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / G;
  const bool valid = r < a.nrows;  // keep the warp converged for the shuffles
  const int kend = min(a.kbeg + a.nslab, a.kbeg + (int)blockIdx.y * sb + sb);
  for (int k0 = a.kbeg + blockIdx.y * sb; k0 < kend; k0 += U) {
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.0;
#pragma unroll
    for (int ti = 0; ti < 4; ++ti) {
      if (ti >= a.nterms || !valid) break;
      const SpTerm &t = a.t[ti];
      const int b = t.beg[r];
      const int e = t.end ? t.end[r] : t.beg[r + 1];
      const double *v[U];
      const double *x[U];
      bool on[U];
      int64_t base[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u, kx = k - t.lag;
        on[u] = k < kend && kx >= 0;
        v[u] = t.val + (int64_t)(k - t.val_shift) * t.val_stride;
        x[u] = t.x + (int64_t)kx * t.x_stride - t.col_off;
        base[u] = (int64_t)kx * t.x_stride - t.col_off;
      }
      double sacc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) sacc[u] = 0.0;
      for (int q = b + lane; q < e; q += G) {
        const int c = t.col[q];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (on[u] && (!t.rel || base[u] + c >= 0)) sacc[u] += v[u][q] * x[u][c];
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (on[u]) acc[u] += t.alpha * sacc[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double sum = group_sum<G>(acc[u]);
      const int k = k0 + u;
      if (lane == 0 && valid && k < kend) {
        double out = sum;
        if (a.z) out += a.beta * a.z[(int64_t)k * a.z_stride + r];
        a.y[(int64_t)k * a.y_stride + r] = out;
      }
    }
  }
}

// Row per thread, U slabs per thread (large slab batches): consecutive threads take
// consecutive rows, so every slab's z reads and y writes are coalesced, and each
// entry issues U gathers at once.  Per slab the entries are summed in row order.
template <int U>
__global__ void __launch_bounds__(256) spmv_rows_kernel(SpmvArgs a) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  const int k0 = a.kbeg + blockIdx.y * U, kend = min(a.kbeg + a.nslab, k0 + U);
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
#pragma unroll
  for (int ti = 0; ti < 4; ++ti) {
    if (ti >= a.nterms) break;
    const SpTerm &t = a.t[ti];
    const int b = t.beg[r];
    const int e = t.end ? t.end[r] : t.beg[r + 1];
    double sacc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sacc[u] = 0.0;
    for (int q = b; q < e; ++q) {
      const int c = t.col[q];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + u, kx = k - t.lag;
        const int64_t xi = (int64_t)kx * t.x_stride + c - t.col_off;
        if (k < kend && kx >= 0 && (!t.rel || xi >= 0))
          sacc[u] += t.val[(int64_t)(k - t.val_shift) * t.val_stride + q] * t.x[xi];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < kend && k0 + u - t.lag >= 0) acc[u] += t.alpha * sacc[u];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int k = k0 + u;
    if (k < kend) {
      double out = acc[u];
      if (a.z) out += a.beta * a.z[(int64_t)k * a.z_stride + r];
      a.y[(int64_t)k * a.y_stride + r] = out;
    }
  }
}

void spmv(const SpmvArgs &a, cudaStream_t s, int group) {
  if (a.nrows <= 0 || a.nslab <= 0) return;
  const int threads = 256;
  // large slab batches (>= 128 slabs: the 64^2 and C5 configurations): row per thread,
  // 8 slabs per thread; smaller batches keep the lane-group kernel (and its rounding)
  static const int rows_min = [] {
    const char *e = getenv("STMHD_SPMV_ROWS_MIN");
    return e ? atoi(e) : 128;
  }();
  if (a.nslab >= rows_min) {
    dim3 grid(cdiv((int64_t)a.nrows, threads), (a.nslab + 7) / 8);
    spmv_rows_kernel<8><<<grid, threads, 0, s>>>(a);
    STMHD_LAUNCH_CHECK();
    return;
  }
  const int64_t gx = cdiv((int64_t)a.nrows * group, threads);
  // slabs per CTA: keep >= ~64 CTAs per SM worth of work (8 resident at a time)
  const int64_t want = (int64_t)num_sms() * 64;
  int sb = (int)std::max<int64_t>(1, std::min<int64_t>(16, gx * a.nslab / want));
  const int nby = (int)((a.nslab + sb - 1) / sb);
  dim3 grid(gx, nby);
  if (sb == 1) {  // one slab per CTA (small batches): no interleaving
    switch (group) {
      case 4: spmv_kernel<4, 1><<<grid, threads, 0, s>>>(a, sb); break;
      case 8: spmv_kernel<8, 1><<<grid, threads, 0, s>>>(a, sb); break;
      case 16: spmv_kernel<16, 1><<<grid, threads, 0, s>>>(a, sb); break;
      default: spmv_kernel<32, 1><<<grid, threads, 0, s>>>(a, sb); break;
    }
  } else {
    switch (group) {
      case 4: spmv_kernel<4, 4><<<grid, threads, 0, s>>>(a, sb); break;
      case 8: spmv_kernel<8, 4><<<grid, threads, 0, s>>>(a, sb); break;
      case 16: spmv_kernel<16, 4><<<grid, threads, 0, s>>>(a, sb); break;
      default: spmv_kernel<32, 4><<<grid, threads, 0, s>>>(a, sb); break;
    }
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
