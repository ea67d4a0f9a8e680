// K8: fused Gram-Schmidt / FGMRES vector kernels (reference gmres MGS loop,
// linalg.py:163-199, replaced by classical Gram-Schmidt with one
// re-orthogonalisation, CGS2).  Reductions are two-stage with a fixed order,
// so results are bitwise reproducible run to run.
#include <cstdlib>

#include "disc.hpp"

namespace stmhd {

constexpr int KT = 256;       // threads per block
constexpr int KE = 4;         // elements per thread
constexpr int KCH = KT * KE;  // elements per block

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int nblocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + KCH - 1) / KCH); }

// partial[i*B + blk] = sum_{chunk} V_i . w
__global__ void __launch_bounds__(KT) dots_partial(const double *V, int64_t ldv, int nvec, const double *w,
                                                   int64_t n, double *partial) {
  extern __shared__ double sh[];  // nvec * 8
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
  double wv[KE];
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    int64_t i = base + q * KT;
    wv[q] = i < n ? w[i] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v = 0; v < nvec; ++v) {
    const double *Vi = V + (int64_t)v * ldv;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < KE; ++q) {
      int64_t i = base + q * KT;
      if (i < n) acc += Vi[i] * wv[q];
    }
    acc = warp_sum(acc);
    if (lane == 0) sh[v * 8 + warp] = acc;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nvec; v += KT) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[v * 8 + q];
    partial[(int64_t)v * gridDim.x + blockIdx.x] = s;
  }
}

// Same sums as dots_partial (per vector: the block's 4 x 256 elements in the same order,
// same warp and block reductions, so the results are bitwise identical), with KU basis
// vectors per pass: 4 KU independent loads in flight per thread instead of 4.
constexpr int KU = 4;

__global__ void __launch_bounds__(KT) dots_partial_u(const double *__restrict__ V, int64_t ldv, int nvec,
                                                     const double *__restrict__ w, int64_t n, double *partial) {
  extern __shared__ double sh[];  // nvec * 8
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
  double wv[KE];
  bool ok[KE];
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    const int64_t i = base + q * KT;
    ok[q] = i < n;
    wv[q] = ok[q] ? w[i] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int v0 = 0; v0 < nvec; v0 += KU) {
    double x[KU][KE];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const double *Vi = V + (int64_t)min(v0 + u, nvec - 1) * ldv + base;
#pragma unroll
      for (int q = 0; q < KE; ++q) x[u][q] = ok[q] ? Vi[q * KT] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < KE; ++q)
        if (ok[q]) acc += x[u][q] * wv[q];
      acc = warp_sum(acc);
      if (lane == 0 && v0 + u < nvec) sh[(v0 + u) * 8 + warp] = acc;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nvec; v += KT) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[v * 8 + q];
    partial[(int64_t)v * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void reduce_partial(const double *partial, int nblk, double *out) {
  __shared__ double sh[32];
  const double *p = partial + (int64_t)blockIdx.x * nblk;
  double acc = 0.0;
  int i = threadIdx.x;
  for (; i + 7 * (int)blockDim.x < nblk; i += 8 * blockDim.x) {  // eight loads in flight, added in order
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = p[i + q * blockDim.x];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += x[q];
  }
  for (; i < nblk; i += blockDim.x) acc += p[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

// w -= sum_i h_i V_i ; partial dots of V_i with the new w (+ ||w||^2)
__global__ void __launch_bounds__(KT) update_partial(const double *V, int64_t ldv, int nvec, const double *h,
                                                     double *w, int64_t n, double *partial, int do_dots,
                                                     int do_norm) {
  extern __shared__ double sh[];  // (nvec+1)*8 + nvec
  double *hs = sh + (nvec + 1) * 8;
  for (int v = threadIdx.x; v < nvec; v += KT) hs[v] = h[v];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
  double wv[KE];
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    int64_t i = base + q * KT;
    wv[q] = i < n ? w[i] : 0.0;
  }
  for (int v = 0; v < nvec; ++v) {
    const double *Vi = V + (int64_t)v * ldv;
    const double hv = hs[v];
#pragma unroll
    for (int q = 0; q < KE; ++q) {
      int64_t i = base + q * KT;
      if (i < n) wv[q] -= hv * Vi[i];
    }
  }
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    int64_t i = base + q * KT;
    if (i < n) w[i] = wv[q];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nout = (do_dots ? nvec : 0) + (do_norm ? 1 : 0);
  if (!nout) return;
  if (do_dots)
    for (int v = 0; v < nvec; ++v) {
      const double *Vi = V + (int64_t)v * ldv;
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < KE; ++q) {
        int64_t i = base + q * KT;
        if (i < n) acc += Vi[i] * wv[q];
      }
      acc = warp_sum(acc);
      if (lane == 0) sh[v * 8 + warp] = acc;
    }
  if (do_norm) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < KE; ++q) acc += wv[q] * wv[q];
    acc = warp_sum(acc);
    if (lane == 0) sh[(do_dots ? nvec : 0) * 8 + warp] = acc;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nout; v += KT) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[v * 8 + q];
    partial[(int64_t)v * gridDim.x + blockIdx.x] = s;
  }
}

// update_partial with KU basis vectors per pass (same arithmetic in the same order).
__global__ void __launch_bounds__(KT) update_partial_u(const double *__restrict__ V, int64_t ldv, int nvec,
                                                       const double *__restrict__ h, double *w, int64_t n,
                                                       double *partial, int do_dots, int do_norm) {
  extern __shared__ double sh[];  // (nvec+1)*8 + nvec
  double *hs = sh + (nvec + 1) * 8;
  for (int v = threadIdx.x; v < nvec; v += KT) hs[v] = h[v];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
  double wv[KE];
  bool ok[KE];
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    const int64_t i = base + q * KT;
    ok[q] = i < n;
    wv[q] = ok[q] ? w[i] : 0.0;
  }
  for (int v0 = 0; v0 < nvec; v0 += KU) {
    double x[KU][KE];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const double *Vi = V + (int64_t)min(v0 + u, nvec - 1) * ldv + base;
#pragma unroll
      for (int q = 0; q < KE; ++q) x[u][q] = ok[q] ? Vi[q * KT] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      if (v0 + u >= nvec) break;
      const double hv = hs[v0 + u];
#pragma unroll
      for (int q = 0; q < KE; ++q)
        if (ok[q]) wv[q] -= hv * x[u][q];
    }
  }
#pragma unroll
  for (int q = 0; q < KE; ++q)
    if (ok[q]) w[base + q * KT] = wv[q];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nout = (do_dots ? nvec : 0) + (do_norm ? 1 : 0);
  if (!nout) return;
  if (do_dots)
    for (int v0 = 0; v0 < nvec; v0 += KU) {
      double x[KU][KE];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const double *Vi = V + (int64_t)min(v0 + u, nvec - 1) * ldv + base;
#pragma unroll
        for (int q = 0; q < KE; ++q) x[u][q] = ok[q] ? Vi[q * KT] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < KE; ++q)
          if (ok[q]) acc += x[u][q] * wv[q];
        acc = warp_sum(acc);
        if (lane == 0 && v0 + u < nvec) sh[(v0 + u) * 8 + warp] = acc;
      }
    }
  if (do_norm) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < KE; ++q) acc += wv[q] * wv[q];
    acc = warp_sum(acc);
    if (lane == 0) sh[(do_dots ? nvec : 0) * 8 + warp] = acc;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nout; v += KT) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += sh[v * 8 + q];
    partial[(int64_t)v * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void normalize_kernel(const double *x, double *y, int64_t n, const double *nrm2) {
  const double nv = *nrm2;
  const double inv = nv > 0.0 ? 1.0 / sqrt(nv) : 0.0;  // zero vector on breakdown (the host stops there)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] * inv;
}

__global__ void __launch_bounds__(KT) combine_kernel(const double *Z, int64_t ldz, int nvec, const double *c,
                                                     double *x, int64_t n) {
  extern __shared__ double cs[];
  for (int v = threadIdx.x; v < nvec; v += KT) cs[v] = c[v];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    int64_t i = base + q * KT;
    if (i >= n) continue;
    double acc = 0.0;
    for (int v = 0; v < nvec; ++v) acc += cs[v] * Z[(int64_t)v * ldz + i];
    x[i] += acc;
  }
}

__global__ void __launch_bounds__(KT) axpby_kernel(double a, const double *x, double b, const double *y,
                                                   double *out, int64_t n, double *partial) {
  __shared__ double sh[8];
  const int64_t base = (int64_t)blockIdx.x * KCH + threadIdx.x;
  double nrm = 0.0;
#pragma unroll
  for (int q = 0; q < KE; ++q) {
    int64_t i = base + q * KT;
    if (i < n) {
      double v = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
      out[i] = v;
      nrm += v * v;
    }
  }
  if (!partial) return;
  nrm = warp_sum(nrm);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < KT / 32; ++q) s += sh[q];
    partial[blockIdx.x] = s;
  }
}

int64_t gs_work_size(int64_t n, int nvec) { return (int64_t)(nvec + 1) * nblocks_for(n); }

void gs_dots(cudaStream_t s, const double *V, int64_t ldv, int nvec, const double *w, int64_t n, double *h,
             double *work) {
  if (nvec <= 0) return;
  int B = nblocks_for(n);
  static const int v1 = env_int("STMHD_GS_V1", 0);  // 1: one basis vector per pass (the first version)
  if (v1) dots_partial<<<B, KT, nvec * 8 * sizeof(double), s>>>(V, ldv, nvec, w, n, work);
  else dots_partial_u<<<B, KT, nvec * 8 * sizeof(double), s>>>(V, ldv, nvec, w, n, work);
  STMHD_LAUNCH_CHECK();
  reduce_partial<<<nvec, 256, 0, s>>>(work, B, h);
  STMHD_LAUNCH_CHECK();
}

void gs_update(cudaStream_t s, const double *V, int64_t ldv, int nvec, const double *h, double *w, int64_t n,
               double *h2, double *nrm2, double *work) {
  int B = nblocks_for(n);
  size_t smem = ((nvec + 1) * 8 + nvec) * sizeof(double);
  static const int v1 = env_int("STMHD_GS_V1", 0);
  if (v1) update_partial<<<B, KT, smem, s>>>(V, ldv, nvec, h, w, n, work, h2 != nullptr, nrm2 != nullptr);
  else update_partial_u<<<B, KT, smem, s>>>(V, ldv, nvec, h, w, n, work, h2 != nullptr, nrm2 != nullptr);
  STMHD_LAUNCH_CHECK();
  if (h2) {
    reduce_partial<<<nvec, 256, 0, s>>>(work, B, h2);
    STMHD_LAUNCH_CHECK();
  }
  if (nrm2) {
    reduce_partial<<<1, 256, 0, s>>>(work + (int64_t)(h2 ? nvec : 0) * B, B, nrm2);
    STMHD_LAUNCH_CHECK();
  }
}

void gs_normalize(cudaStream_t s, const double *x, double *y, int64_t n, const double *nrm2) {
  normalize_kernel<<<std::min<int64_t>(cdiv(n, 256), 4 * num_sms()), 256, 0, s>>>(x, y, n, nrm2);
  STMHD_LAUNCH_CHECK();
}

void gs_combine(cudaStream_t s, const double *Z, int64_t ldz, int nvec, const double *c, double *x, int64_t n) {
  if (nvec <= 0) return;
  combine_kernel<<<nblocks_for(n), KT, nvec * sizeof(double), s>>>(Z, ldz, nvec, c, x, n);
  STMHD_LAUNCH_CHECK();
}

void axpby(cudaStream_t s, double a, const double *x, double b, const double *y, double *out, int64_t n,
           double *nrm2, double *work) {
  int B = nblocks_for(n);
  axpby_kernel<<<B, KT, 0, s>>>(a, x, b, y, out, n, nrm2 ? work : nullptr);
  STMHD_LAUNCH_CHECK();
  if (nrm2) {
    reduce_partial<<<1, 256, 0, s>>>(work, B, nrm2);
    STMHD_LAUNCH_CHECK();
  }
}

}  // namespace stmhd
