// Numeric factorisation and solves of the nested-dissection supernodal LU.
//
// Factorisation: one CTA per (supernode, matrix) and tree level; fronts live
// in a global workspace (L2 resident for the small ones); blocked right-
// looking LU with partial pivoting restricted to the supernode's diagonal
// block, smem-tiled FP64 GEMM for the Schur update, explicit triangular
// inverses so the solve is GEMV-only.
//
// Solve: one persistent cooperative kernel.  Level steps are separated by a
// software grid barrier; a time sweep (reference precond.py:122-131,194-205)
// runs all slabs inside the same launch, folding the sub-diagonal coupling
// SpMV into the gather of each supernode's right-hand side.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdio>

#include "nd.hpp"

namespace stmhd {

// ---------------------------------------------------------------------------
// CTA-level FP64 GEMM:  C = beta*C + alpha * A(MxK) B(KxN), row-major, global.
// 256 threads, 64x64 output tiles, 4x4 register micro-tiles, K-tiles of 16.
// ---------------------------------------------------------------------------
constexpr int GT = 64, GK = 16;

__device__ void cta_gemm(int M, int N, int K, double alpha, const double *A, int64_t lda,
                         const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                         double *sm /* 2*GT*GK doubles */, bool transA = false, bool transB = false) {
  // op(A)[i][k] = transA ? A[k*lda+i] : A[i*lda+k];  op(B)[k][j] = transB ? B[j*ldb+k] : B[k*ldb+j]
  if (M <= 0 || N <= 0) return;
  double *As = sm;            // [GK][GT] (k-major so micro-tile loads are contiguous)
  double *Bs = sm + GT * GK;  // [GK][GT]
  const int tid = threadIdx.x;
  const int tr = (tid / 16) * 4, tc = (tid % 16) * 4;
  for (int m0 = 0; m0 < M; m0 += GT)
    for (int n0 = 0; n0 < N; n0 += GT) {
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      for (int k0 = 0; k0 < K; k0 += GK) {
        __syncthreads();
        for (int t = tid; t < GT * GK; t += blockDim.x) {
          if (!transA) {
            int r = t / GK, k = t % GK;
            int gr = m0 + r, gk = k0 + k;
            As[k * GT + r] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.0;
          } else {
            int k = t / GT, r = t % GT;
            int gr = m0 + r, gk = k0 + k;
            As[k * GT + r] = (gr < M && gk < K) ? A[gk * lda + gr] : 0.0;
          }
          if (!transB) {
            int kb = t / GT, c = t % GT;
            int gkb = k0 + kb, gc = n0 + c;
            Bs[kb * GT + c] = (gkb < K && gc < N) ? B[gkb * ldb + gc] : 0.0;
          } else {
            int c = t / GK, kb = t % GK;
            int gkb = k0 + kb, gc = n0 + c;
            Bs[kb * GT + c] = (gkb < K && gc < N) ? B[gc * ldb + gkb] : 0.0;
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < GK; ++k) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = As[k * GT + tr + i];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Bs[k * GT + tc + j];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int gr = m0 + tr + i;
        if (gr >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          int gc = n0 + tc + j;
          if (gc >= N) continue;
          double *c = C + gr * ldc + gc;
          *c = (beta == 0.0 ? 0.0 : beta * *c) + alpha * acc[i][j];
        }
      }
    }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Front factorisation kernel (one level).
// ---------------------------------------------------------------------------
struct FactorArgs {
  const int *lvl_sn;  // supernodes of this level
  const int *ns, *nb;
  const int64_t *idx_off, *child_ptr_i64;  // unused placeholder
  const int *child_ptr, *child_list;
  const int64_t *emap_off;
  const int *emap;
  const int64_t *scat_ptr, *scat_src, *scat_dst;
  const int64_t *sfl_off, *sfu_off, *front_off;
  const double *values;
  int64_t value_stride;
  int batch0;  // first matrix of this chunk
  double *fronts;
  int64_t front_size;
  double *stage;  // column-major factors of this chunk of matrices (relaid out afterwards)
  int64_t stage_size;
  int *status;
};

__global__ void __launch_bounds__(256, 4) nd_factor_level(FactorArgs a) {
  extern __shared__ double smem[];
  __shared__ double red_v[8], red_c[8];
  __shared__ int red_i[8];
  float prat = 1.0f;  // thread 0: smallest pivot ratio of this front
  const int s = a.lvl_sn[blockIdx.x];
  const int bl = blockIdx.y;  // batch slot within chunk
  const int b = a.batch0 + bl;
  const int ns = a.ns[s], nb = a.nb[s], f = ns + nb;
  double *F = a.fronts + (int64_t)bl * a.front_size + a.front_off[s];
  const double *vals = a.values + (int64_t)b * a.value_stride;
  const int tid = threadIdx.x, nt = blockDim.x;

  // 1. zero + scatter original entries
  for (int64_t t = tid; t < (int64_t)f * f; t += nt) F[t] = 0.0;
  __syncthreads();
  for (int64_t e = a.scat_ptr[s] + tid; e < a.scat_ptr[s + 1]; e += nt) F[a.scat_dst[e]] = vals[a.scat_src[e]];
  __syncthreads();
  // 2. extend-add children contribution blocks (fixed child order: deterministic)
  for (int ci = a.child_ptr[s]; ci < a.child_ptr[s + 1]; ++ci) {
    int c = a.child_list[ci];
    int nsc = a.ns[c], nbc = a.nb[c], fc = nsc + nbc;
    const double *Fc = a.fronts + (int64_t)bl * a.front_size + a.front_off[c];
    const int *em = a.emap + a.emap_off[c];
    for (int64_t t = tid; t < (int64_t)nbc * nbc; t += nt) {
      int i = (int)(t / nbc), j = (int)(t % nbc);
      F[(int64_t)em[i] * f + em[j]] += Fc[(int64_t)(nsc + i) * fc + nsc + j];
    }
    __syncthreads();
  }
  // 3. blocked LU with partial pivoting inside the ns x ns block
  int *perm = reinterpret_cast<int *>(smem + 2 * GT * GK);  // ns ints
  for (int i = tid; i < ns; i += nt) perm[i] = i;
  __syncthreads();
  bool singular = false;
  const int PB = 32;
  for (int p0 = 0; p0 < ns; p0 += PB) {
    int pw = min(PB, ns - p0);
    for (int jj = 0; jj < pw; ++jj) {
      int col = p0 + jj;
      // pivot search over rows col..ns-1
      double best = -1.0, cbm = 0.0;
      int bi = col;
      for (int r = col + tid; r < ns; r += nt) {
        double v = fabs(F[(int64_t)r * f + col]);
        if (v > best) { best = v; bi = r; }
      }
      for (int r = ns + tid; r < f; r += nt) cbm = fmax(cbm, fabs(F[(int64_t)r * f + col]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        cbm = fmax(cbm, __shfl_xor_sync(0xffffffffu, cbm, o));
      }
      if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; red_c[tid >> 5] = cbm; }
      __syncthreads();
      // every thread folds the eight warp results itself (same order, same pivot): no
      // serial section on thread 0 and no second barrier to broadcast it
      int piv;
      {
        double bv = red_v[0], cm = red_c[0];
        int bidx = red_i[0];
        for (int w = 1; w < nt / 32; ++w) {
          if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bidx)) { bv = red_v[w]; bidx = red_i[w]; }
          cm = fmax(cm, red_c[w]);
        }
        piv = (bv > 0.0 && isfinite(bv)) ? bidx : -1;
        if (tid == 0) {
          // pivot ratio: the chosen pivot against the largest entry of its column below
          // the diagonal including the contribution-block rows the restricted pivoting
          // does not search (1 = as good as unrestricted partial pivoting)
          if (piv >= 0) prat = fmin(prat, bv / fmax(bv, cm));
          if (piv >= 0 && piv != col) {
            int t = perm[col]; perm[col] = perm[piv]; perm[piv] = t;
          }
        }
      }
      if (piv < 0) { singular = true; break; }
      if (piv != col)
        for (int c = tid; c < f; c += nt) {
          double t = F[(int64_t)col * f + c];
          F[(int64_t)col * f + c] = F[(int64_t)piv * f + c];
          F[(int64_t)piv * f + c] = t;
        }
      __syncthreads();
      double inv = 1.0 / F[(int64_t)col * f + col];
      int rows = f - col - 1, cols = p0 + pw - col - 1;
      for (int r = tid; r < rows; r += nt) F[(int64_t)(col + 1 + r) * f + col] *= inv;
      __syncthreads();
      if (cols > 0) {  // rank-1 update of the panel: W (power of two >= cols) threads per row, no divisions
        int lw = 0;
        while ((1 << lw) < cols) ++lw;
        const int c = tid & ((1 << lw) - 1), rstep = nt >> lw;
        if (c < cols) {
          const double u = F[(int64_t)col * f + col + 1 + c];
          for (int r = tid >> lw; r < rows; r += rstep) {
            double *row = F + (int64_t)(col + 1 + r) * f;
            row[col + 1 + c] -= row[col] * u;
          }
        }
      }
      __syncthreads();
    }
    if (singular) break;
    // U12 block row: rows p0..p0+pw-1, cols p0+pw..f-1 (unit lower solve)
    for (int c = p0 + pw + tid; c < f; c += nt)
      for (int r = 1; r < pw; ++r) {
        double acc = F[(int64_t)(p0 + r) * f + c];
        for (int k = 0; k < r; ++k) acc -= F[(int64_t)(p0 + r) * f + p0 + k] * F[(int64_t)(p0 + k) * f + c];
        F[(int64_t)(p0 + r) * f + c] = acc;
      }
    __syncthreads();
    // trailing update
    int m = f - p0 - pw;
    cta_gemm(m, m, pw, -1.0, F + (int64_t)(p0 + pw) * f + p0, f, F + (int64_t)p0 * f + p0 + pw, f, 1.0,
             F + (int64_t)(p0 + pw) * f + p0 + pw, f, smem);
  }
  if (singular) {
    if (tid == 0) atomicCAS(a.status, 0, s + 1);
    return;
  }
  if (tid == 0) atomicMin(a.status + 1, __float_as_int(prat));  // positive floats order as ints
  // 4. inverse-based factors, column-major in the staging buffer (relaid out
  //    into row-chunk blocks by nd_relayout afterwards):
  //    FLT[t*f + r] = FL[r][t] (FL = [L11^-1 P ; L21 L11^-1 P], f x ns)
  //    FUT[t*ns + r] = FU[r][t] (FU = [U11^-1 | -U11^-1 U12], ns x f)
  double *FLT = a.stage + (int64_t)bl * a.stage_size + a.sfl_off[s];
  double *FUT = a.stage + (int64_t)bl * a.stage_size + a.sfu_off[s];
  // L11^{-1} P: column i of L^{-1} goes to column perm[i]
  for (int i = tid; i < ns; i += nt) {
    int ci = perm[i];
    for (int r = 0; r < ns; ++r) FLT[(int64_t)ci * f + r] = (r == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  // (one thread per column of L11^-1 P, rows in sequence: the same sums in the same
  // order as a row-by-row sweep with a barrier per row, without the barriers)
  for (int i = tid; i < ns; i += nt) {
    double *cl = FLT + (int64_t)perm[i] * f;
    for (int r = i + 1; r < ns; ++r) {
      const double *fr = F + (int64_t)r * f;
      double acc = 0.0;
      for (int k = i; k < r; ++k) acc -= fr[k] * cl[k];
      cl[r] = acc;
    }
  }
  __syncthreads();
  // G^T = (L11^{-1} P)^T L21^T  ->  FLT[c*f + ns + i]
  cta_gemm(ns, nb, ns, 1.0, FLT, f, F + (int64_t)ns * f, f, 0.0, FLT + ns, f, smem, false, true);
  // U11^{-1}: FUT[j*ns + i] for i <= j
  for (int j = tid; j < ns; j += nt)
    for (int i = 0; i < ns; ++i) FUT[(int64_t)j * ns + i] = 0.0;
  __syncthreads();
  for (int j = tid; j < ns; j += nt) {  // one thread per column of U11^-1, rows upwards (same sums, no barriers)
    double *cu = FUT + (int64_t)j * ns;
    for (int i = j; i >= 0; --i) {
      const double *fi = F + (int64_t)i * f;
      const double dinv = 1.0 / fi[i];
      double acc = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) acc -= fi[k] * cu[k];
      cu[i] = acc * dinv;
    }
  }
  __syncthreads();
  // (-U11^{-1} U12)^T = -U12^T U11^{-T}  ->  FUT[(ns+j)*ns + i]
  cta_gemm(nb, ns, ns, -1.0, F + ns, f, FUT, ns, 0.0, FUT + (int64_t)ns * ns, ns, smem, true, false);
}

// Shared-memory variant for fronts that fit on chip (the many small fronts of the
// lower tree levels): the global-memory kernel above runs ~5 block barriers per pivot
// column, each step a chain of L2 round trips; here the front, the triangular
// inverses and the GEMM tiles live in shared memory.  Same operations in the same
// order (identical results); only the contribution block goes back to the global
// front workspace, for the parent's extend-add.
// Shared layout (doubles): Fs [f*f] | T [ns*ns] (L11^-1 P, then U11^-1) | GEMM tiles
// [2*GT*GK] | perm (ints).
__global__ void __launch_bounds__(256, 4) nd_factor_level_smem(FactorArgs a) {
  extern __shared__ double smem[];
  __shared__ double red_v[8], red_c[8];
  __shared__ int red_i[8];
  float prat = 1.0f;  // thread 0: smallest pivot ratio of this front
  const int s = a.lvl_sn[blockIdx.x];
  const int bl = blockIdx.y;
  const int b = a.batch0 + bl;
  const int ns = a.ns[s], nb = a.nb[s], f = ns + nb;
  double *Fg = a.fronts + (int64_t)bl * a.front_size + a.front_off[s];
  const double *vals = a.values + (int64_t)b * a.value_stride;
  const int tid = threadIdx.x, nt = blockDim.x;
  double *F = smem;
  double *T = F + (int64_t)f * f;
  double *gs = T + (int64_t)ns * ns;
  int *perm = reinterpret_cast<int *>(gs + 2 * GT * GK);

  for (int t = tid; t < f * f; t += nt) F[t] = 0.0;
  __syncthreads();
  for (int64_t e = a.scat_ptr[s] + tid; e < a.scat_ptr[s + 1]; e += nt) F[a.scat_dst[e]] = vals[a.scat_src[e]];
  __syncthreads();
  for (int ci = a.child_ptr[s]; ci < a.child_ptr[s + 1]; ++ci) {
    const int c = a.child_list[ci];
    const int nsc = a.ns[c], nbc = a.nb[c], fc = nsc + nbc;
    const double *Fc = a.fronts + (int64_t)bl * a.front_size + a.front_off[c];
    const int *em = a.emap + a.emap_off[c];
    for (int t = tid; t < nbc * nbc; t += nt) {
      const int i = t / nbc, j = t - i * nbc;
      F[em[i] * f + em[j]] += Fc[(int64_t)(nsc + i) * fc + nsc + j];
    }
    __syncthreads();
  }
  for (int i = tid; i < ns; i += nt) perm[i] = i;
  __syncthreads();
  bool singular = false;
  const int PB = 32;
  for (int p0 = 0; p0 < ns; p0 += PB) {
    const int pw = min(PB, ns - p0);
    for (int jj = 0; jj < pw; ++jj) {
      const int col = p0 + jj;
      double best = -1.0, cbm = 0.0;
      int bi = col;
      for (int r = col + tid; r < ns; r += nt) {
        const double v = fabs(F[r * f + col]);
        if (v > best) { best = v; bi = r; }
      }
      for (int r = ns + tid; r < f; r += nt) cbm = fmax(cbm, fabs(F[r * f + col]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        cbm = fmax(cbm, __shfl_xor_sync(0xffffffffu, cbm, o));
      }
      if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; red_c[tid >> 5] = cbm; }
      __syncthreads();
      int piv;  // (every thread folds the eight warp results itself, as in nd_factor_level)
      {
        double bv = red_v[0], cm = red_c[0];
        int bidx = red_i[0];
        for (int w = 1; w < nt / 32; ++w) {
          if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bidx)) { bv = red_v[w]; bidx = red_i[w]; }
          cm = fmax(cm, red_c[w]);
        }
        piv = (bv > 0.0 && isfinite(bv)) ? bidx : -1;
        if (tid == 0) {
          if (piv >= 0) prat = fmin(prat, bv / fmax(bv, cm));
          if (piv >= 0 && piv != col) {
            const int t = perm[col]; perm[col] = perm[piv]; perm[piv] = t;
          }
        }
      }
      if (piv < 0) { singular = true; break; }
      if (piv != col)
        for (int c = tid; c < f; c += nt) {
          const double t = F[col * f + c];
          F[col * f + c] = F[piv * f + c];
          F[piv * f + c] = t;
        }
      __syncthreads();
      const double inv = 1.0 / F[col * f + col];
      const int rows = f - col - 1, cols = p0 + pw - col - 1;
      for (int r = tid; r < rows; r += nt) F[(col + 1 + r) * f + col] *= inv;
      __syncthreads();
      if (cols > 0) {  // rank-1 update of the panel: W (power of two >= cols) threads per row, no divisions
        int lw = 0;
        while ((1 << lw) < cols) ++lw;
        const int c = tid & ((1 << lw) - 1), rstep = nt >> lw;
        if (c < cols) {
          const double u = F[col * f + col + 1 + c];
          for (int r = tid >> lw; r < rows; r += rstep) {
            double *row = F + (col + 1 + r) * f;
            row[col + 1 + c] -= row[col] * u;
          }
        }
      }
      __syncthreads();
    }
    if (singular) break;
    for (int c = p0 + pw + tid; c < f; c += nt)
      for (int r = 1; r < pw; ++r) {
        double acc = F[(p0 + r) * f + c];
        for (int k = 0; k < r; ++k) acc -= F[(p0 + r) * f + p0 + k] * F[(p0 + k) * f + c];
        F[(p0 + r) * f + c] = acc;
      }
    __syncthreads();
    const int m = f - p0 - pw;
    cta_gemm(m, m, pw, -1.0, F + (p0 + pw) * f + p0, f, F + p0 * f + p0 + pw, f, 1.0, F + (p0 + pw) * f + p0 + pw, f,
             gs);
  }
  if (singular) {
    if (tid == 0) atomicCAS(a.status, 0, s + 1);
    return;
  }
  if (tid == 0) atomicMin(a.status + 1, __float_as_int(prat));
  // contribution block back to the global workspace (the parent's extend-add)
  for (int t = tid; t < nb * nb; t += nt) {
    const int i = t / nb, j = t - i * nb;
    Fg[(int64_t)(ns + i) * f + ns + j] = F[(ns + i) * f + ns + j];
  }
  double *FLT = a.stage + (int64_t)bl * a.stage_size + a.sfl_off[s];
  double *FUT = a.stage + (int64_t)bl * a.stage_size + a.sfu_off[s];
  // L11^{-1} P in T (T[ci*ns + r] = FLT[ci*f + r]), rows in sequence
  for (int i = tid; i < ns; i += nt) {
    const int ci = perm[i];
    for (int r = 0; r < ns; ++r) T[ci * ns + r] = (r == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < ns; i += nt) {  // one thread per column, rows in sequence (same sums, no barriers)
    double *cl = T + perm[i] * ns;
    for (int r = i + 1; r < ns; ++r) {
      const double *fr = F + r * f;
      double acc = 0.0;
      for (int k = i; k < r; ++k) acc -= fr[k] * cl[k];
      cl[r] = acc;
    }
  }
  __syncthreads();
  for (int t = tid; t < ns * ns; t += nt) {
    const int ci = t / ns, r = t - ci * ns;
    FLT[(int64_t)ci * f + r] = T[t];
  }
  // G^T = (L11^{-1} P)^T L21^T  ->  FLT[c*f + ns + i]
  cta_gemm(ns, nb, ns, 1.0, T, ns, F + ns * f, f, 0.0, FLT + ns, f, gs, false, true);
  // U11^{-1} in T (T[j*ns + i] = FUT[j*ns + i])
  for (int t = tid; t < ns * ns; t += nt) T[t] = 0.0;
  __syncthreads();
  for (int j = tid; j < ns; j += nt) {  // one thread per column of U11^-1, rows upwards (same sums, no barriers)
    double *cu = T + j * ns;
    for (int i = j; i >= 0; --i) {
      const double *fi = F + i * f;
      const double dinv = 1.0 / fi[i];
      double acc = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) acc -= fi[k] * cu[k];
      cu[i] = acc * dinv;
    }
  }
  __syncthreads();
  for (int t = tid; t < ns * ns; t += nt) FUT[t] = T[t];
  // (-U11^{-1} U12)^T = -U12^T U11^{-T}  ->  FUT[(ns+j)*ns + i]
  cta_gemm(nb, ns, ns, -1.0, F + ns, f, T, ns, 0.0, FUT + (int64_t)ns * ns, ns, gs, true, false);
}

// Warp-per-front variant for the small fronts of the bottom levels (f <= 64, ns <= 32):
// a CTA-wide kernel spends ~5 block barriers per pivot column on fronts this small, so
// here one warp factors one (front, matrix) pair with __syncwarp only, several pairs
// per CTA.  Same restricted partial pivoting (largest |entry| in the column among rows
// col..ns-1, ties to the smaller row); the elimination is the unblocked right-looking
// form (same operations as the blocked one, in a different order); the inverse-based
// factors and the contribution block go where the CTA kernels put them.
// Shared layout per warp (doubles): F [f][fs] (fs = f | 1, odd stride) | T [ns*ns] | perm.
constexpr int kWarpFrontMax = 64, kWarpFrontNs = 32;

__global__ void __launch_bounds__(256) nd_factor_level_warp(FactorArgs a, int cnt, int nbch, int wstride) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int item = blockIdx.x * (blockDim.x >> 5) + wl;
  if (item >= cnt * nbch) return;
  const int s = a.lvl_sn[item % cnt];
  const int bl = item / cnt;
  const int b = a.batch0 + bl;
  const int ns = a.ns[s], nb = a.nb[s], f = ns + nb, fs = f | 1;
  double *F = smem + (int64_t)wl * wstride;
  double *T = F + f * fs;
  const int ts = ns | 1;  // odd column stride of T: lanes on different columns hit different banks
  int *perm = reinterpret_cast<int *>(T + kWarpFrontNs * (kWarpFrontNs + 1));
  double *Fg = a.fronts + (int64_t)bl * a.front_size + a.front_off[s];
  const double *vals = a.values + (int64_t)b * a.value_stride;
  // 1. zero, scatter, extend-add (children in the fixed order)
  for (int t = lane; t < f * fs; t += 32) F[t] = 0.0;
  __syncwarp();
  {
    // 8 entries per lane in flight (the value gathers are random accesses into the
    // matrix; one at a time would serialise on their latency)
    const int64_t e0 = a.scat_ptr[s], e1 = a.scat_ptr[s + 1];
    for (int64_t eb = e0 + lane; eb < e1; eb += 256) {
      int64_t src[8];
      int dst[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t e = eb + 32 * q;
        src[q] = e < e1 ? a.scat_src[e] : -1;
        dst[q] = e < e1 ? (int)a.scat_dst[e] : 0;  // row-major f x f position (< 64^2)
      }
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = src[q] >= 0 ? vals[src[q]] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (src[q] >= 0) F[(dst[q] / f) * fs + dst[q] % f] = v[q];
    }
  }
  __syncwarp();
  for (int ci = a.child_ptr[s]; ci < a.child_ptr[s + 1]; ++ci) {
    const int c = a.child_list[ci];
    const int nsc = a.ns[c], nbc = a.nb[c], fc = nsc + nbc;
    const double *Fc = a.fronts + (int64_t)bl * a.front_size + a.front_off[c];
    const int *em = a.emap + a.emap_off[c];
    for (int t = lane; t < nbc * nbc; t += 32) {
      const int i = t / nbc, j = t - i * nbc;
      F[em[i] * fs + em[j]] += Fc[(int64_t)(nsc + i) * fc + nsc + j];
    }
    __syncwarp();
  }
  if (lane < ns) perm[lane] = lane;
  __syncwarp();
  // 2. LU with pivoting restricted to the ns x ns block, unblocked right-looking
  float prat = 1.0f;
  for (int col = 0; col < ns; ++col) {
    double best = -1.0, cbm = 0.0;
    int bi = col;
    for (int r = col + lane; r < ns; r += 32) {
      const double v = fabs(F[r * fs + col]);
      if (v > best) { best = v; bi = r; }
    }
    for (int r = ns + lane; r < f; r += 32) cbm = fmax(cbm, fabs(F[r * fs + col]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      cbm = fmax(cbm, __shfl_xor_sync(0xffffffffu, cbm, o));
    }
    if (!(best > 0.0 && isfinite(best))) {
      if (lane == 0) atomicCAS(a.status, 0, s + 1);
      return;
    }
    prat = fminf(prat, (float)(best / fmax(best, cbm)));
    if (bi != col) {
      for (int c = lane; c < f; c += 32) {
        const double t = F[col * fs + c];
        F[col * fs + c] = F[bi * fs + c];
        F[bi * fs + c] = t;
      }
      if (lane == 0) {
        const int t = perm[col];
        perm[col] = perm[bi];
        perm[bi] = t;
      }
    }
    __syncwarp();
    const double inv = 1.0 / F[col * fs + col];
    for (int r = col + 1 + lane; r < f; r += 32) {
      const double l = F[r * fs + col] * inv;
      F[r * fs + col] = l;
      double *fr = F + r * fs;
      const double *fc = F + col * fs;
      int c = col + 1;
      for (; c + 4 <= f; c += 4) {  // loads of a group first (the rows cannot alias)
        const double m0 = fc[c], m1 = fc[c + 1], m2 = fc[c + 2], m3 = fc[c + 3];
        const double v0 = fr[c], v1 = fr[c + 1], v2 = fr[c + 2], v3 = fr[c + 3];
        fr[c] = v0 - l * m0;
        fr[c + 1] = v1 - l * m1;
        fr[c + 2] = v2 - l * m2;
        fr[c + 3] = v3 - l * m3;
      }
      for (; c < f; ++c) fr[c] -= l * fc[c];
    }
    __syncwarp();
  }
  if (lane == 0) atomicMin(a.status + 1, __float_as_int(prat));
  // 3. contribution block -> global (the parent's extend-add)
  for (int t = lane; t < nb * nb; t += 32) {
    const int i = t / nb, j = t - i * nb;
    Fg[(int64_t)(ns + i) * f + ns + j] = F[(ns + i) * fs + ns + j];
  }
  double *FLT = a.stage + (int64_t)bl * a.stage_size + a.sfl_off[s];
  double *FUT = a.stage + (int64_t)bl * a.stage_size + a.sfu_off[s];
  // 4a. L11^{-1} P: lane i solves the unit lower system for e_i (column perm[i])
  if (lane < ns) {
    const int ci = perm[lane];
    double *tc = T + ci * ts;
    for (int r = 0; r < ns; ++r) {
      double acc = (r == lane) ? 1.0 : 0.0;
      if (r > lane)
        for (int k = lane; k < r; ++k) acc -= F[r * fs + k] * tc[k];
      tc[r] = acc;
    }
  }
  __syncwarp();
  for (int t = lane; t < ns * ns; t += 32) {
    const int ci = t / ns, r = t - ci * ns;
    FLT[(int64_t)ci * f + r] = T[ci * ts + r];
  }
  // 4b. G^T = (L11^{-1} P)^T L21^T -> FLT[c*f + ns + i]
  for (int t = lane; t < ns * nb; t += 32) {
    const int c = t / nb, i = t - c * nb;
    double acc = 0.0;
    for (int k = 0; k < ns; ++k) acc += T[c * ts + k] * F[(ns + i) * fs + k];
    FLT[(int64_t)c * f + ns + i] = acc;
  }
  __syncwarp();
  // 4c. U11^{-1}: lane j solves for column j (T[j*ns + i], i <= j)
  if (lane < ns) {
    double *tj = T + lane * ts;
    for (int i = ns - 1; i >= 0; --i) {
      double acc = 0.0;
      if (i <= lane) {
        acc = (i == lane) ? 1.0 : 0.0;
        for (int k = i + 1; k <= lane; ++k) acc -= F[i * fs + k] * tj[k];
        acc *= 1.0 / F[i * fs + i];
      }
      tj[i] = acc;
    }
  }
  __syncwarp();
  for (int t = lane; t < ns * ns; t += 32) FUT[t] = T[(t / ns) * ts + t % ns];
  // 4d. (-U11^{-1} U12)^T -> FUT[(ns+i)*ns + j] = -sum_k U12[k][i] U11inv^T[k][j]
  for (int t = lane; t < nb * ns; t += 32) {
    const int i = t / ns, j = t - i * ns;
    double acc = 0.0;
    for (int k = 0; k < ns; ++k) acc += F[k * fs + ns + i] * T[k * ts + j];
    FUT[(int64_t)(ns + i) * ns + j] = -acc;
  }
}

static size_t factor_warp_smem_per_warp(int f) {
  return ((size_t)f * (f | 1) + kWarpFrontNs * (kWarpFrontNs + 1)) * sizeof(double) + kWarpFrontNs * sizeof(int) + 16;
}

// shared-memory bytes of nd_factor_level_smem for a front (f, ns)
static size_t factor_smem_bytes(int f, int ns) {
  return ((size_t)f * f + (size_t)ns * ns + 2 * GT * GK) * sizeof(double) + (size_t)(ns + 1) * sizeof(int);
}

// Column-major staging -> row-chunk blocks [K][R] (zero padded).
__global__ void nd_relayout(const int *lvl_sn_all, const int *ns_, const int *nb_, const int *rf_, const int *rb_,
                            const int64_t *bszf, const int64_t *bszb, const int64_t *sfl, const int64_t *sfu,
                            const int64_t *fl, const int64_t *fu, const double *stage, int64_t stage_size,
                            double *factors, int64_t factor_size, int batch0) {
  const int s = lvl_sn_all[blockIdx.x];
  const int bl = blockIdx.y;
  const int ns = ns_[s], f = ns + nb_[s];
  const double *st = stage + (int64_t)bl * stage_size;
  double *fa = factors + (int64_t)(batch0 + bl) * factor_size;
  // forward FL: rows f, K = ns, staged as FLT[t*f + r]
  {
    const int R = rf_[s];
    const int64_t B = bszf[s];
    const int nc = (f + R - 1) / R;
    const int64_t total = (int64_t)nc * B;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int c = (int)(e / B);
      const int64_t w = e % B;
      const int t = (int)(w / R), rl = (int)(w % R);
      const int r = c * R + rl;
      fa[fl[s] + e] = (t < ns && r < f) ? st[sfl[s] + (int64_t)t * f + r] : 0.0;
    }
  }
  // backward FU: rows ns, K = f, staged as FUT[t*ns + r]
  {
    const int R = rb_[s];
    const int64_t B = bszb[s];
    const int nc = (ns + R - 1) / R;
    const int64_t total = (int64_t)nc * B;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int c = (int)(e / B);
      const int64_t w = e % B;
      const int t = (int)(w / R), rl = (int)(w % R);
      const int r = c * R + rl;
      fa[fu[s] + e] = (t < f && r < ns) ? st[sfu[s] + (int64_t)t * ns + r] : 0.0;
    }
  }
}

void NDDevice::build(const NDPlan &p, cudaStream_t s) {
  plan = &p;
  max_front = p.max_front;
  this->ns = upload_vec(p.ns, s);
  this->nb = upload_vec(p.nb, s);
  first = upload_vec(p.first, s);
  idx_off = upload_vec(p.idx_off, s);
  idx = upload_vec(p.idx, s);
  child_ptr = upload_vec(p.child_ptr, s);
  child_list = upload_vec(p.child_list, s);
  emap_off = upload_vec(p.emap_off, s);
  emap = upload_vec(p.emap, s);
  scat_ptr = upload_vec(p.scat_ptr, s);
  scat_src = upload_vec(p.scat_src, s);
  scat_dst = upload_vec(p.scat_dst, s);
  fl_off = upload_vec(p.fl_off, s);
  fu_off = upload_vec(p.fu_off, s);
  sfl_off = upload_vec(p.sfl_off, s);
  sfu_off = upload_vec(p.sfu_off, s);
  rf = upload_vec(p.rf, s);
  rb = upload_vec(p.rb, s);
  bsz_f = upload_vec(p.bsz_f, s);
  bsz_b = upload_vec(p.bsz_b, s);
  front_off = upload_vec(p.front_off, s);
  cbv_off = upload_vec(p.cbv_off, s);
  std::vector<int> lsn, lptr{0};
  for (auto &l : p.level_sn) {
    lsn.insert(lsn.end(), l.begin(), l.end());
    lptr.push_back((int)lsn.size());
  }
  lvl_sn = upload_vec(lsn, s);
  lvl_ptr = upload_vec(lptr, s);
  // batched-solve work items: one row chunk (a contiguous factor block) each
  std::vector<SolveItem> fw, bw;
  fwd_ptr.assign(1, 0);
  bwd_ptr.assign(1, 0);
  auto item = [&](int sn, int c, int R, int rows, int64_t off) {
    SolveItem it{};
    it.s = sn; it.r0 = c * R; it.r1 = std::min(rows, (c + 1) * R); it.kl = 32 / R;
    it.ns = p.ns[sn]; it.f = p.ns[sn] + p.nb[sn];
    it.wide = p.wide(sn);
    it.foff = off; it.goff = p.idx_off[sn]; it.first = p.first[sn]; it.cboff = p.cbv_off[sn];
    return it;
  };
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int f = p.ns[sn] + p.nb[sn];
      if (f == 0) continue;
      int R = p.rf[sn], nc = (f + R - 1) / R;
      for (int c = 0; c < nc; ++c) fw.push_back(item(sn, c, R, f, p.fl_off[sn] + c * p.bsz_f[sn]));
    }
    fwd_ptr.push_back((int)fw.size());
  }
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int n = p.ns[sn];
      int R = p.rb[sn], nc = (n + R - 1) / R;
      for (int c = 0; c < nc; ++c) bw.push_back(item(sn, c, R, n, p.fu_off[sn] + c * p.bsz_b[sn]));
    }
    bwd_ptr.push_back((int)bw.size());
  }
  // child update slots per front position: children 0, 1 -> y, z; children 2, 3 of an
  // amalgamated (wide) supernode -> w and the parallel table g4
  std::vector<int4> g3(p.idx.size(), make_int4(-1, -1, -1, -1));
  std::vector<int> g4(std::max<size_t>(p.idx.size(), 1), -1);
  for (int sn = 0; sn < p.nsn; ++sn) {
    int64_t o = p.idx_off[sn];
    for (int t = 0; t < p.ns[sn]; ++t) g3[o + t].x = p.idx[o + t];
    int which = 0;
    for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci, ++which) {
      int c = p.child_list[ci];
      require(which < 4, "nd solve: supernode with more than four children");
      for (int a = 0; a < p.nb[c]; ++a) {
        int pos = p.emap[p.emap_off[c] + a];
        int src = (int)(p.cbv_off[c] + a);
        if (which == 0) g3[o + pos].y = src;
        else if (which == 1) g3[o + pos].z = src;
        else if (which == 2) g3[o + pos].w = src;
        else g4[o + pos] = src;
      }
    }
  }
  gather3 = upload_vec(g3, s);
  gather4 = upload_vec(g4, s);
  fwd_items = upload_vec(fw, s);
  bwd_items = upload_vec(bw, s);
  fwd_ptr_d = upload_vec(fwd_ptr, s);
  bwd_ptr_d = upload_vec(bwd_ptr, s);
}

void NDFactor::factor(const double *values, int64_t value_stride, cudaStream_t s) {
  const NDPlan &p = *dev->plan;
  ++gen;  // invalidates derived data (dense top inverse)
  if (factors.bytes != (size_t)nbatch * p.factor_size * sizeof(double))
    factors.alloc_async((size_t)nbatch * p.factor_size * sizeof(double), s);
  if (!status.ptr) status.alloc_async(2 * sizeof(int), s);
  {
    const int init[2] = {0, 0x7f800000};  // ok, smallest pivot ratio = +inf (float bits)
    STMHD_CUDA_CHECK(cudaMemcpyAsync(status.ptr, init, sizeof(init), cudaMemcpyHostToDevice, s));
  }
  // chunk the batch so front workspace + staging stay within a budget: the top tree
  // levels have one front per matrix, so a level launch has (fronts x chunk) CTAs --
  // a small chunk leaves most SMs idle on the largest fronts.  Budget: STMHD_FACTOR_WS_GB
  // (default 16 GiB), at most a quarter of the free device memory, at least 3 GiB.
  static const int ws_env = [] {
    const char *e = getenv("STMHD_FACTOR_WS_GB");
    return e ? atoi(e) : 16;
  }();
  static const int frac_env = [] {  // percent of the free device memory the workspace may take
    const char *e = getenv("STMHD_FACTOR_WS_FRAC");
    return e ? atoi(e) : 25;
  }();
  int64_t budget = (int64_t)std::max(ws_env, 1) << 30;
  {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) budget = std::min<int64_t>(budget, (int64_t)(free_b * frac_env / 100));
    budget = std::max<int64_t>(budget, int64_t(3) << 30);
  }
  int64_t per = (std::max<int64_t>(p.front_size, 1) + p.stage_size) * (int64_t)sizeof(double);
  int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(nbatch, budget / per));
  // equal chunks (a short last chunk would run its levels on few CTAs)
  {
    const int nch = (int)((nbatch + chunk - 1) / chunk);
    chunk = (int)((nbatch + nch - 1) / nch);
  }
  if (getenv("STMHD_FACTOR_INFO")) {
    fprintf(stderr, "[factor] n=%lld nbatch=%d front %.1f MB + stage %.1f MB per matrix, chunk %d, levels %d\n",
            (long long)p.n, nbatch, p.front_size * 8e-6, p.stage_size * 8e-6, chunk, p.nlevels);
    for (int l = 0; l < p.nlevels; ++l) {
      int fmx = 0, nsmx = 0;
      double fs = 0;
      for (int sn : p.level_sn[l]) {
        fmx = std::max(fmx, p.ns[sn] + p.nb[sn]);
        nsmx = std::max(nsmx, p.ns[sn]);
        fs += p.ns[sn] + p.nb[sn];
      }
      fprintf(stderr, "[factor]   level %d: %zu fronts, f max %d mean %.0f, ns max %d\n", l, p.level_sn[l].size(), fmx,
              p.level_sn[l].empty() ? 0.0 : fs / p.level_sn[l].size(), nsmx);
    }
  }
  DevBuf fronts, stage;  // stream-ordered pool: reused by the next factorisation
  fronts.alloc_async((size_t)chunk * std::max<int64_t>(p.front_size, 1) * sizeof(double), s);
  stage.alloc_async((size_t)chunk * std::max<int64_t>(p.stage_size, 1) * sizeof(double), s);
  size_t smem = (2 * GT * GK) * sizeof(double) + (size_t)(p.max_front + 1) * sizeof(int);
  static bool attr_set = false;
  if (smem > 48 * 1024 || !attr_set) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_factor_level, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)std::max<size_t>(smem, 48 * 1024)));
    attr_set = true;
  }
  std::vector<int> lptr{0};
  for (auto &l : p.level_sn) lptr.push_back(lptr.back() + (int)l.size());
  // levels whose largest front fits shared memory run the on-chip kernel
  // (STMHD_FACTOR_SMEM=0: every level in global memory)
  static const int smem_env = [] {
    const char *e = getenv("STMHD_FACTOR_SMEM");
    return e ? atoi(e) : 1;
  }();
  constexpr size_t kFactorSmemMax = 200 * 1024;
  std::vector<size_t> lvl_smem(p.nlevels, 0);
  // levels of small fronts (f <= 64, ns <= 32): one warp per front (STMHD_FACTOR_WARP=0 off)
  static const int warp_env = [] {
    const char *e = getenv("STMHD_FACTOR_WARP");
    return e ? atoi(e) : 1;
  }();
  std::vector<int> lvl_wf(p.nlevels, 0);  // max front of a warp-per-front level, else 0
  static bool warp_attr = false;
  for (int l = 0; l < p.nlevels && warp_env; ++l) {
    int fmx = 0, nsmx = 0;
    for (int sn : p.level_sn[l]) {
      fmx = std::max(fmx, p.ns[sn] + p.nb[sn]);
      nsmx = std::max(nsmx, p.ns[sn]);
    }
    if (fmx > 0 && fmx <= kWarpFrontMax && nsmx <= kWarpFrontNs) lvl_wf[l] = fmx;
  }
  if (!warp_attr) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_factor_level_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kFactorSmemMax));
    warp_attr = true;
  }
  static size_t smem_attr = 0;
  for (int l = 0; l < p.nlevels && smem_env; ++l) {
    size_t need = 0;
    for (int sn : p.level_sn[l]) need = std::max(need, factor_smem_bytes(p.ns[sn] + p.nb[sn], p.ns[sn]));
    if (need <= kFactorSmemMax) lvl_smem[l] = std::max<size_t>(need, 1);
    if (lvl_smem[l] > smem_attr) {
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_factor_level_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)kFactorSmemMax));
      smem_attr = kFactorSmemMax;
    }
  }
  // STMHD_FACTOR_TRACE=1: per level of the first chunk, the kernel, front count, largest
  // front and duration (events; diagnostics only)
  static const bool ftrace = getenv("STMHD_FACTOR_TRACE") != nullptr;
  std::vector<cudaEvent_t> fev;
  for (int b0 = 0; b0 < nbatch; b0 += chunk) {
    int nbch = std::min(chunk, nbatch - b0);
    for (int l = 0; l < p.nlevels; ++l) {
      int cnt = (int)p.level_sn[l].size();
      if (!cnt) continue;
      if (ftrace && b0 == 0) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        fev.push_back(e);
      }
      FactorArgs a{};
      a.lvl_sn = dev->lvl_sn.as<int>() + lptr[l];
      a.ns = dev->ns.as<int>();
      a.nb = dev->nb.as<int>();
      a.idx_off = dev->idx_off.as<int64_t>();
      a.child_ptr = dev->child_ptr.as<int>();
      a.child_list = dev->child_list.as<int>();
      a.emap_off = dev->emap_off.as<int64_t>();
      a.emap = dev->emap.as<int>();
      a.scat_ptr = dev->scat_ptr.as<int64_t>();
      a.scat_src = dev->scat_src.as<int64_t>();
      a.scat_dst = dev->scat_dst.as<int64_t>();
      a.sfl_off = dev->sfl_off.as<int64_t>();
      a.sfu_off = dev->sfu_off.as<int64_t>();
      a.front_off = dev->front_off.as<int64_t>();
      a.values = values;
      a.value_stride = value_stride;
      a.batch0 = b0;
      a.fronts = fronts.as<double>();
      a.front_size = p.front_size;
      a.stage = stage.as<double>();
      a.stage_size = p.stage_size;
      a.status = status.as<int>();
      if (lvl_wf[l] > 0) {
        const size_t pw = (factor_warp_smem_per_warp(lvl_wf[l]) + 15) / 16 * 16;
        const int wpc = (int)std::max<size_t>(1, std::min<size_t>(8, kFactorSmemMax / pw));
        const int64_t pairs = (int64_t)cnt * nbch;
        nd_factor_level_warp<<<(unsigned)((pairs + wpc - 1) / wpc), 32 * wpc, pw * wpc, s>>>(a, cnt, nbch,
                                                                                           (int)(pw / 8));
      } else if (lvl_smem[l] > 0)
        nd_factor_level_smem<<<dim3(cnt, nbch), 256, lvl_smem[l], s>>>(a);
      else
        nd_factor_level<<<dim3(cnt, nbch), 256, smem, s>>>(a);
      STMHD_LAUNCH_CHECK();
    }
    nd_relayout<<<dim3(p.nsn, nbch), 256, 0, s>>>(
        dev->lvl_sn.as<int>(), dev->ns.as<int>(), dev->nb.as<int>(), dev->rf.as<int>(), dev->rb.as<int>(),
        dev->bsz_f.as<int64_t>(), dev->bsz_b.as<int64_t>(), dev->sfl_off.as<int64_t>(), dev->sfu_off.as<int64_t>(),
        dev->fl_off.as<int64_t>(), dev->fu_off.as<int64_t>(), stage.as<double>(), p.stage_size, factors.as<double>(),
        p.factor_size, b0);
    STMHD_LAUNCH_CHECK();
    if (ftrace && b0 == 0) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      fev.push_back(e);
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      fev.push_back(e);
      cudaEventSynchronize(e);
      size_t i = 0;
      for (int l = 0; l < p.nlevels; ++l) {
        const int cnt = (int)p.level_sn[l].size();
        if (!cnt) continue;
        int mf = 0, mns = 0;
        for (int sn : p.level_sn[l]) {
          mf = std::max(mf, p.ns[sn] + p.nb[sn]);
          mns = std::max(mns, p.ns[sn]);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, fev[i], fev[i + 1]);
        fprintf(stderr, "[factor-trace] level %d %s fronts %d x %d max f %d ns %d: %.3f ms\n", l,
                lvl_wf[l] > 0 ? "warp" : (lvl_smem[l] > 0 ? "smem" : "global"), cnt, nbch, mf, mns, ms);
        ++i;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, fev[i], fev[i + 1]);
      fprintf(stderr, "[factor-trace] relayout %.3f ms (chunk of %d of %d matrices)\n", ms, nbch, nbatch);
      for (auto e : fev) cudaEventDestroy(e);
      fev.clear();
    }
  }
  // keep the workspaces alive until the kernels finish
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
}

int NDFactor::check_status(cudaStream_t s) const {
  int h[2] = {0, 0x7f800000};
  STMHD_CUDA_CHECK(cudaMemcpyAsync(h, status.ptr, sizeof(h), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  float r;
  memcpy(&r, &h[1], sizeof(r));
  min_pivot_ratio = r;
  static const double warn_below = [] {
    const char *e = getenv("STMHD_PIVOT_WARN");
    return e ? atof(e) : 1e-8;
  }();
  if (!h[0] && r < warn_below)
    fprintf(stderr, "[stmhd] warning: restricted-pivoting ratio %.3g (n=%lld, %d matrices): a contribution-block "
                    "entry dominates the chosen pivot\n", (double)r, (long long)dev->plan->n, nbatch);
  return h[0];
}

// ---------------------------------------------------------------------------
// Batched solve (many right-hand sides, e.g. the constant mass/stiffness
// factors applied to every slab): one cooperative launch over the whole GPU,
// warp work items = (row chunk, right-hand side), a software grid barrier
// between tree levels.
// ---------------------------------------------------------------------------
struct SolveArgs {
  const SolveItem *fwd_items, *bwd_items;
  const int4 *gather3;
  const int *gather4;
  const int *idx;
  const int *fwd_ptr, *bwd_ptr;
  int nlevels;
  const double *factors;
  int64_t factor_stride;  // 0 when all right-hand sides share one factor
  const double *rhs;
  int64_t ld_rhs;
  double *x;
  int64_t ld_x;
  int nrhs;
  double *ybuf;  // nrhs * n (elimination order)
  int64_t n;
  double *cbv;  // nrhs * cbv_size
  int64_t cbv_size;
  unsigned *bar;
  int vstride;
};

__device__ __forceinline__ void grid_barrier(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    unsigned g = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ void warp_gather(const SolveArgs &a, const double *rhs, const SolveItem &it, const double *cb, double *v) {
  const int lane = threadIdx.x & 31;
  const int4 *g = a.gather3 + it.goff;
  for (int t0 = lane; t0 < it.f; t0 += 128) {
    int4 gg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + 32 * q;
      gg[q] = t < it.f ? g[t] : make_int4(-1, -1, -1, -1);
    }
    double vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double r = gg[q].x >= 0 ? rhs[gg[q].x] : 0.0;
      const double c1 = gg[q].y >= 0 ? cb[gg[q].y] : 0.0;
      const double c2 = gg[q].z >= 0 ? cb[gg[q].z] : 0.0;
      vv[q] = (r + c1) + c2;
    }
    if (it.wide) {  // amalgamated supernode: children 2 and 3
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = t0 + 32 * q;
        const int g4 = t < it.f ? a.gather4[it.goff + t] : -1;
        const double c3 = gg[q].w >= 0 ? cb[gg[q].w] : 0.0;
        const double c4 = g4 >= 0 ? cb[g4] : 0.0;
        vv[q] += c3 + c4;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (t0 + 32 * q < it.f) v[t0 + 32 * q] = vv[q];
  }
  __syncwarp();
}

__device__ void warp_forward(const SolveArgs &a, const double *rhs, const SolveItem &it, int b, double *v) {
  double *cb = a.cbv + (int64_t)b * a.cbv_size;
  warp_gather(a, rhs, it, cb, v);
  const int lane = threadIdx.x & 31, R = 32 / it.kl;
  const int r = it.r0 + (lane & (R - 1));
  const double out = chunk_gemv<true>(a.factors + (int64_t)b * a.factor_stride + it.foff, R, it.ns, v, lane);
  if (lane < R && r < it.r1) {
    if (r < it.ns) a.ybuf[(int64_t)b * a.n + it.first + r] = out;
    else cb[it.cboff + r - it.ns] = v[r] - out;
  }
  __syncwarp();
}

__device__ void warp_backward(const SolveArgs &a, const SolveItem &it, int b, double *w) {
  const int lane = threadIdx.x & 31;
  const int ns = it.ns, f = it.f;
  const int *idx = a.idx + it.goff;
  const double *y = a.ybuf + (int64_t)b * a.n + it.first;
  double *x = a.x + (int64_t)b * a.ld_x;
  for (int t0 = lane; t0 < f; t0 += 128) {
    int ii[4];
    double vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + 32 * q;
      ii[q] = (t >= ns && t < f) ? idx[t] : -1;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + 32 * q;
      vv[q] = t < ns ? y[t] : (ii[q] >= 0 ? x[ii[q]] : 0.0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (t0 + 32 * q < f) w[t0 + 32 * q] = vv[q];
  }
  __syncwarp();
  const int R = 32 / it.kl;
  const int r = it.r0 + (lane & (R - 1));
  const double out = chunk_gemv<true>(a.factors + (int64_t)b * a.factor_stride + it.foff, R, f, w, lane);
  if (lane < R && r < it.r1) x[idx[r]] = out;
  __syncwarp();
}

__global__ void __launch_bounds__(512, 1) nd_solve_kernel(SolveArgs a) {
  extern __shared__ double vbuf[];
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const int nw = gridDim.x * (blockDim.x >> 5);
  double *v = vbuf + (threadIdx.x >> 5) * a.vstride;
  for (int l = 0; l < a.nlevels; ++l) {
    const int i0 = a.fwd_ptr[l], i1 = a.fwd_ptr[l + 1];
    const int64_t total = (int64_t)(i1 - i0) * a.nrhs;
    for (int64_t w = gw; w < total; w += nw) {
      const SolveItem it = a.fwd_items[i0 + (int)(w / a.nrhs)];
      const int b = (int)(w % a.nrhs);
      warp_forward(a, a.rhs + (int64_t)b * a.ld_rhs, it, b, v);
    }
    grid_barrier(a.bar);
  }
  for (int l = a.nlevels - 1; l >= 0; --l) {
    const int i0 = a.bwd_ptr[l], i1 = a.bwd_ptr[l + 1];
    const int64_t total = (int64_t)(i1 - i0) * a.nrhs;
    for (int64_t w = gw; w < total; w += nw) {
      const SolveItem it = a.bwd_items[i0 + (int)(w / a.nrhs)];
      warp_backward(a, it, (int)(w % a.nrhs), v);
    }
    if (l > 0) grid_barrier(a.bar);
  }
}

// One CTA per right-hand side: every right-hand side is an independent tree solve,
// so levels only need __syncthreads (the grid-wide version pays a 2.3 us software
// barrier per level).  Used when there are enough right-hand sides to fill the GPU.
__global__ void __launch_bounds__(512, 1) nd_solve_cta_kernel(SolveArgs a) {
  extern __shared__ double vbuf[];
  const int b = blockIdx.x;
  const int w = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  double *v = vbuf + w * a.vstride;
  const double *rhs = a.rhs + (int64_t)b * a.ld_rhs;
  for (int l = 0; l < a.nlevels; ++l) {
    for (int i = a.fwd_ptr[l] + w; i < a.fwd_ptr[l + 1]; i += nwarp) warp_forward(a, rhs, a.fwd_items[i], b, v);
    __syncthreads();
  }
  for (int l = a.nlevels - 1; l >= 0; --l) {
    for (int i = a.bwd_ptr[l] + w; i < a.bwd_ptr[l + 1]; i += nwarp) warp_backward(a, a.bwd_items[i], b, v);
    __syncthreads();
  }
}


// Multi-right-hand-side variant for a shared factor (nbatch == 1): a CTA solves G
// right-hand sides together, so every factor element a warp loads feeds G dot
// products and the G gathers of a front are in flight at once.  Same per-RHS
// arithmetic order as chunk_gemv (16 loads per step, 4 partial sums).
template <int G>
__device__ __forceinline__ void chunk_gemv_multi(const double *__restrict__ blk, int R, int K, const double *v,
                                                 int vs, int lane, double (&out)[G]) {
  const int kl = 32 / R, rl = lane & (R - 1), kq = lane / R;
  double acc[G][4];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[g][i] = 0.0;
  for (int t = kq; t < K; t += 16 * kl) {
    double m[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) m[q] = __ldg(blk + (int64_t)min(t + q * kl, K - 1) * R + rl);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int tq = t + q * kl;
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g][q & 3] = fma(m[q], tq < K ? v[g * vs + tq] : 0.0, acc[g][q & 3]);
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double o = (acc[g][0] + acc[g][1]) + (acc[g][2] + acc[g][3]);
    for (int sh = R; sh < 32; sh <<= 1) o += __shfl_xor_sync(0xffffffffu, o, sh);
    out[g] = o;
  }
}

template <int G>
__global__ void __launch_bounds__(512, 1) nd_solve_cta_multi_kernel(SolveArgs a) {
  extern __shared__ double vbuf[];
  const int b0 = blockIdx.x * G;
  const int w = threadIdx.x >> 5, nwarp = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int vs = a.vstride;
  double *v = vbuf + (int64_t)w * G * vs;
  int nb = min(G, a.nrhs - b0);
  for (int l = 0; l < a.nlevels; ++l) {
    for (int i = a.fwd_ptr[l] + w; i < a.fwd_ptr[l + 1]; i += nwarp) {
      const SolveItem it = a.fwd_items[i];
      const int4 *gt = a.gather3 + it.goff;
      for (int t = lane; t < it.f; t += 32) {
        const int4 gg = gt[t];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int b = min(b0 + g, a.nrhs - 1);
          const double *rhs = a.rhs + (int64_t)b * a.ld_rhs;
          const double *cb = a.cbv + (int64_t)b * a.cbv_size;
          const double r = gg.x >= 0 ? rhs[gg.x] : 0.0;
          const double c1 = gg.y >= 0 ? cb[gg.y] : 0.0;
          const double c2 = gg.z >= 0 ? cb[gg.z] : 0.0;
          double vv = (r + c1) + c2;
          if (it.wide) {
            const int g4 = a.gather4[it.goff + t];
            vv += (gg.w >= 0 ? cb[gg.w] : 0.0) + (g4 >= 0 ? cb[g4] : 0.0);
          }
          v[g * vs + t] = vv;
        }
      }
      __syncwarp();
      const int R = 32 / it.kl;
      const int r = it.r0 + (lane & (R - 1));
      double out[G];
      chunk_gemv_multi<G>(a.factors + it.foff, R, it.ns, v, vs, lane, out);
      if (lane < R && r < it.r1)
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (g >= nb) break;
          const int b = b0 + g;
          if (r < it.ns) a.ybuf[(int64_t)b * a.n + it.first + r] = out[g];
          else a.cbv[(int64_t)b * a.cbv_size + it.cboff + r - it.ns] = v[g * vs + r] - out[g];
        }
      __syncwarp();
    }
    __syncthreads();
  }
  for (int l = a.nlevels - 1; l >= 0; --l) {
    for (int i = a.bwd_ptr[l] + w; i < a.bwd_ptr[l + 1]; i += nwarp) {
      const SolveItem it = a.bwd_items[i];
      const int *idx = a.idx + it.goff;
      for (int t = lane; t < it.f; t += 32) {
        const int ii = t >= it.ns ? idx[t] : -1;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int b = min(b0 + g, a.nrhs - 1);
          v[g * vs + t] = t < it.ns ? a.ybuf[(int64_t)b * a.n + it.first + t] : a.x[(int64_t)b * a.ld_x + ii];
        }
      }
      __syncwarp();
      const int R = 32 / it.kl;
      const int r = it.r0 + (lane & (R - 1));
      double out[G];
      chunk_gemv_multi<G>(a.factors + it.foff, R, it.f, v, vs, lane, out);
      if (lane < R && r < it.r1) {
        const int xi = idx[r];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (g >= nb) break;
          a.x[(int64_t)(b0 + g) * a.ld_x + xi] = out[g];
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// C = A B for A (n x n, column-major), B (n x nrhs, ld ldb), split over K in S parts:
// part s writes ws[s][c][m]; FP64 tensor cores (mma.sync m8n8k4).  CTA tile 32 x 32,
// 8 warps of one 8-row m-subtile x two 8-column c-subtiles, 8 k-steps of loads in
// flight per iteration.
__global__ void __launch_bounds__(256) dense_gemm_kernel(const double *__restrict__ A, int n,
                                                         const double *__restrict__ B, int64_t ldb, int nrhs,
                                                         int kchunk, double *__restrict__ ws) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 32 + (warp >> 1) * 8;
  const int c0 = blockIdx.y * 32 + (warp & 1) * 16;
  const int kb = blockIdx.z * kchunk, ke = min(n, kb + kchunk);
  const int am = m0 + (lane >> 2), kq = lane & 3;
  const int bc0 = c0 + (lane >> 2), bc1 = c0 + 8 + (lane >> 2);
  double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int k0 = kb; k0 < ke; k0 += 32) {
    double a[8], b0[8], b1[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int kk = k0 + ks * 4 + kq;
      const bool ok = kk < ke;
      a[ks] = (ok && am < n) ? A[(int64_t)kk * n + am] : 0.0;
      b0[ks] = (ok && bc0 < nrhs) ? B[(int64_t)bc0 * ldb + kk] : 0.0;
      b1[ks] = (ok && bc1 < nrhs) ? B[(int64_t)bc1 * ldb + kk] : 0.0;
    }
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[0][0]), "+d"(d[0][1])
                   : "d"(a[ks]), "d"(b0[ks]));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[1][0]), "+d"(d[1][1])
                   : "d"(a[ks]), "d"(b1[ks]));
    }
  }
  // D fragment: row m0 + lane/4, columns c + 2*(lane%4) + {0, 1}
  const int row = m0 + (lane >> 2);
  double *w = ws + (int64_t)blockIdx.z * nrhs * n;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int col = c0 + 8 * j + 2 * kq + i;
      if (row < n && col < nrhs) w[(int64_t)col * n + row] = d[j][i];
    }
}

__global__ void dense_gemm_reduce(const double *ws, int n, int nrhs, int nsplit, double *x, int64_t ldx) {
  const int64_t tot = (int64_t)n * nrhs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int sp = 0; sp < nsplit; ++sp) v += ws[sp * tot + t];  // fixed order: deterministic
    x[(t / n) * ldx + t % n] = v;
  }
}

__global__ void identity_kernel(double *m, int n) {
  const int64_t tot = (int64_t)n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x)
    m[t] = (t / n == t % n) ? 1.0 : 0.0;
}

void NDFactor::solve(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                     cudaStream_t s) const {
  const NDPlan &p = *dev->plan;
  static const int dense_env = [] {
    const char *e = getenv("STMHD_DENSE_INV");
    return e ? atoi(e) : 1;
  }();
  if (!(dense_env && dense_ok && nbatch == 1 && p.n <= 2048 && nrhs >= 8)) {
    solve_nd(rhs, ld_rhs, x, ld_x, nrhs, s);
    return;
  }
  const int n = (int)p.n;
  if (dinv_gen != gen) {  // A^{-1} = solve(A, I), once per factorisation
    DevBuf eye((size_t)n * n * sizeof(double));
    identity_kernel<<<std::min<int64_t>(cdiv((int64_t)n * n, 256), 4096), 256, 0, s>>>(eye.as<double>(), n);
    STMHD_LAUNCH_CHECK();
    if (dinv.bytes < eye.bytes) dinv.alloc_async(eye.bytes, s);
    solve_nd(eye.as<double>(), n, dinv.as<double>(), n, n, s);
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));  // eye dies here
    dinv_gen = gen;
  }
  const int mt = (n + 31) / 32, ct = (nrhs + 31) / 32;
  int nsplit = std::max(1, std::min((2 * num_sms() + mt * ct - 1) / (mt * ct), (n + 127) / 128));
  const int kchunk = ((n + nsplit - 1) / nsplit + 31) / 32 * 32;
  nsplit = (n + kchunk - 1) / kchunk;
  const size_t wsb = (size_t)nsplit * n * nrhs * sizeof(double);
  if (gemm_ws.bytes < wsb) gemm_ws.alloc_async(wsb, s);
  dense_gemm_kernel<<<dim3(mt, ct, nsplit), 256, 0, s>>>(dinv.as<double>(), n, rhs, ld_rhs, nrhs, kchunk,
                                                          gemm_ws.as<double>());
  STMHD_LAUNCH_CHECK();
  dense_gemm_reduce<<<std::min<int64_t>(cdiv((int64_t)n * nrhs, 256), 2048), 256, 0, s>>>(gemm_ws.as<double>(), n, nrhs,
                                                                                        nsplit, x, ld_x);
  STMHD_LAUNCH_CHECK();
}

void NDFactor::solve_nd(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                        cudaStream_t s) const {
  const NDPlan &p = *dev->plan;
  require(nbatch == 1 || nrhs <= nbatch, "lu solve: more right-hand sides than factors");
  if (!bar.ptr) {
    bar.alloc_async(2 * sizeof(unsigned), s);
    STMHD_CUDA_CHECK(cudaMemsetAsync(bar.ptr, 0, 2 * sizeof(unsigned), s));
  }
  SolveArgs a{};
  a.fwd_items = dev->fwd_items.as<SolveItem>();
  a.bwd_items = dev->bwd_items.as<SolveItem>();
  a.gather3 = dev->gather3.as<int4>();
  a.gather4 = dev->gather4.as<int>();
  a.idx = dev->idx.as<int>();
  a.fwd_ptr = dev->fwd_ptr_d.as<int>();
  a.bwd_ptr = dev->bwd_ptr_d.as<int>();
  a.nlevels = p.nlevels;
  a.factors = factors.as<double>();
  a.factor_stride = nbatch == 1 ? 0 : p.factor_size;
  a.rhs = rhs;
  a.ld_rhs = ld_rhs;
  a.x = x;
  a.ld_x = ld_x;
  a.nrhs = nrhs;
  // per-factor scratch from the stream-ordered pool (factors may solve on different streams)
  const size_t need = (size_t)nrhs * (p.n + p.cbv_size) * sizeof(double);
  if (scratch.bytes < need) scratch.alloc_async(need, s);
  double *scr = scratch.as<double>();
  a.ybuf = scr;
  a.n = p.n;
  a.cbv = scr + (int64_t)nrhs * p.n;
  a.cbv_size = p.cbv_size;
  a.bar = bar.as<unsigned>();
  a.vstride = std::max(dev->max_front, 1) + 8;
  const int threads = 512;
  const size_t smem = (size_t)(threads / 32) * a.vstride * sizeof(double);
  require(smem <= 220 * 1024, "nd solve: front too large for shared memory");
  static bool attr = false;
  if (!attr) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  void *args[] = {&a};
  static const int cta_min = [] {
    const char *e = getenv("STMHD_SOLVE_CTA_MIN");
    return e ? atoi(e) : 8;
  }();
  // shared factor, many right-hand sides: G per CTA (STMHD_SOLVE_MULTI, default 4;
  // 1 = one right-hand side per CTA)
  static const int multi_env = [] {
    const char *e = getenv("STMHD_SOLVE_MULTI");
    return e ? atoi(e) : 4;
  }();
  if (nbatch == 1 && nrhs >= 2 * num_sms() && multi_env > 1) {
    int G = multi_env >= 4 ? 4 : 2;
    while (G > 1 && (size_t)(threads / 32) * G * a.vstride * sizeof(double) > 220 * 1024) G /= 2;
    if (G > 1) {
      const size_t sm = (size_t)(threads / 32) * G * a.vstride * sizeof(double);
      static bool attr3 = false;
      if (!attr3) {
        STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_cta_multi_kernel<4>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_cta_multi_kernel<2>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr3 = true;
      }
      const int nblk = (nrhs + G - 1) / G;
      if (G == 4) nd_solve_cta_multi_kernel<4><<<nblk, threads, sm, s>>>(a);
      else nd_solve_cta_multi_kernel<2><<<nblk, threads, sm, s>>>(a);
      STMHD_LAUNCH_CHECK();
      return;
    }
  }
  if (nrhs >= cta_min) {  // independent right-hand sides: one CTA each, no grid barrier
    static bool attr2 = false;
    if (!attr2) {
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            220 * 1024));
      attr2 = true;
    }
    nd_solve_cta_kernel<<<nrhs, threads, smem, s>>>(a);
    STMHD_LAUNCH_CHECK();
    return;
  }
  STMHD_CUDA_CHECK(cudaLaunchCooperativeKernel((void *)nd_solve_kernel, dim3(num_sms()), dim3(threads), args, smem, s));
  count_launch();
}

void NDFactor::sweep(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                     const SweepCoupling *cpl, int ncpl, cudaStream_t s) const {
  nd_sweep(*this, rhs, ld_rhs, x, ld_x, nrhs, cpl, ncpl, s);
}

}  // namespace stmhd
