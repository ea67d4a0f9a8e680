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

#include "nd.hpp"

namespace stmhd {

// ---------------------------------------------------------------------------
// CTA-level FP64 GEMM:  C = beta*C + alpha * A(MxK) B(KxN), row-major, global.
// 256 threads, 64x64 output tiles, 4x4 register micro-tiles, K-tiles of 16.
// ---------------------------------------------------------------------------
constexpr int GT = 64, GK = 16;

__device__ void cta_gemm(int M, int N, int K, double alpha, const double *A, int64_t lda,
                         const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                         double *sm /* 2*GT*GK doubles */) {
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
          int r = t / GK, k = t % GK;  // A tile: row r, col k
          int gr = m0 + r, gk = k0 + k;
          As[k * GT + r] = (gr < M && gk < K) ? A[gr * lda + gk] : 0.0;
          int kb = t / GT, c = t % GT;  // B tile: row kb, col c
          int gkb = k0 + kb, gc = n0 + c;
          Bs[kb * GT + c] = (gkb < K && gc < N) ? B[gkb * ldb + gc] : 0.0;
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
  const int64_t *fl_off, *fu_off, *front_off;
  const double *values;
  int64_t value_stride;
  int batch0;  // first matrix of this chunk
  double *fronts;
  int64_t front_size;
  double *factors;
  int64_t factor_size;
  int *status;
};

__global__ void __launch_bounds__(256) nd_factor_level(FactorArgs a) {
  extern __shared__ double smem[];
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  __shared__ int piv_sh;
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
      double best = -1.0;
      int bi = col;
      for (int r = col + tid; r < ns; r += nt) {
        double v = fabs(F[(int64_t)r * f + col]);
        if (v > best) { best = v; bi = r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
      __syncthreads();
      if (tid == 0) {
        double bv = red_v[0];
        int bidx = red_i[0];
        for (int w = 1; w < nt / 32; ++w)
          if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bidx)) { bv = red_v[w]; bidx = red_i[w]; }
        piv_sh = (bv > 0.0 && isfinite(bv)) ? bidx : -1;
        if (piv_sh >= 0 && piv_sh != col) {
          int t = perm[col]; perm[col] = perm[piv_sh]; perm[piv_sh] = t;
        }
      }
      __syncthreads();
      int piv = piv_sh;
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
      for (int64_t t = tid; t < (int64_t)rows * cols; t += nt) {
        int r = col + 1 + (int)(t / cols), c = col + 1 + (int)(t % cols);
        F[(int64_t)r * f + c] -= F[(int64_t)r * f + col] * F[(int64_t)col * f + c];
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
  // 4. inverse-based factors
  double *FL = a.factors + (int64_t)b * a.factor_size + a.fl_off[s];  // f x ns
  double *FU = a.factors + (int64_t)b * a.factor_size + a.fu_off[s];  // ns x f
  // L11^{-1} P: column i of L^{-1} goes to column perm[i]
  for (int i = tid; i < ns; i += nt) {
    int ci = perm[i];
    for (int r = 0; r < ns; ++r) FL[(int64_t)r * ns + ci] = (r == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int r = 1; r < ns; ++r) {
    for (int i = tid; i < r; i += nt) {
      int ci = perm[i];
      double acc = 0.0;
      for (int k = i; k < r; ++k) acc -= F[(int64_t)r * f + k] * FL[(int64_t)k * ns + ci];
      FL[(int64_t)r * ns + ci] = acc;
    }
    __syncthreads();
  }
  // G = L21 * (L11^{-1} P)
  cta_gemm(nb, ns, ns, 1.0, F + (int64_t)ns * f, f, FL, ns, 0.0, FL + (int64_t)ns * ns, ns, smem);
  // U11^{-1} into FU[:, 0:ns]
  for (int j = tid; j < ns; j += nt)
    for (int i = 0; i < ns; ++i) FU[(int64_t)i * f + j] = 0.0;
  __syncthreads();
  for (int i = ns - 1; i >= 0; --i) {
    double dinv = 1.0 / F[(int64_t)i * f + i];
    for (int j = i + tid; j < ns; j += nt) {
      double acc = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) acc -= F[(int64_t)i * f + k] * FU[(int64_t)k * f + j];
      FU[(int64_t)i * f + j] = acc * dinv;
    }
    __syncthreads();
  }
  // -U11^{-1} U12 into FU[:, ns:f]
  cta_gemm(ns, nb, ns, -1.0, FU, f, F + ns, f, 0.0, FU + ns, f, smem);
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
  front_off = upload_vec(p.front_off, s);
  cbv_off = upload_vec(p.cbv_off, s);
  std::vector<int> lsn, lptr{0};
  for (auto &l : p.level_sn) {
    lsn.insert(lsn.end(), l.begin(), l.end());
    lptr.push_back((int)lsn.size());
  }
  lvl_sn = upload_vec(lsn, s);
  lvl_ptr = upload_vec(lptr, s);
  // solve work items: row chunks of <= RCH rows
  const int RCH = 64;
  std::vector<int4> fw, bw;
  fwd_ptr.assign(1, 0);
  bwd_ptr.assign(1, 0);
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int f = p.ns[sn] + p.nb[sn];
      if (f == 0) continue;
      for (int r = 0; r < std::max(f, 1); r += RCH) fw.push_back(make_int4(sn, r, std::min(f, r + RCH), 0));
    }
    fwd_ptr.push_back((int)fw.size());
  }
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int n = p.ns[sn];
      for (int r = 0; r < n; r += RCH) bw.push_back(make_int4(sn, r, std::min(n, r + RCH), 0));
    }
    bwd_ptr.push_back((int)bw.size());
  }
  fwd_items = upload_vec(fw, s);
  bwd_items = upload_vec(bw, s);
  fwd_ptr_d = upload_vec(fwd_ptr, s);
  bwd_ptr_d = upload_vec(bwd_ptr, s);
}

void NDFactor::factor(const double *values, int64_t value_stride, cudaStream_t s) {
  const NDPlan &p = *dev->plan;
  factors.alloc((size_t)nbatch * p.factor_size * sizeof(double));
  if (!status.ptr) status.alloc(sizeof(int));
  STMHD_CUDA_CHECK(cudaMemsetAsync(status.ptr, 0, sizeof(int), s));
  // chunk the batch so the front workspace stays below ~2 GiB
  int64_t per = std::max<int64_t>(p.front_size, 1) * (int64_t)sizeof(double);
  int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(nbatch, (int64_t(2) << 30) / per));
  DevBuf fronts((size_t)chunk * per);
  size_t smem = (2 * GT * GK) * sizeof(double) + (size_t)(p.max_front + 1) * sizeof(int);
  static bool attr_set = false;
  if (smem > 48 * 1024 || !attr_set) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_factor_level, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)std::max<size_t>(smem, 48 * 1024)));
    attr_set = true;
  }
  std::vector<int> lptr{0};
  for (auto &l : p.level_sn) lptr.push_back(lptr.back() + (int)l.size());
  for (int b0 = 0; b0 < nbatch; b0 += chunk) {
    int nbch = std::min(chunk, nbatch - b0);
    for (int l = 0; l < p.nlevels; ++l) {
      int cnt = (int)p.level_sn[l].size();
      if (!cnt) continue;
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
      a.fl_off = dev->fl_off.as<int64_t>();
      a.fu_off = dev->fu_off.as<int64_t>();
      a.front_off = dev->front_off.as<int64_t>();
      a.values = values;
      a.value_stride = value_stride;
      a.batch0 = b0;
      a.fronts = fronts.as<double>();
      a.front_size = p.front_size;
      a.factors = factors.as<double>();
      a.factor_size = p.factor_size;
      a.status = status.as<int>();
      nd_factor_level<<<dim3(cnt, nbch), 256, smem, s>>>(a);
      STMHD_LAUNCH_CHECK();
    }
  }
  // keep `fronts` alive until the kernels finish
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
}

int NDFactor::check_status(cudaStream_t s) const {
  int h = 0;
  STMHD_CUDA_CHECK(cudaMemcpyAsync(&h, status.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  return h;
}

// ---------------------------------------------------------------------------
// Persistent solve kernel.
// ---------------------------------------------------------------------------
struct SolveArgs {
  const int *ns, *nb;
  const int64_t *first, *idx_off, *emap_off, *fl_off, *fu_off, *cbv_off;
  const int *idx, *child_ptr, *child_list, *emap;
  const int4 *fwd_items, *bwd_items;
  const int *fwd_ptr, *bwd_ptr;
  int nlevels;
  const double *factors;
  int64_t factor_stride;  // 0 when all right-hand sides share one factor
  const double *rhs;
  int64_t ld_rhs;
  double *x;
  int64_t ld_x;
  int nrhs;
  int sweep;  // 1: sequential slabs with coupling
  SweepCoupling cpl[2];
  int ncpl;
  double *ybuf;  // nrhs * n  (indexed by elimination position)
  int64_t n;
  double *cbv;  // nrhs * cbv_size
  int64_t cbv_size;
  unsigned *bar;  // [0] count, [1] generation
  int max_front;
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
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// Gather the front vector of supernode s for right-hand side b into v[0..f).
__device__ void gather_front(const SolveArgs &a, int s, int b, double *v) {
  const int ns = a.ns[s], nb = a.nb[s], f = ns + nb;
  const int *idx = a.idx + a.idx_off[s];
  const double *rhs = a.rhs + (int64_t)b * a.ld_rhs;
  for (int t = threadIdx.x; t < f; t += blockDim.x) {
    double val = 0.0;
    if (t < ns) {
      int i = idx[t];
      val = rhs[i];
      if (a.sweep) {
        for (int c = 0; c < a.ncpl; ++c) {
          const SweepCoupling &cp = a.cpl[c];
          int kp = b - cp.lag;
          if (kp < 0) continue;
          const double *xv = a.x + (int64_t)kp * a.ld_x;
          const double *cv = cp.val + (int64_t)(b - cp.val_shift) * cp.val_stride;
          double acc = 0.0;
          for (int e = cp.rowptr[i]; e < cp.rowptr[i + 1]; ++e) acc += cv[e] * xv[cp.col[e]];
          val += cp.coef * acc;
        }
      }
    }
    v[t] = val;
  }
  __syncthreads();
  const double *cb = a.cbv + (int64_t)b * a.cbv_size;
  for (int ci = a.child_ptr[s]; ci < a.child_ptr[s + 1]; ++ci) {
    int c = a.child_list[ci];
    int nbc = a.nb[c];
    const int *em = a.emap + a.emap_off[c];
    const double *cc = cb + a.cbv_off[c];
    for (int t = threadIdx.x; t < nbc; t += blockDim.x) v[em[t]] += cc[t];
    __syncthreads();
  }
}

__device__ void forward_item(const SolveArgs &a, int4 it, int b, double *v) {
  const int s = it.x, ns = a.ns[s];
  gather_front(a, s, b, v);
  const double *FL = a.factors + (int64_t)b * a.factor_stride + a.fl_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *y = a.ybuf + (int64_t)b * a.n + a.first[s];
  double *cb = a.cbv + (int64_t)b * a.cbv_size + a.cbv_off[s];
  for (int r = it.y + warp; r < it.z; r += nw) {
    const double *row = FL + (int64_t)r * ns;
    double acc = 0.0;
    for (int t = lane; t < ns; t += 32) acc += row[t] * v[t];
    acc = warp_sum(acc);
    if (lane == 0) {
      if (r < ns) y[r] = acc;
      else cb[r - ns] = v[r] - acc;
    }
  }
  __syncthreads();
}

__device__ void backward_item(const SolveArgs &a, int4 it, int b, double *w) {
  const int s = it.x, ns = a.ns[s], nb = a.nb[s], f = ns + nb;
  const int *idx = a.idx + a.idx_off[s];
  const double *y = a.ybuf + (int64_t)b * a.n + a.first[s];
  double *x = a.x + (int64_t)b * a.ld_x;
  for (int t = threadIdx.x; t < f; t += blockDim.x) w[t] = t < ns ? y[t] : x[idx[t]];
  __syncthreads();
  const double *FU = a.factors + (int64_t)b * a.factor_stride + a.fu_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = it.y + warp; r < it.z; r += nw) {
    const double *row = FU + (int64_t)r * f;
    double acc = 0.0;
    for (int t = lane; t < f; t += 32) acc += row[t] * w[t];
    acc = warp_sum(acc);
    if (lane == 0) x[idx[r]] = acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) nd_solve_kernel(SolveArgs a) {
  extern __shared__ double vbuf[];
  const int nblk = gridDim.x;
  const int nslab = a.sweep ? a.nrhs : 1;
  const int nb_per = a.sweep ? 1 : a.nrhs;
  for (int k = 0; k < nslab; ++k) {
    for (int l = 0; l < a.nlevels; ++l) {
      int i0 = a.fwd_ptr[l], i1 = a.fwd_ptr[l + 1];
      int64_t total = (int64_t)(i1 - i0) * nb_per;
      for (int64_t w = blockIdx.x; w < total; w += nblk) {
        int item = i0 + (int)(w / nb_per);
        int b = a.sweep ? k : (int)(w % nb_per);
        forward_item(a, a.fwd_items[item], b, vbuf);
      }
      grid_barrier(a.bar);
    }
    for (int l = a.nlevels - 1; l >= 0; --l) {
      int i0 = a.bwd_ptr[l], i1 = a.bwd_ptr[l + 1];
      int64_t total = (int64_t)(i1 - i0) * nb_per;
      for (int64_t w = blockIdx.x; w < total; w += nblk) {
        int item = i0 + (int)(w / nb_per);
        int b = a.sweep ? k : (int)(w % nb_per);
        backward_item(a, a.bwd_items[item], b, vbuf);
      }
      grid_barrier(a.bar);
    }
  }
}

static void launch_solve(SolveArgs &a, const NDDevice &dev, cudaStream_t s) {
  static DevBuf bar;
  if (!bar.ptr) {
    bar.alloc(2 * sizeof(unsigned));
    STMHD_CUDA_CHECK(cudaMemset(bar.ptr, 0, 2 * sizeof(unsigned)));
  }
  a.bar = bar.as<unsigned>();
  size_t smem = (size_t)std::max(dev.max_front, 1) * sizeof(double);
  if (smem > 48 * 1024)
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  STMHD_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nd_solve_kernel, 256, smem));
  per_sm = std::max(1, std::min(per_sm, 4));
  int grid = per_sm * num_sms();
  void *args[] = {&a};
  STMHD_CUDA_CHECK(cudaLaunchCooperativeKernel((void *)nd_solve_kernel, dim3(grid), dim3(256), args, smem, s));
}

static SolveArgs base_args(const NDDevice &dev, const double *factors, int64_t fstride) {
  const NDPlan &p = *dev.plan;
  SolveArgs a{};
  a.ns = dev.ns.as<int>();
  a.nb = dev.nb.as<int>();
  a.first = dev.first.as<int64_t>();
  a.idx_off = dev.idx_off.as<int64_t>();
  a.emap_off = dev.emap_off.as<int64_t>();
  a.fl_off = dev.fl_off.as<int64_t>();
  a.fu_off = dev.fu_off.as<int64_t>();
  a.cbv_off = dev.cbv_off.as<int64_t>();
  a.idx = dev.idx.as<int>();
  a.child_ptr = dev.child_ptr.as<int>();
  a.child_list = dev.child_list.as<int>();
  a.emap = dev.emap.as<int>();
  a.fwd_items = dev.fwd_items.as<int4>();
  a.bwd_items = dev.bwd_items.as<int4>();
  a.fwd_ptr = dev.fwd_ptr_d.as<int>();
  a.bwd_ptr = dev.bwd_ptr_d.as<int>();
  a.nlevels = p.nlevels;
  a.factors = factors;
  a.factor_stride = fstride;
  a.n = p.n;
  a.cbv_size = p.cbv_size;
  a.max_front = p.max_front;
  return a;
}

// Scratch for solves, grown on demand (per process; one stream at a time).
static double *solve_scratch(size_t doubles) {
  static DevBuf buf;
  if (buf.bytes < doubles * sizeof(double)) {
    cudaDeviceSynchronize();
    buf.alloc(doubles * sizeof(double) * 5 / 4 + 1024);
  }
  return buf.as<double>();
}

void NDFactor::solve(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                     cudaStream_t s) const {
  const NDPlan &p = *dev->plan;
  SolveArgs a = base_args(*dev, factors.as<double>(), nbatch == 1 ? 0 : p.factor_size);
  require(nbatch == 1 || nrhs <= nbatch, "lu solve: more right-hand sides than factors");
  double *scr = solve_scratch((size_t)nrhs * (p.n + p.cbv_size));
  a.rhs = rhs; a.ld_rhs = ld_rhs; a.x = x; a.ld_x = ld_x; a.nrhs = nrhs; a.sweep = 0; a.ncpl = 0;
  a.ybuf = scr;
  a.cbv = scr + (int64_t)nrhs * p.n;
  launch_solve(a, *dev, s);
}

void NDFactor::sweep(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                     const SweepCoupling *cpl, int ncpl, cudaStream_t s) const {
  const NDPlan &p = *dev->plan;
  SolveArgs a = base_args(*dev, factors.as<double>(), nbatch == 1 ? 0 : p.factor_size);
  require(ncpl <= 2, "sweep: at most two coupling terms");
  require(nbatch == 1 || nrhs <= nbatch, "sweep: more slabs than factors");
  double *scr = solve_scratch((size_t)nrhs * (p.n + p.cbv_size));
  a.rhs = rhs; a.ld_rhs = ld_rhs; a.x = x; a.ld_x = ld_x; a.nrhs = nrhs; a.sweep = 1;
  a.ncpl = ncpl;
  for (int i = 0; i < ncpl; ++i) a.cpl[i] = cpl[i];
  a.ybuf = scr;
  a.cbv = scr + (int64_t)nrhs * p.n;
  launch_solve(a, *dev, s);
}

}  // namespace stmhd
