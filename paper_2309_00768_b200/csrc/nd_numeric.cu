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
  // 4. inverse-based factors, stored column-major so the solve GEMVs read
  //    coalesced columns with one thread per output row:
  //    FLT[t*f + r] = FL[r][t] (FL = [L11^-1 P ; L21 L11^-1 P], f x ns)
  //    FUT[t*ns + r] = FU[r][t] (FU = [U11^-1 | -U11^-1 U12], ns x f)
  double *FLT = a.factors + (int64_t)b * a.factor_size + a.fl_off[s];
  double *FUT = a.factors + (int64_t)b * a.factor_size + a.fu_off[s];
  // L11^{-1} P: column i of L^{-1} goes to column perm[i]
  for (int i = tid; i < ns; i += nt) {
    int ci = perm[i];
    for (int r = 0; r < ns; ++r) FLT[(int64_t)ci * f + r] = (r == i) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int r = 1; r < ns; ++r) {
    for (int i = tid; i < r; i += nt) {
      int ci = perm[i];
      double acc = 0.0;
      for (int k = i; k < r; ++k) acc -= F[(int64_t)r * f + k] * FLT[(int64_t)ci * f + k];
      FLT[(int64_t)ci * f + r] = acc;
    }
    __syncthreads();
  }
  // G^T = (L11^{-1} P)^T L21^T  ->  FLT[c*f + ns + i]
  cta_gemm(ns, nb, ns, 1.0, FLT, f, F + (int64_t)ns * f, f, 0.0, FLT + ns, f, smem, false, true);
  // U11^{-1}: FUT[j*ns + i] for i <= j
  for (int j = tid; j < ns; j += nt)
    for (int i = 0; i < ns; ++i) FUT[(int64_t)j * ns + i] = 0.0;
  __syncthreads();
  for (int i = ns - 1; i >= 0; --i) {
    double dinv = 1.0 / F[(int64_t)i * f + i];
    for (int j = i + tid; j < ns; j += nt) {
      double acc = (i == j) ? 1.0 : 0.0;
      for (int k = i + 1; k <= j; ++k) acc -= F[(int64_t)i * f + k] * FUT[(int64_t)j * ns + k];
      FUT[(int64_t)j * ns + i] = acc * dinv;
    }
    __syncthreads();
  }
  // (-U11^{-1} U12)^T = -U12^T U11^{-T}  ->  FUT[(ns+j)*ns + i]
  cta_gemm(nb, ns, ns, -1.0, F + ns, f, FUT, ns, 0.0, FUT + (int64_t)ns * ns, ns, smem, true, false);
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
  // solve work items: a warp computes 32/kl rows, kl lanes share each row's K loop
  auto klanes = [](int K) { return K > 96 ? 8 : (K > 8 ? 4 : 1); };
  std::vector<SolveItem> fw, bw;
  fwd_ptr.assign(1, 0);
  bwd_ptr.assign(1, 0);
  auto item = [&](int sn, int r0, int r1, int kl, int64_t foff) {
    SolveItem it{};
    it.s = sn; it.r0 = r0; it.r1 = r1; it.kl = kl;
    it.ns = p.ns[sn]; it.f = p.ns[sn] + p.nb[sn];
    it.foff = foff; it.goff = p.idx_off[sn]; it.first = p.first[sn]; it.cboff = p.cbv_off[sn];
    return it;
  };
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int f = p.ns[sn] + p.nb[sn];
      if (f == 0) continue;
      int kl = klanes(p.ns[sn]), rows = 32 / kl;
      for (int r = 0; r < f; r += rows) fw.push_back(item(sn, r, std::min(f, r + rows), kl, p.fl_off[sn]));
    }
    fwd_ptr.push_back((int)fw.size());
  }
  for (int l = 0; l < p.nlevels; ++l) {
    for (int sn : p.level_sn[l]) {
      int n = p.ns[sn], f = p.ns[sn] + p.nb[sn];
      int kl = klanes(f), rows = 32 / kl;
      for (int r = 0; r < n; r += rows) bw.push_back(item(sn, r, std::min(n, r + rows), kl, p.fu_off[sn]));
    }
    bwd_ptr.push_back((int)bw.size());
  }
  // flat forward gather table
  std::vector<int4> g3(p.idx.size(), make_int4(-1, -1, -1, 0));
  for (int sn = 0; sn < p.nsn; ++sn) {
    int64_t o = p.idx_off[sn];
    for (int t = 0; t < p.ns[sn]; ++t) g3[o + t].x = p.idx[o + t];
    int which = 0;
    for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci, ++which) {
      int c = p.child_list[ci];
      require(which < 2, "nd solve: supernode with more than two children");
      for (int a = 0; a < p.nb[c]; ++a) {
        int pos = p.emap[p.emap_off[c] + a];
        int src = (int)(p.cbv_off[c] + a);
        if (which == 0) g3[o + pos].y = src;
        else g3[o + pos].z = src;
      }
    }
  }
  gather3 = upload_vec(g3, s);
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
// Persistent solve kernel: warp-granular work items.
//
// A work item is (supernode, 32-row chunk); one warp gathers the front vector
// into its own shared-memory slice and computes its rows with one lane per
// row over the column-major factor (coalesced, unrolled loads).  Level steps
// are separated by a barrier: the hardware cluster barrier when the whole
// kernel is one thread-block cluster (time sweeps: latency bound), or a
// software grid barrier for batched solves over many right-hand sides.
// ---------------------------------------------------------------------------
struct SolveArgs {
  const int *ns, *nb;
  const int64_t *first, *idx_off, *emap_off, *fl_off, *fu_off, *cbv_off;
  const int *idx, *child_ptr, *child_list, *emap;
  const SolveItem *fwd_items, *bwd_items;
  const int4 *gather3;
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
  int vstride;    // doubles of shared memory per warp
  double *reff;   // sweep: effective right-hand side of the current slab (n)
  unsigned long long *trace;  // optional: globaltimer after every level step
  int prefetch;
  unsigned long long *wtrace;  // optional: per (step, warp) {gather, gemv} cycles of slab 1
  int wtrace_nw;
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

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <bool CLUSTER>
__device__ __forceinline__ void level_barrier(unsigned *bar) {
  if (CLUSTER)
    cluster_barrier();
  else
    grid_barrier(bar);
}

__device__ __forceinline__ void trace_step(const SolveArgs &a, int &step) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[step] = t;
  }
  ++step;
}

// Gather the front vector of a work item's supernode for right-hand side b
// into v[0..f): one round for the flat gather table, one for the values
// (right-hand side + up to two child update vectors, fixed summation order).
__device__ __forceinline__ void warp_gather(const SolveArgs &a, const double *rhs, const SolveItem &it,
                                            const double *cb, double *v) {
  const int lane = threadIdx.x & 31;
  const int4 *g = a.gather3 + it.goff;
  for (int t0 = lane; t0 < it.f; t0 += 128) {
    int4 gg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + 32 * q;
      gg[q] = t < it.f ? g[t] : make_int4(-1, -1, -1, 0);
    }
    double vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double r = gg[q].x >= 0 ? rhs[gg[q].x] : 0.0;
      const double c1 = gg[q].y >= 0 ? cb[gg[q].y] : 0.0;
      const double c2 = gg[q].z >= 0 ? cb[gg[q].z] : 0.0;
      vv[q] = (r + c1) + c2;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (t0 + 32 * q < it.f) v[t0 + 32 * q] = vv[q];
  }
  __syncwarp();
}

// Rows r0.. of a column-major block: lane = (row sub-index, k-lane).  Loads
// are issued 16 deep per lane so one item costs a couple of memory latencies.
__device__ __forceinline__ double warp_gemv(const double *__restrict__ Mt, int64_t ld, int K, const double *v,
                                            int r, int kl, int kq, bool active) {
  constexpr int U = 16;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (K > 0) {
    const double *col = Mt + (active ? r : 0);
    for (int t = kq; t < K; t += U * kl) {
      double m[U];
      // unpredicated loads with clamped addresses: all U issue back to back
#pragma unroll
      for (int q = 0; q < U; ++q) m[q] = __ldg(col + (int64_t)min(t + q * kl, K - 1) * ld);
      asm volatile("" ::: "memory");
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int tq = t + q * kl;
        acc[q & 3] = fma(m[q], tq < K ? v[tq] : 0.0, acc[q & 3]);
      }
    }
  }
  double out = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (int o = 1; o < kl; o <<= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
  return out;
}

__device__ void warp_forward(const SolveArgs &a, const double *rhs, const SolveItem &it, int b, double *v,
                             unsigned long long *wt = nullptr) {
  double *cb = a.cbv + (int64_t)b * a.cbv_size;
  long long c0 = clock64();
  warp_gather(a, rhs, it, cb, v);
  long long c1 = clock64();
  const int lane = threadIdx.x & 31, kl = it.kl, kq = lane % kl;
  const int r = it.r0 + lane / kl;
  const bool active = r < it.r1;
  const double *FLT = a.factors + (int64_t)b * a.factor_stride + it.foff;
  const double out = warp_gemv(FLT, it.f, it.ns, v, r, kl, kq, active);
  if (active && kq == 0) {
    if (r < it.ns) a.ybuf[(int64_t)b * a.n + it.first + r] = out;
    else cb[it.cboff + r - it.ns] = v[r] - out;
  }
  __syncwarp();
  if (wt && (threadIdx.x & 31) == 0) {
    long long c2 = clock64();
    wt[0] += c1 - c0;
    wt[1] += c2 - c1;
  }
}

__device__ void warp_backward(const SolveArgs &a, const SolveItem &it, int b, double *w) {
  const int lane = threadIdx.x & 31;
  const int ns = it.ns, f = it.f;
  const int *idx = a.idx + it.goff;
  const double *y = a.ybuf + (int64_t)b * a.n + it.first;
  double *x = a.x + (int64_t)b * a.ld_x;
  const int kl = it.kl, kq = lane % kl;
  const int r = it.r0 + lane / kl;
  const bool active = r < it.r1;
  const int xr = (active && kq == 0) ? idx[r] : 0;
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
  const double *FUT = a.factors + (int64_t)b * a.factor_stride + it.foff;
  const double out = warp_gemv(FUT, ns, f, w, r, kl, kq, active);
  if (active && kq == 0) x[xr] = out;
  __syncwarp();
}

// rhs_eff = rhs_k + sum_c coef_c C_c x_(k-lag_c)  over all rows (4 lanes per row)
__device__ void sweep_rhs(const SolveArgs &a, int k, double *out, int gw, int nw) {
  const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
  const double *rhs = a.rhs + (int64_t)k * a.ld_rhs;
  for (int64_t i0 = (int64_t)gw * 8; i0 < a.n; i0 += (int64_t)nw * 8) {
    const int64_t i = i0 + g;
    double acc = 0.0;
    if (i < a.n) {
      for (int c = 0; c < a.ncpl; ++c) {
        const SweepCoupling &cp = a.cpl[c];
        const int kp = k - cp.lag;
        if (kp < 0) continue;
        const double *xv = a.x + (int64_t)kp * a.ld_x;
        const double *cv = cp.val + (int64_t)(k - cp.val_shift) * cp.val_stride;
        double part = 0.0;
        const int e0 = cp.rowptr[i], e1 = cp.rowptr[i + 1];
#pragma unroll 4
        for (int e = e0 + gl; e < e1; e += 4) part += cv[e] * xv[cp.col[e]];
        acc += cp.coef * part;
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (i < a.n && gl == 0) out[i] = rhs[i] + acc;
  }
}

// Pull a byte range into L2 with bulk prefetches (fire and forget).
__device__ __forceinline__ void l2_prefetch(const void *base, int64_t bytes, int gw, int nw) {
  const int64_t chunk = 64 * 1024;
  const char *p = static_cast<const char *>(base);
  if ((threadIdx.x & 31) != 0) return;
  for (int64_t off = (int64_t)gw * chunk; off < bytes; off += (int64_t)nw * chunk) {
    int64_t len = bytes - off < chunk ? bytes - off : chunk;
    len &= ~int64_t(15);
    if (len > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p + off), "r"((unsigned)len) : "memory");
  }
}

template <bool CLUSTER>
__global__ void __launch_bounds__(512, 1) nd_solve_kernel(SolveArgs a) {
  extern __shared__ double vbuf[];
  const int warps_per_cta = blockDim.x >> 5;
  // interleave warps across CTAs so small levels spread over every SM
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  const int nw = gridDim.x * warps_per_cta;
  double *v = vbuf + (threadIdx.x >> 5) * a.vstride;
  const int nslab = a.sweep ? a.nrhs : 1;
  const int nb_per = a.sweep ? 1 : a.nrhs;
  const int64_t fbytes = a.factor_stride * (int64_t)sizeof(double);
  int step = 0;
  trace_step(a, step);
  if (a.sweep && a.factor_stride && a.prefetch) l2_prefetch(a.factors, fbytes, gw, nw);
  for (int k = 0; k < nslab; ++k) {
    const double *rhs = a.rhs;
    if (a.sweep) {
      if (a.prefetch && a.factor_stride && k + 1 < nslab) l2_prefetch(a.factors + (int64_t)(k + 1) * a.factor_stride, fbytes, gw, nw);
      rhs = a.rhs + (int64_t)k * a.ld_rhs;
      if (a.ncpl && k > 0) {
        sweep_rhs(a, k, a.reff, gw, nw);
        level_barrier<CLUSTER>(a.bar);
        trace_step(a, step);
        rhs = a.reff;
      }
    }
    for (int l = 0; l < a.nlevels; ++l) {
      const int i0 = a.fwd_ptr[l], i1 = a.fwd_ptr[l + 1];
      const int64_t total = (int64_t)(i1 - i0) * nb_per;
      for (int64_t w = gw; w < total; w += nw) {
        const int item = i0 + (int)(w / nb_per);
        const int b = a.sweep ? k : (int)(w % nb_per);
        const SolveItem it = a.fwd_items[item];
        unsigned long long *wt = (a.wtrace && k == 1) ? a.wtrace + ((int64_t)step * a.wtrace_nw + gw) * 2 : nullptr;
        warp_forward(a, a.sweep ? rhs : a.rhs + (int64_t)b * a.ld_rhs, it, b, v, wt);
      }
      level_barrier<CLUSTER>(a.bar);
      trace_step(a, step);
    }
    for (int l = a.nlevels - 1; l >= 0; --l) {
      const int i0 = a.bwd_ptr[l], i1 = a.bwd_ptr[l + 1];
      const int64_t total = (int64_t)(i1 - i0) * nb_per;
      for (int64_t w = gw; w < total; w += nw) {
        const int item = i0 + (int)(w / nb_per);
        const int b = a.sweep ? k : (int)(w % nb_per);
        const SolveItem it = a.bwd_items[item];
        warp_backward(a, it, b, v);
      }
      if (l > 0 || k + 1 < nslab) level_barrier<CLUSTER>(a.bar);
      trace_step(a, step);
    }
  }
}

static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

static void launch_solve(SolveArgs &a, const NDDevice &dev, cudaStream_t s) {
  static DevBuf bar;
  if (!bar.ptr) {
    bar.alloc(2 * sizeof(unsigned));
    STMHD_CUDA_CHECK(cudaMemset(bar.ptr, 0, 2 * sizeof(unsigned)));
  }
  a.bar = bar.as<unsigned>();
  a.vstride = std::max(dev.max_front, 1);
  // sweeps: one cluster (hardware barrier); batched solves: whole GPU
  static const int cluster = std::max(1, std::min(16, env_int("STMHD_SWEEP_CLUSTER", 16)));
  const bool use_cluster = a.sweep && cluster > 1;
  int threads = 512;
  size_t smem = (size_t)(threads / 32) * a.vstride * sizeof(double);
  while (smem > 200 * 1024 && threads > 128) {
    threads /= 2;
    smem = (size_t)(threads / 32) * a.vstride * sizeof(double);
  }
  require(smem <= 227 * 1024, "nd solve: front too large for shared memory");
  static const int trace_on = env_int("STMHD_SWEEP_TRACE", 0);
  static const int prefetch_on = env_int("STMHD_SWEEP_PREFETCH", 1);
  a.prefetch = prefetch_on;
  static const int same_factor = env_int("STMHD_SWEEP_SAMEFACTOR", 0);  // diagnostics only
  if (same_factor) a.factor_stride = 0;
  DevBuf tr;
  int nsteps = 0;
  DevBuf wtr;
  int wnw = 0;
  if (trace_on && a.sweep) {
    nsteps = 2 + a.nrhs * (2 * a.nlevels + 1);
    tr.alloc(nsteps * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(tr.ptr, 0, nsteps * sizeof(unsigned long long), s));
    a.trace = tr.as<unsigned long long>();
    wnw = (use_cluster ? cluster : num_sms()) * (threads / 32);
    wtr.alloc((size_t)nsteps * wnw * 2 * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(wtr.ptr, 0, wtr.bytes, s));
    a.wtrace = wtr.as<unsigned long long>();
    a.wtrace_nw = wnw;
  }
  void *args[] = {&a};
  if (use_cluster) {
    static bool attr = false;
    if (!attr) {
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    STMHD_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void *)nd_solve_kernel<true>, args));
    count_launch();
  } else {
    static bool attr = false;
    if (!attr) {
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_solve_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr = true;
    }
    int per_sm = 0;
    STMHD_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nd_solve_kernel<false>, threads, smem));
    per_sm = std::max(1, std::min(per_sm, 1));
    int grid = per_sm * num_sms();
    STMHD_CUDA_CHECK(cudaLaunchCooperativeKernel((void *)nd_solve_kernel<false>, dim3(grid), dim3(threads), args, smem, s));
    count_launch();
  }
  if (a.trace) {
    std::vector<unsigned long long> h(nsteps);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(h.data(), tr.ptr, nsteps * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    // per-step durations of slab 1 (steady state): coupling, forward levels, backward levels
    int per = 2 * a.nlevels + 1;
    int base = 1 + per;  // after slab 0 (slab 0 has no coupling step)
    fprintf(stderr, "[trace] n=%lld levels=%d total=%.1f us | slab1 steps (us):", (long long)a.n, a.nlevels,
            (*std::max_element(h.begin(), h.end()) - h[0]) / 1e3);
    for (int i = 0; i < per && base + i < nsteps; ++i)
      fprintf(stderr, " %.2f", (h[base + i] - h[base + i - 1]) / 1e3);
    fprintf(stderr, "\n");
    std::vector<unsigned long long> w((size_t)nsteps * wnw * 2);
    STMHD_CUDA_CHECK(cudaMemcpy(w.data(), wtr.ptr, w.size() * 8, cudaMemcpyDeviceToHost));
    fprintf(stderr, "[trace] forward steps of slab 1: max-warp gather/gemv cycles (busy warps):");
    for (int i = 0; i < per && base + i < nsteps; ++i) {
      unsigned long long mg = 0, mm = 0;
      int busy = 0;
      for (int q = 0; q < wnw; ++q) {
        unsigned long long g = w[((size_t)(base + i - 1) * wnw + q) * 2], m = w[((size_t)(base + i - 1) * wnw + q) * 2 + 1];
        if (g + m) ++busy;
        if (g + m > mg + mm) { mg = g; mm = m; }
      }
      if (busy) fprintf(stderr, " [%llu/%llu x%d]", mg, mm, busy);
    }
    fprintf(stderr, "\n");
  }
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
  a.fwd_items = dev.fwd_items.as<SolveItem>();
  a.bwd_items = dev.bwd_items.as<SolveItem>();
  a.gather3 = dev.gather3.as<int4>();
  a.fwd_ptr = dev.fwd_ptr_d.as<int>();
  a.bwd_ptr = dev.bwd_ptr_d.as<int>();
  a.nlevels = p.nlevels;
  a.factors = factors;
  a.factor_stride = fstride;
  a.n = p.n;
  a.cbv_size = p.cbv_size;
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
  static const int legacy = env_int("STMHD_SWEEP_LEGACY", 0);
  if (!legacy) {
    nd_sweep(*this, rhs, ld_rhs, x, ld_x, nrhs, cpl, ncpl, s);
    return;
  }
  const NDPlan &p = *dev->plan;
  SolveArgs a = base_args(*dev, factors.as<double>(), nbatch == 1 ? 0 : p.factor_size);
  require(ncpl <= 2, "sweep: at most two coupling terms");
  require(nbatch == 1 || nrhs <= nbatch, "sweep: more slabs than factors");
  double *scr = solve_scratch((size_t)nrhs * (p.n + p.cbv_size) + p.n);
  a.rhs = rhs; a.ld_rhs = ld_rhs; a.x = x; a.ld_x = ld_x; a.nrhs = nrhs; a.sweep = 1;
  a.reff = scr + (int64_t)nrhs * (p.n + p.cbv_size);
  a.ncpl = ncpl;
  for (int i = 0; i < ncpl; ++i) a.cpl[i] = cpl[i];
  a.ybuf = scr;
  a.cbv = scr + (int64_t)nrhs * p.n;
  launch_solve(a, *dev, s);
}

}  // namespace stmhd
