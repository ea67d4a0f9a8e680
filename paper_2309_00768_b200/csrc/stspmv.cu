// Space-time SpMV in the sliced-ELL layout of stspmv.hpp.
//
// The space-time operators apply ONE sparsity pattern to every time slab: the
// Jacobian's per-slab f_u|z_j|z_a / y|f_a rows with the shared couplings
// (spacetime.py:131-153) and configuration 5's F_k / -M/dt bidiagonal.  A warp owns a
// slice of 32 length-sorted rows (thread = row) for one slab; every value and column
// load is a coalesced 256-byte warp access, consecutive warps stream consecutive
// slices, and blockIdx.y walks the slabs, so the per-slab value stream is read
// front to back while that slab's x stays L1/L2 resident.  Four independent
// accumulators keep four value loads and four x gathers in flight per thread.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <numeric>

#include "capi_common.hpp"
#include "stspmv.hpp"


namespace stmhd {

struct SellArgs {
  int nslices, nt;
  const int4 *slice;
  const int2 *lane;  // {row, lenA | lenB << 16}
  const int *col_a, *col_b;
  const double *val_b;
  const double *sell;
  int64_t sell_a;
  double alpha_a, alpha_b;
  const double *x;
  int64_t xs;
  double *y;
  int64_t ys;
};

// S slabs per thread share every column (and coupling) load: per batch of 4 entries
// a thread has 4 column loads and 4*S value loads + 4*S x gathers in flight.
template <int S, int B, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) sell_spmv_kernel(SellArgs a) {
  const int sidx = blockIdx.x * WARPS + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (sidx >= a.nslices) return;
  const int k0 = blockIdx.y * S;
  const int ns = min(S, a.nt - k0);
  const int4 sl = a.slice[sidx];
  const int2 li = a.lane[sidx * 32 + lane];
  const int lenA = li.y & 0xffff, lenB = li.y >> 16;
  const double *va = a.sell + (int64_t)k0 * a.sell_a + (int64_t)sl.z * 32 + lane;
  const int *ca = a.col_a + (int64_t)sl.z * 32 + lane;
  double sa[S][2];
#pragma unroll
  for (int q = 0; q < S; ++q) sa[q][0] = sa[q][1] = 0.0;
  // slabs past the end re-read the last slab (valid addresses, results dropped), so
  // every load of a batch is issued back to back without branches
  const double *vq[S];
  const double *xq[S];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    const int kq = min(q, ns - 1);
    vq[q] = va + (int64_t)kq * a.sell_a;
    xq[q] = a.x + (int64_t)(k0 + kq) * a.xs;
  }
  // column indices run one batch ahead of the value loads and x gathers, so the
  // col -> x dependency does not serialise two memory latencies per batch
  int c[B];
#pragma unroll
  for (int i = 0; i < B; ++i) c[i] = i < lenA ? ca[i * 32] : 0;
  for (int j = 0; j < sl.x; j += B) {
    bool on[B];
    int cn[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      on[i] = j + i < lenA;
      cn[i] = (j + B + i < lenA) ? ca[(j + B + i) * 32] : 0;
    }
    double v[S][B], xv[S][B];
#pragma unroll
    for (int q = 0; q < S; ++q)
#pragma unroll
      for (int i = 0; i < B; ++i) {
        v[q][i] = on[i] ? vq[q][(j + i) * 32] : 0.0;
        xv[q][i] = on[i] ? xq[q][c[i]] : 0.0;
      }
#pragma unroll
    for (int q = 0; q < S; ++q)
#pragma unroll
      for (int i = 0; i < B; ++i) sa[q][i & 1] = fma(v[q][i], xv[q][i], sa[q][i & 1]);
#pragma unroll
    for (int i = 0; i < B; ++i) c[i] = cn[i];
  }
  double sb[S];
#pragma unroll
  for (int q = 0; q < S; ++q) sb[q] = 0.0;
  if (sl.y) {
    const int *cb = a.col_b + (int64_t)sl.w * 32 + lane;
    const double *vb = a.val_b + (int64_t)sl.w * 32 + lane;
    for (int j = 0; j < lenB; ++j) {
      const int c = cb[j * 32];
      const double bv = vb[j * 32];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const int64_t xi = (int64_t)(k0 + min(q, ns - 1)) * a.xs + c;
        if (xi >= 0) sb[q] = fma(bv, a.x[xi], sb[q]);
      }
    }
  }
  if (li.x >= 0) {
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (q < ns) a.y[(int64_t)(k0 + q) * a.ys + li.x] = a.alpha_a * (sa[q][0] + sa[q][1]) + a.alpha_b * sb[q];
  }
}

__global__ void sell_relayout_kernel(const int *src, int64_t n, int nt, const double *csr, int64_t stride,
                                     double *sell) {
  const int k = blockIdx.y;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int q = src[e];
    sell[(int64_t)k * n + e] = q >= 0 ? csr[(int64_t)k * stride + q] : 0.0;
  }
}

void StSpmvPlan::build(int n, const int *rpA, const int *colA, const int *rpB, const int *colB, const double *valB,
                       int col_b_shift, cudaStream_t s) {
  require(!rpB || (colB && valB), "stspmv: the coupling needs columns and values");
  nrows = n;
  has_b = rpB != nullptr;
  nnz_a = rpA[n];
  nnz_b = has_b ? rpB[n] : 0;
  auto la = [&](int r) { return rpA[r + 1] - rpA[r]; };
  auto lb = [&](int r) { return has_b ? rpB[r + 1] - rpB[r] : 0; };
  // rows sorted by length (A, then B) inside windows of kStSigma rows
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  for (int w0 = 0; w0 < n; w0 += kStSigma) {
    const int w1 = std::min(n, w0 + kStSigma);
    std::stable_sort(order.begin() + w0, order.begin() + w1, [&](int x, int y) {
      return la(x) != la(y) ? la(x) > la(y) : lb(x) > lb(y);
    });
  }
  nslices = (n + 31) / 32;
  std::vector<int4> sl(nslices);
  std::vector<int2> ln((size_t)nslices * 32, make_int2(-1, 0));
  int64_t oa = 0, ob = 0;
  for (int si = 0; si < nslices; ++si) {
    int wa = 0, wb = 0;
    for (int l = 0; l < 32 && si * 32 + l < n; ++l) {
      const int r = order[si * 32 + l];
      require(la(r) < 65536 && lb(r) < 32768, "stspmv: row too long");
      wa = std::max(wa, la(r));
      wb = std::max(wb, lb(r));
      ln[(size_t)si * 32 + l] = make_int2(r, la(r) | lb(r) << 16);
    }
    require(oa / 32 < INT32_MAX && ob / 32 < INT32_MAX, "stspmv: pattern too large");
    sl[si] = make_int4(wa, wb, (int)(oa / 32), (int)(ob / 32));
    oa += 32LL * wa;
    ob += 32LL * wb;
  }
  sell_a = std::max<int64_t>(oa, 1);
  sell_b = std::max<int64_t>(ob, 1);
  std::vector<int> sa(sell_a, -1), ca(sell_a, 0), cb(sell_b, 0);
  std::vector<double> vb(sell_b, 0.0);
  for (int si = 0; si < nslices; ++si)
    for (int l = 0; l < 32 && si * 32 + l < n; ++l) {
      const int r = order[si * 32 + l];
      for (int j = 0; j < la(r); ++j) {
        const int64_t e = ((int64_t)sl[si].z + j) * 32 + l;
        sa[e] = rpA[r] + j;
        ca[e] = colA[rpA[r] + j];
      }
      for (int j = 0; j < lb(r); ++j) {
        const int64_t e = ((int64_t)sl[si].w + j) * 32 + l;
        cb[e] = colB[rpB[r] + j] + col_b_shift;
        vb[e] = valB[rpB[r] + j];
      }
    }
  slice = upload_vec(sl, s);
  rowmap = upload_vec(ln, s);
  src_a = upload_vec(sa, s);
  col_a = upload_vec(ca, s);
  col_b = upload_vec(cb, s);
  val_b = upload_vec(vb, s);
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors die here
}

void StSpmvPlan::relayout(int nt, const double *csr, int64_t val_stride, double *sell, cudaStream_t s) const {
  if (nt <= 0) return;
  const unsigned gx = (unsigned)std::min<int64_t>(cdiv(sell_a, 256), std::max(1, 4 * num_sms() / nt + 1));
  sell_relayout_kernel<<<dim3(gx, nt), 256, 0, s>>>(src_a.as<int>(), sell_a, nt, csr, val_stride, sell);
  STMHD_LAUNCH_CHECK();
}

void StSpmvPlan::apply(int nt, const double *sell, double alpha_a, double alpha_b, const double *x, int64_t xs,
                       double *y, int64_t ys, cudaStream_t s) const {
  if (nt <= 0 || nrows == 0) return;
  require(nt <= 65535, "stspmv: at most 65535 slabs per launch");
  SellArgs a{};
  a.nslices = nslices;
  a.slice = slice.as<int4>();
  a.lane = rowmap.as<int2>();
  a.col_a = col_a.as<int>();
  a.col_b = col_b.as<int>();
  a.val_b = val_b.as<double>();
  a.sell = sell;
  a.sell_a = sell_a;
  a.alpha_a = alpha_a;
  a.alpha_b = has_b ? alpha_b : 0.0;
  a.x = x;
  a.xs = xs;
  a.y = y;
  a.ys = ys;
  a.nt = nt;
  // slabs per thread x entries per batch (STMHD_SELL_SB = 10*S + B for experiments)
  static const int sb = [] {
    const char *e = getenv("STMHD_SELL_SB");
    return e ? atoi(e) : 0;
  }();
  // measured (r01, 128-thread CTAs): 2 slabs x 4 entries per thread is best for both
  // J.v (rows ~45 entries; C3 62 % of HBM) and C5 (rows ~14; 62 %)
  const int S = sb ? sb / 10 : 2, B = sb ? sb % 10 : 4;
  static const int wenv = [] {
    const char *e = getenv("STMHD_SELL_WARPS");
    return e ? atoi(e) : 4;  // r01 sweep: 128-thread CTAs (finer tail, more CTAs/SM) 0.40 -> 0.34 ms at C3
  }();
  auto launch = [&](auto kern, int s_, int w_) {
    kern<<<dim3(cdiv(nslices, w_), cdiv(nt, s_)), w_ * 32, 0, s>>>(a);
  };
  if (wenv == 4) {
    if (S == 1 && B == 8) launch(sell_spmv_kernel<1, 8, 4>, 1, 4);
    else if (S == 1 && B == 2) launch(sell_spmv_kernel<1, 2, 4>, 1, 4);
    else if (S == 1) launch(sell_spmv_kernel<1, 4, 4>, 1, 4);
    else if (S == 2 && B == 2) launch(sell_spmv_kernel<2, 2, 4>, 2, 4);
    else if (S == 2) launch(sell_spmv_kernel<2, 4, 4>, 2, 4);
    else launch(sell_spmv_kernel<4, 4, 4>, 4, 4);
  } else {
    if (S == 1 && B == 8) launch(sell_spmv_kernel<1, 8, 8>, 1, 8);
    else if (S == 1 && B == 2) launch(sell_spmv_kernel<1, 2, 8>, 1, 8);
    else if (S == 1) launch(sell_spmv_kernel<1, 4, 8>, 1, 8);
    else if (S == 2 && B == 2) launch(sell_spmv_kernel<2, 2, 8>, 2, 8);
    else if (S == 2) launch(sell_spmv_kernel<2, 4, 8>, 2, 8);
    else launch(sell_spmv_kernel<4, 4, 8>, 4, 8);
  }
  STMHD_LAUNCH_CHECK();
}

}  // namespace stmhd

// ---- C-ABI ----

struct stmhd_spmv_s {
  stmhd::StSpmvPlan plan;
};

using namespace stmhd;

extern "C" {

int stmhd_spmv_create(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *c_rowptr,
                      const int32_t *c_col, const double *c_val, int32_t c_col_shift, void *stream,
                      stmhd_spmv_s **out) {
  CAPI_BEGIN
  require(n >= 1 && n < INT32_MAX && rowptr && col && out && (!c_rowptr || (c_col && c_val)),
          "stmhd_spmv_create: bad arguments");
  auto h = std::make_unique<stmhd_spmv_s>();
  h->plan.build((int)n, rowptr, col, c_rowptr, c_col, c_val, c_col_shift, (cudaStream_t)stream);
  *out = h.release();
  CAPI_END
}

int stmhd_spmv_destroy(stmhd_spmv_s *plan) {
  CAPI_BEGIN
  delete plan;
  CAPI_END
}

int64_t stmhd_spmv_sell_size(stmhd_spmv_s *plan) { return plan ? plan->plan.sell_a : 0; }

int stmhd_spmv_relayout(stmhd_spmv_s *plan, void *stream, int nt, const double *vals, int64_t val_stride,
                        double *sell) {
  CAPI_BEGIN
  require(plan && vals && sell && nt >= 0, "stmhd_spmv_relayout: bad arguments");
  plan->plan.relayout(nt, vals, val_stride, sell, (cudaStream_t)stream);
  CAPI_END
}

int stmhd_spmv_apply(stmhd_spmv_s *plan, void *stream, int nt, const double *sell, double alpha, double c_coef,
                     const double *x, double *y) {
  CAPI_BEGIN
  require(plan && sell && x && y && nt >= 0, "stmhd_spmv_apply: bad arguments");
  const int64_t n = plan->plan.nrows;
  plan->plan.apply(nt, sell, alpha, c_coef, x, n, y, n, (cudaStream_t)stream);
  CAPI_END
}

}  // extern "C"
