// Cluster-resident sequential time sweep through a batch of supernodal LU
// factors (reference: solve_velocity / solve_wave / solve_potential /
// solve_pressure_cd, pkg/src/stmhd/precond.py:122-205):
//
//   x_k = A_k^{-1} ( rhs_k + sum_c coef_c C_c x_{k-lag_c} ),  k = 0..nt-1.
//
// The slabs are strictly sequential, so the sweep is latency bound.  One
// thread-block cluster runs the whole sweep in a single launch (hardware
// cluster barrier between tree levels; a software grid barrier costs 2.3 us,
// tools/bench_barrier.py).  Inside:
//  * everything runs in the nested-dissection ordering, so a supernode's own
//    unknowns are contiguous; rhs / solutions are permuted in and out by two
//    bandwidth-bound kernels around the sweep;
//  * each warp owns a contiguous range of row chunks of one supernode per
//    level (LPT balanced); a chunk's factor block [K][R] is one contiguous
//    range that the TMA engine copies into the warp's shared-memory slot
//    (cp.async.bulk + mbarrier, double buffered), overlapped with the front
//    gather; the GEMV then reads shared memory;
//  * the next slab's factors are bulk-prefetched into L2 while a slab runs;
//  * couplings are ELL tables in elimination order.
#include <algorithm>
#include <cstdlib>
#include <map>

#include "nd.hpp"

namespace stmhd {

static int env_int2(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

const NDSweepPlan &NDDevice::get_sweep_plan(int ncta, int warps, cudaStream_t s) const {
  if (sweep_plan && sweep_plan->ncta == ncta && sweep_plan->warps == warps) return *sweep_plan;
  const NDPlan &p = *plan;
  auto sp = std::make_unique<NDSweepPlan>();
  sp->ncta = ncta;
  sp->warps = warps;
  const int W = ncta * warps;
  std::vector<int> pos(p.n), iperm(p.n);
  for (int sn = 0; sn < p.nsn; ++sn)
    for (int t = 0; t < p.ns[sn]; ++t) {
      int i = p.idx[p.idx_off[sn] + t];
      pos[i] = (int)(p.first[sn] + t);
      iperm[p.first[sn] + t] = i;
    }
  std::vector<int4> g3(p.idx.size(), make_int4(-1, -1, -1, 0));
  std::vector<int> bpos(p.idx.size());
  for (int sn = 0; sn < p.nsn; ++sn) {
    int64_t o = p.idx_off[sn];
    int f = p.ns[sn] + p.nb[sn];
    for (int t = 0; t < f; ++t) bpos[o + t] = pos[p.idx[o + t]];
    for (int t = 0; t < p.ns[sn]; ++t) g3[o + t].x = (int)(p.first[sn] + t);
    int which = 0;
    for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci, ++which) {
      int c = p.child_list[ci];
      require(which < 2, "nd sweep: supernode with more than two children");
      for (int a = 0; a < p.nb[c]; ++a) {
        int ps = p.emap[p.emap_off[c] + a];
        int src = (int)(p.cbv_off[c] + a);
        if (which == 0) g3[o + ps].y = src;
        else g3[o + ps].z = src;
      }
    }
  }
  auto build_dir = [&](bool fwd, DevBuf &tasks_d, DevBuf &wptr_d) {
    std::vector<SweepTask> tasks;
    std::vector<int> wptr;
    for (int l = 0; l < p.nlevels; ++l) {
      struct SN {
        int s, rows, K, R, m;
        double cg, cc;
      };
      std::vector<SN> sns;
      for (int sn : p.level_sn[l]) {
        int f = p.ns[sn] + p.nb[sn];
        int rows = fwd ? f : p.ns[sn];
        if (rows == 0) continue;
        int K = fwd ? p.ns[sn] : f;
        int R = fwd ? p.rf[sn] : p.rb[sn];
        int m = (rows + R - 1) / R;
        // cost model in memory rounds: gather ~2, one chunk ~1 + K/(16 kl)
        sns.push_back({sn, rows, K, R, m, 2.0, 1.0 + (double)((K + 16 * (32 / R) - 1) / (16 * (32 / R)))});
      }
      double total = 0;
      for (auto &x : sns) total += x.cg + x.m * x.cc;
      struct Piece {
        int idx, c0, c1;
        double cost;
      };
      std::vector<Piece> pieces;
      for (int i = 0; i < (int)sns.size(); ++i) {
        auto &x = sns[i];
        double c = x.cg + x.m * x.cc;
        int np = 1;
        if ((int)sns.size() < W) np = std::max(1, std::min(x.m, (int)(W * c / total)));
        for (int q = 0; q < np; ++q) {
          int c0 = (int)((int64_t)x.m * q / np), c1 = (int)((int64_t)x.m * (q + 1) / np);
          if (c1 > c0) pieces.push_back({i, c0, c1, x.cg + (c1 - c0) * x.cc});
        }
      }
      std::sort(pieces.begin(), pieces.end(), [](const Piece &a, const Piece &b) { return a.cost > b.cost; });
      std::vector<std::vector<Piece>> per(W);
      std::vector<double> load(W, 0.0);
      for (auto &pc : pieces) {
        int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        per[w].push_back(pc);
        load[w] += pc.cost;
      }
      for (int w = 0; w < W; ++w) {
        wptr.push_back((int)tasks.size());
        for (auto &pc : per[w]) {
          auto &x = sns[pc.idx];
          SweepTask t{};
          t.s = x.s; t.c0 = pc.c0; t.c1 = pc.c1; t.R = x.R;
          t.ns = p.ns[x.s]; t.f = p.ns[x.s] + p.nb[x.s]; t.rows = x.rows;
          t.bsz = (int)(fwd ? p.bsz_f[x.s] : p.bsz_b[x.s]);
          t.foff = fwd ? p.fl_off[x.s] : p.fu_off[x.s];
          t.goff = p.idx_off[x.s]; t.first = p.first[x.s]; t.cboff = p.cbv_off[x.s];
          tasks.push_back(t);
        }
      }
    }
    wptr.push_back((int)tasks.size());
    tasks_d = upload_vec(tasks, s);
    wptr_d = upload_vec(wptr, s);
  };
  build_dir(true, sp->fwd_tasks, sp->fwd_wptr);
  build_dir(false, sp->bwd_tasks, sp->bwd_wptr);
  sp->g3p = upload_vec(g3, s);
  sp->bpos = upload_vec(bpos, s);
  sp->pos = upload_vec(pos, s);
  sp->iperm = upload_vec(iperm, s);
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  sweep_plan = std::move(sp);
  return *sweep_plan;
}

struct SweepCpl {
  int width;        // ELL width (max entries per row)
  const int *colp;  // [j*n + q]: permuted column of slot j of permuted row q (-1: pad)
  const int *eidx;  // original entry index of that slot (value lookup)
  const double *val;
  int64_t val_stride, val_shift;
  int lag;
  double coef;
};

struct SweepArgs {
  const SweepTask *ftask, *btask;
  const int *fwptr, *bwptr;  // per level W entries (+ one final sentinel)
  const int4 *g3p;
  const int *bpos;
  int nlevels, nw;
  int64_t n;
  const double *factors;
  int64_t fstride;
  const double *rhsp;  // nslab x n (permuted)
  double *xp;          // nslab x n (permuted)
  double *reff, *ybuf, *cbv;
  int nslab;
  SweepCpl cpl[2];
  int ncpl;
  int vstride;  // doubles per warp: gather buffer + 2 TMA slots
  int slot;     // doubles per TMA slot (largest chunk block)
  int prefetch;
  int null_work;  // diagnostics: skip all task work (barrier/loop floor)
  unsigned long long *trace;
};

__device__ __forceinline__ void sweep_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void sweep_trace(const SweepArgs &a, int &step) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[step] = t;
  }
  ++step;
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// one lane: stream `dbl` doubles from global `src` into shared `dst`, completing on `bar`
__device__ __forceinline__ void tma_load(double *dst, const double *src, int dbl, unsigned long long *bar) {
  const unsigned bytes = (unsigned)dbl * 8u;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// Issue the first (up to) two factor-chunk loads of a task.
__device__ __forceinline__ void task_begin(const SweepTask &tk, const double *F, double *const *slot,
                                           unsigned long long (*bar)[2], int wl) {
  tma_load(slot[0], F + tk.foff + (int64_t)tk.c0 * tk.bsz, tk.bsz, &bar[wl][0]);
  if (tk.c0 + 1 < tk.c1) tma_load(slot[1], F + tk.foff + (int64_t)(tk.c0 + 1) * tk.bsz, tk.bsz, &bar[wl][1]);
}

__global__ void __launch_bounds__(512, 1) nd_sweep_kernel(SweepArgs a) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long mbar[16][2];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int gw = wl * gridDim.x + blockIdx.x;  // interleaved across CTAs
  double *v = sm + wl * a.vstride;
  double *slot[2] = {v + (a.vstride - 2 * a.slot), v + (a.vstride - a.slot)};
  unsigned phase[2] = {0u, 0u};
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[wl][0])) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[wl][1])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int64_t n = a.n;
  const int L = a.nlevels;
  int step = 0;
  sweep_trace(a, step);
  // The first task of the next level step is static (descriptor and factor
  // chunks do not depend on the barrier), so it is fetched and its first TMA
  // loads are issued before the warp waits at the barrier.
  SweepTask next{};
  bool have_next = false;
  auto preload = [&](int kk, bool fwd, int l) {
    have_next = false;
    if (kk >= a.nslab) return;
    const int *wp = (fwd ? a.fwptr : a.bwptr) + (int64_t)l * a.nw;
    const int t0 = wp[gw], t1 = wp[gw + 1];
    if (t0 < t1 && !a.null_work) {
      next = (fwd ? a.ftask : a.btask)[t0];
      have_next = true;
      if (lane == 0) task_begin(next, a.factors + (int64_t)kk * a.fstride, slot, mbar, wl);
    }
  };
  preload(0, true, 0);
  for (int k = 0; k < a.nslab; ++k) {
    if (a.prefetch && a.fstride && k + 1 < a.nslab && lane == 0) {
      const char *base = reinterpret_cast<const char *>(a.factors + (int64_t)(k + 1) * a.fstride);
      const int64_t bytes = a.fstride * 8, chunk = 32 * 1024;
      for (int64_t off = (int64_t)gw * chunk; off < bytes; off += (int64_t)a.nw * chunk) {
        int64_t len = min(chunk, bytes - off) & ~int64_t(15);
        if (len > 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base + off), "r"((unsigned)len)
                       : "memory");
      }
    }
    const double *rhs = a.rhsp + (int64_t)k * n;
    double *x = a.xp + (int64_t)k * n;
    if (k > 0 && a.ncpl && !a.null_work) {
      // rhs_eff = rhs_k + sum_c coef_c C_c x_{k-lag}: permuted rows, up to two rows
      // per thread processed together (one pass), ELL slots 8 at a time
      const int64_t nth = (int64_t)a.nw * 32;
      for (int64_t p0 = (int64_t)gw * 32 + lane; p0 < n; p0 += 2 * nth) {
        const int64_t prr[2] = {p0, p0 + nth};
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c >= a.ncpl) break;
          const SweepCpl &cp = a.cpl[c];
          const int kp = k - cp.lag;
          if (kp < 0) continue;
          const double *xv = a.xp + (int64_t)kp * n;
          const double *cv = cp.val + (k - cp.val_shift) * cp.val_stride;
          double part[2] = {0.0, 0.0};
          for (int j0 = 0; j0 < cp.width; j0 += 8) {
            int ci[2][8], ei[2][8];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const bool ok = j0 + q < cp.width && prr[r] < n;
                ci[r][q] = ok ? __ldg(cp.colp + (int64_t)(j0 + q) * n + prr[r]) : -1;
                ei[r][q] = ok ? __ldg(cp.eidx + (int64_t)(j0 + q) * n + prr[r]) : 0;
              }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
              for (int q = 0; q < 8; ++q)
                if (ci[r][q] >= 0) part[r] += cv[ei[r][q]] * xv[ci[r][q]];
          }
          acc[0] += cp.coef * part[0];
          acc[1] += cp.coef * part[1];
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
          if (prr[r] < n) a.reff[prr[r]] = rhs[prr[r]] + acc[r];
      }
      sweep_barrier();
      sweep_trace(a, step);
      rhs = a.reff;
    }
    const double *F = a.factors + (int64_t)k * a.fstride;
    // ---- forward (L) levels, bottom-up ----
    for (int l = 0; l < L; ++l) {
      const int *wp = a.fwptr + (int64_t)l * a.nw;
      const int t0 = wp[gw], t1 = a.null_work ? t0 : wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        SweepTask tk;
        if (ti == t0 && have_next) {
          tk = next;
        } else {
          tk = a.ftask[ti];
          if (lane == 0) task_begin(tk, F, slot, mbar, wl);
        }
        const int4 *g = a.g3p + tk.goff;
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int4 gg[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) gg[q] = (b0 + 32 * q < tk.f) ? __ldg(g + b0 + 32 * q) : make_int4(-1, -1, -1, 0);
          double vv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            vv[q] = ((gg[q].x >= 0 ? rhs[gg[q].x] : 0.0) + (gg[q].y >= 0 ? a.cbv[gg[q].y] : 0.0)) +
                    (gg[q].z >= 0 ? a.cbv[gg[q].z] : 0.0);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (b0 + 32 * q < tk.f) v[b0 + 32 * q] = vv[q];
        }
        __syncwarp();
        const int R = tk.R;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int sl = (c - tk.c0) & 1;
          mbar_wait(&mbar[wl][sl], phase[sl]);
          phase[sl] ^= 1u;
          const double out = chunk_gemv<false>(slot[sl], R, tk.ns, v, lane);
          const int r = c * R + (lane & (R - 1));
          if (lane < R && r < tk.rows) {
            if (r < tk.ns) a.ybuf[tk.first + r] = out;
            else a.cbv[tk.cboff + r - tk.ns] = v[r] - out;
          }
          __syncwarp();
          if (lane == 0 && c + 2 < tk.c1) tma_load(slot[sl], F + tk.foff + (int64_t)(c + 2) * tk.bsz, tk.bsz, &mbar[wl][sl]);
        }
        __syncwarp();
      }
      if (l + 1 < L) preload(k, true, l + 1);
      else preload(k, false, L - 1);
      sweep_barrier();
      sweep_trace(a, step);
    }
    // ---- backward (U) levels, top-down ----
    for (int l = L - 1; l >= 0; --l) {
      const int *wp = a.bwptr + (int64_t)l * a.nw;
      const int t0 = wp[gw], t1 = a.null_work ? t0 : wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        SweepTask tk;
        if (ti == t0 && have_next) {
          tk = next;
        } else {
          tk = a.btask[ti];
          if (lane == 0) task_begin(tk, F, slot, mbar, wl);
        }
        const int *bp = a.bpos + tk.goff;
        const double *y = a.ybuf + tk.first;
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int ii[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = b0 + 32 * q;
            ii[q] = (t >= tk.ns && t < tk.f) ? __ldg(bp + t) : -1;
          }
          double vv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = b0 + 32 * q;
            vv[q] = t < tk.ns ? y[t] : (ii[q] >= 0 ? x[ii[q]] : 0.0);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (b0 + 32 * q < tk.f) v[b0 + 32 * q] = vv[q];
        }
        __syncwarp();
        const int R = tk.R;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int sl = (c - tk.c0) & 1;
          mbar_wait(&mbar[wl][sl], phase[sl]);
          phase[sl] ^= 1u;
          const double out = chunk_gemv<false>(slot[sl], R, tk.f, v, lane);
          const int r = c * R + (lane & (R - 1));
          if (lane < R && r < tk.rows) x[tk.first + r] = out;
          __syncwarp();
          if (lane == 0 && c + 2 < tk.c1) tma_load(slot[sl], F + tk.foff + (int64_t)(c + 2) * tk.bsz, tk.bsz, &mbar[wl][sl]);
        }
        __syncwarp();
      }
      if (l > 0) preload(k, false, l - 1);
      else preload(k + 1, true, 0);
      if (l > 0 || k + 1 < a.nslab) sweep_barrier();
      sweep_trace(a, step);
    }
  }
}

__global__ void permute_in_kernel(const double *rhs, int64_t ld, const int *pos, int64_t n, int nslab,
                                  double *out) {
  const int k = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[(int64_t)k * n + pos[i]] = rhs[(int64_t)k * ld + i];
}

__global__ void permute_out_kernel(const double *xp, const int *pos, int64_t n, int nslab, double *x, int64_t ld) {
  const int k = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[(int64_t)k * ld + i] = xp[(int64_t)k * n + pos[i]];
}

// Coupling matrix as an ELL table in elimination order, cached in the sweep plan.
static const std::vector<DevBuf> &permuted_ell(const NDSweepPlan &sp, const NDPlan &p, const int *rowptr,
                                               const int *col, cudaStream_t s, int *width) {
  auto &cache = sp.colp_cache;
  auto it = cache.find(col);
  if (it != cache.end()) {
    *width = (int)(it->second->at(0).bytes / sizeof(int) / std::max<int64_t>(p.n, 1));
    return *it->second;
  }
  const int64_t n = p.n;
  std::vector<int> rp(n + 1);
  STMHD_CUDA_CHECK(cudaMemcpyAsync(rp.data(), rowptr, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  const int nnz = rp[n];
  std::vector<int> cl(std::max(nnz, 1));
  if (nnz) STMHD_CUDA_CHECK(cudaMemcpy(cl.data(), col, nnz * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> pos(n), iperm(n);
  for (int sn = 0; sn < p.nsn; ++sn)
    for (int t = 0; t < p.ns[sn]; ++t) {
      int i = p.idx[p.idx_off[sn] + t];
      pos[i] = (int)(p.first[sn] + t);
      iperm[p.first[sn] + t] = i;
    }
  int w = 1;
  for (int64_t i = 0; i < n; ++i) w = std::max(w, rp[i + 1] - rp[i]);
  std::vector<int> colp((size_t)w * n, -1), eidx((size_t)w * n, 0);
  for (int64_t q = 0; q < n; ++q) {
    int io = iperm[q], j = 0;
    for (int e = rp[io]; e < rp[io + 1]; ++e, ++j) {
      colp[(size_t)j * n + q] = pos[cl[e]];
      eidx[(size_t)j * n + q] = e;
    }
  }
  auto pc = std::make_unique<std::vector<DevBuf>>();
  pc->push_back(upload_vec(colp, s));
  pc->push_back(upload_vec(eidx, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  const std::vector<DevBuf> &r = *pc;
  cache[col] = std::move(pc);
  *width = w;
  return r;
}

void nd_sweep(const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
              const SweepCoupling *cpl, int ncpl, cudaStream_t s) {
  const NDDevice &dev = *fac.dev;
  const NDPlan &p = *dev.plan;
  static const int cluster = std::max(2, std::min(16, env_int2("STMHD_SWEEP_CLUSTER", 16)));
  const int warps = 16;
  const NDSweepPlan &sp = dev.get_sweep_plan(cluster, warps, s);
  const int64_t n = p.n;
  static DevBuf scratch;
  const size_t need = ((size_t)2 * nrhs * n + 2 * n + p.cbv_size + 16) * sizeof(double);
  if (scratch.bytes < need) {
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    scratch.alloc(need * 5 / 4);
  }
  double *rhsp = scratch.as<double>();
  double *xp = rhsp + (int64_t)nrhs * n;
  double *reff = xp + (int64_t)nrhs * n;
  double *ybuf = reff + n;
  double *cbv = ybuf + n;
  permute_in_kernel<<<dim3(std::min<int64_t>(cdiv(n, 256), 256), nrhs), 256, 0, s>>>(rhs, ld_rhs, sp.pos.as<int>(), n,
                                                                                    nrhs, rhsp);
  STMHD_LAUNCH_CHECK();
  SweepArgs a{};
  a.ftask = sp.fwd_tasks.as<SweepTask>();
  a.btask = sp.bwd_tasks.as<SweepTask>();
  a.fwptr = sp.fwd_wptr.as<int>();
  a.bwptr = sp.bwd_wptr.as<int>();
  a.g3p = sp.g3p.as<int4>();
  a.bpos = sp.bpos.as<int>();
  a.nlevels = p.nlevels;
  a.nw = cluster * warps;
  a.n = n;
  a.factors = fac.factors.as<double>();
  a.fstride = fac.nbatch == 1 ? 0 : p.factor_size;
  a.rhsp = rhsp;
  a.xp = xp;
  a.reff = reff;
  a.ybuf = ybuf;
  a.cbv = cbv;
  a.nslab = nrhs;
  require(ncpl <= 2, "sweep: at most two coupling terms");
  a.ncpl = ncpl;
  for (int c = 0; c < ncpl; ++c) {
    int width = 0;
    const std::vector<DevBuf> &pcs = permuted_ell(sp, p, cpl[c].rowptr, cpl[c].col, s, &width);
    a.cpl[c].width = width;
    a.cpl[c].colp = pcs[0].as<int>();
    a.cpl[c].eidx = pcs[1].as<int>();
    a.cpl[c].val = cpl[c].val;
    a.cpl[c].val_stride = cpl[c].val_stride;
    a.cpl[c].val_shift = cpl[c].val_shift;
    a.cpl[c].lag = cpl[c].lag;
    a.cpl[c].coef = cpl[c].coef;
  }
  // per warp: gather buffer (max front, rounded to 16 doubles) + two TMA slots
  int64_t maxb = 2;
  for (int sn = 0; sn < p.nsn; ++sn) maxb = std::max({maxb, p.bsz_f[sn], p.bsz_b[sn]});
  a.slot = (int)((maxb + 15) / 16 * 16);
  a.vstride = (int)(((std::max(dev.max_front, 1) + 15) / 16) * 16 + 2 * a.slot);
  static const int prefetch = env_int2("STMHD_SWEEP_PREFETCH", 0);  // TMA streaming makes it redundant
  a.prefetch = prefetch;
  a.null_work = env_int2("STMHD_SWEEP_NULL", 0);
  const int threads = warps * 32;
  const size_t smem = (size_t)warps * a.vstride * sizeof(double);
  require(smem <= 224 * 1024, "nd sweep: front too large for shared memory");
  static bool attr = false;
  if (!attr) {
    cudaFuncAttributes fa{};
    STMHD_CUDA_CHECK(cudaFuncGetAttributes(&fa, (const void *)nd_sweep_kernel));
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_sweep_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(nd_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(227 * 1024 - fa.sharedSizeBytes)));
    attr = true;
  }
  static const int trace_on = env_int2("STMHD_SWEEP_TRACE", 0);
  DevBuf tr;
  int nsteps = 0;
  if (trace_on) {
    nsteps = 2 + nrhs * (2 * p.nlevels + 1);
    tr.alloc(nsteps * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(tr.ptr, 0, tr.bytes, s));
    a.trace = tr.as<unsigned long long>();
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
  void *args[] = {&a};
  STMHD_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void *)nd_sweep_kernel, args));
  count_launch();
  permute_out_kernel<<<dim3(std::min<int64_t>(cdiv(n, 256), 256), nrhs), 256, 0, s>>>(xp, sp.pos.as<int>(), n, nrhs, x,
                                                                                     ld_x);
  STMHD_LAUNCH_CHECK();
  if (trace_on) {
    std::vector<unsigned long long> h(nsteps);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(h.data(), tr.ptr, nsteps * 8, cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    const int per = 2 * p.nlevels + 1, base = 1 + per;
    fprintf(stderr, "[sweep] n=%lld levels=%d total=%.1f us | slab1 (us):", (long long)n, p.nlevels,
            (*std::max_element(h.begin(), h.end()) - h[0]) / 1e3);
    for (int i = 0; i < per && base + i < nsteps; ++i) fprintf(stderr, " %.2f", (h[base + i] - h[base + i - 1]) / 1e3);
    fprintf(stderr, "\n");
  }
}

}  // namespace stmhd
