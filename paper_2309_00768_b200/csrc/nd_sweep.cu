// Cluster-resident sequential time sweep through a batch of supernodal LU
// factors (reference: solve_velocity / solve_wave / solve_potential /
// solve_pressure_cd, pkg/src/stmhd/precond.py:122-205):
//
//   x_k = A_k^{-1} ( rhs_k + sum_c coef_c C_c x_{k-lag_c} ),  k = 0..nt-1.
//
// The slabs are strictly sequential, so the sweep is latency bound: one
// thread-block cluster (hardware barrier between tree levels) runs the whole
// sweep in a single launch.  Everything inside runs in the nested-dissection
// ordering: a supernode's own unknowns are a contiguous range, so front
// gathers and result stores are coalesced.  The right-hand sides are permuted
// in and the solutions permuted out by two bandwidth-bound kernels around the
// sweep.  Each warp owns a contiguous range of row chunks of one supernode
// per task, so a front is gathered once per warp; factor columns are read
// with 16 loads in flight per lane.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <map>

#include "nd.hpp"

namespace stmhd {

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
        int s, rows, K, kl, R, m;
        double cost_gather, cost_chunk;
      };
      std::vector<SN> sns;
      // lanes per row: if the level's finest chunking still leaves warps idle, use
      // 8 lanes per row (most parallel chunks, fewest rounds per chunk); otherwise
      // minimise the total number of serial load rounds
      int64_t chunks8 = 0;
      for (int sn : p.level_sn[l]) {
        int rows = fwd ? p.ns[sn] + p.nb[sn] : p.ns[sn];
        chunks8 += (rows + 3) / 4;
      }
      const bool rich = chunks8 <= W;
      for (int sn : p.level_sn[l]) {
        int f = p.ns[sn] + p.nb[sn];
        int rows = fwd ? f : p.ns[sn];
        if (rows == 0) continue;
        int K = fwd ? p.ns[sn] : f;
        int kl = 8;
        if (!rich) {
          int best = INT32_MAX;
          for (int c : {1, 2, 4, 8}) {
            int Rc = 32 / c, mc = (rows + Rc - 1) / Rc, rounds = mc * std::max(1, (K + 16 * c - 1) / (16 * c));
            if (rounds <= best) { best = rounds; kl = c; }
          }
        }
        int R = 32 / kl;
        int m = (rows + R - 1) / R;
        sns.push_back({sn, rows, K, kl, R, m, 2.0 * ((f + 255) / 256), 1.0 + (double)((K + 16 * kl - 1) / (16 * kl))});
      }
      // pieces: split big supernodes so every warp gets work, then LPT onto warps
      double total = 0;
      for (auto &x : sns) total += x.cost_gather + x.m * x.cost_chunk;
      struct Piece {
        int idx, c0, c1;
        double cost;
      };
      std::vector<Piece> pieces;
      for (int i = 0; i < (int)sns.size(); ++i) {
        auto &x = sns[i];
        double c = x.cost_gather + x.m * x.cost_chunk;
        int np = 1;
        if ((int)sns.size() < W) np = std::max(1, std::min(x.m, (int)(W * c / total)));
        for (int q = 0; q < np; ++q) {
          int c0 = (int)((int64_t)x.m * q / np), c1 = (int)((int64_t)x.m * (q + 1) / np);
          if (c1 > c0) pieces.push_back({i, c0, c1, x.cost_gather + (c1 - c0) * x.cost_chunk});
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
          t.s = x.s; t.c0 = pc.c0; t.c1 = pc.c1; t.kl = x.kl;
          t.ns = p.ns[x.s]; t.f = p.ns[x.s] + p.nb[x.s]; t.rows = x.rows;
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
  std::vector<int> sep;
  for (int sn = 0; sn < p.nsn; ++sn)
    if (p.level[sn] > 0)
      for (int t = 0; t < p.ns[sn]; ++t) sep.push_back((int)(p.first[sn] + t));
  sp->nsep = (int64_t)sep.size();
  if (sep.empty()) sep.push_back(0);
  sp->seprows = upload_vec(sep, s);
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  sweep_plan = std::move(sp);
  return *sweep_plan;
}

struct SweepCpl {
  int width;                 // ELL width (max entries per row)
  const int *colp;           // [j*n + q]: permuted column of slot j of permuted row q (-1: pad)
  const int *eidx;           // original entry index of that slot (value lookup)
  const double *val;
  int64_t val_stride, val_shift;
  int lag;
  double coef;
};

struct SweepArgs {
  const SweepTask *ftask, *btask;
  const int *fwptr, *bwptr;  // per level W entries (+ one final sentinel)
  const int4 *g3p;
  const int *bpos, *iperm;
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
  int vstride;
  int prefetch;
  unsigned long long *trace;
  unsigned long long *wtrace;  // per (step, warp): {task-load, gather, gemv} cycles (slab 1 only)
  // distributed-shared-memory layout (nd_sweep_dsm_kernel)
  int ncta, lc;        // cluster size and log2
  int64_t dsm_local;   // doubles of the distributed vectors held by each CTA
  const int *seprows;  // permuted rows of non-leaf supernodes
  int64_t nsep;
  const double *rhs_g; // unused placeholder
};

__device__ __forceinline__ void sweep_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ double sweep_gemv(const double *__restrict__ Mt, int64_t ld, int K, const double *v,
                                             int r, int kl, int kq, bool active) {
  constexpr int U = 16;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const double *col = Mt + (active ? r : 0);
  for (int t = kq; t < K; t += U * kl) {
    double m[U];
#pragma unroll
    for (int q = 0; q < U; ++q) m[q] = __ldg(col + (int64_t)min(t + q * kl, K - 1) * ld);
    asm volatile("" ::: "memory");
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int tq = t + q * kl;
      acc[q & 3] = fma(m[q], tq < K ? v[tq] : 0.0, acc[q & 3]);
    }
  }
  double out = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (int o = 1; o < kl; o <<= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
  return out;
}

__device__ __forceinline__ void sweep_trace(const SweepArgs &a, int &step) {
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[step] = t;
    if (a.wtrace) a.wtrace[step] = (unsigned long long)clock64();  // SM cycles beside the wall clock
  }
  ++step;
}

__global__ void __launch_bounds__(512, 1) nd_sweep_kernel(SweepArgs a) {
  extern __shared__ double vbuf[];
  const int lane = threadIdx.x & 31;
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;  // interleaved across CTAs
  double *v = vbuf + (threadIdx.x >> 5) * a.vstride;
  const int64_t n = a.n;
  int step = 0;
  sweep_trace(a, step);
  for (int k = 0; k < a.nslab; ++k) {
    if (a.prefetch && a.fstride && k + 1 < a.nslab && lane == 0) {
      // pull the next slab's factors into L2 while this slab runs
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
    if (k > 0 && a.ncpl) {
      // rhs_eff = rhs_k + sum_c coef_c C_c x_{k-lag}: one permuted row per thread,
      // ELL slots loaded 8 at a time (coalesced across threads)
      const int64_t nth = (int64_t)a.nw * 32;
      for (int64_t pr = (int64_t)gw * 32 + lane; pr < n; pr += nth) {
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c >= a.ncpl) break;
          const SweepCpl &cp = a.cpl[c];
          const int kp = k - cp.lag;
          if (kp < 0) continue;
          const double *xv = a.xp + (int64_t)kp * n;
          const double *cv = cp.val + (k - cp.val_shift) * cp.val_stride;
          double part = 0.0;
          for (int j0 = 0; j0 < cp.width; j0 += 8) {
            int ci[8], ei[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const bool ok = j0 + q < cp.width;
              ci[q] = ok ? cp.colp[(int64_t)(j0 + q) * n + pr] : -1;
              ei[q] = ok ? cp.eidx[(int64_t)(j0 + q) * n + pr] : 0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (ci[q] >= 0) part += cv[ei[q]] * xv[ci[q]];
          }
          acc += cp.coef * part;
        }
        a.reff[pr] = rhs[pr] + acc;
      }
      sweep_barrier();
      sweep_trace(a, step);
      rhs = a.reff;
    }
    const double *F = a.factors + (int64_t)k * a.fstride;
    // ---- forward (L) levels, bottom-up ----
    for (int l = 0; l < a.nlevels; ++l) {
      const int *wp = a.fwptr + (int64_t)l * a.nw;  // nw entries per level + final sentinel
      const int t0 = wp[gw], t1 = wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        long long c0 = clock64();
        const SweepTask tk = a.ftask[ti];
        const int4 *g = a.g3p + tk.goff;
        long long c1 = clock64() + (tk.f & 0);
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int4 gg[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) gg[q] = (b0 + 32 * q < tk.f) ? g[b0 + 32 * q] : make_int4(-1, -1, -1, 0);
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
        long long c2 = clock64();
        const int kl = tk.kl, kq = lane % kl, R = 32 / kl;
        const double *FLT = F + tk.foff;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int r = c * R + lane / kl;
          const bool act = r < tk.rows;
          const double out = sweep_gemv(FLT, tk.f, tk.ns, v, r, kl, kq, act);
          if (act && kq == 0) {
            if (r < tk.ns) a.ybuf[tk.first + r] = out;
            else a.cbv[tk.cboff + r - tk.ns] = v[r] - out;
          }
        }
        __syncwarp();
        if (a.wtrace && k == 1 && lane == 0) {
          long long c3 = clock64();
          unsigned long long *w = a.wtrace + ((int64_t)step * a.nw + gw) * 3;
          w[0] += c1 - c0;
          w[1] += c2 - c1;
          w[2] += c3 - c2;
        }
      }
      sweep_barrier();
      sweep_trace(a, step);
    }
    // ---- backward (U) levels, top-down ----
    for (int l = a.nlevels - 1; l >= 0; --l) {
      const int *wp = a.bwptr + (int64_t)l * a.nw;
      const int t0 = wp[gw], t1 = wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        const SweepTask tk = a.btask[ti];
        const int *bp = a.bpos + tk.goff;
        const double *y = a.ybuf + tk.first;
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int ii[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = b0 + 32 * q;
            ii[q] = (t >= tk.ns && t < tk.f) ? bp[t] : -1;
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
        const int kl = tk.kl, kq = lane % kl, R = 32 / kl;
        const double *FUT = F + tk.foff;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int r = c * R + lane / kl;
          const bool act = r < tk.rows;
          const double out = sweep_gemv(FUT, tk.ns, tk.f, v, r, kl, kq, act);
          if (act && kq == 0) x[tk.first + r] = out;
        }
        __syncwarp();
      }
      if (l > 0 || k + 1 < a.nslab) sweep_barrier();
      sweep_trace(a, step);
    }
  }
}


// ---------------------------------------------------------------------------
// Distributed-shared-memory variant.  All vectors exchanged between tree
// levels inside a slab (x ring for the lag-1/2 couplings, y, effective rhs,
// update vectors) live in the cluster's shared memory, interleaved across the
// CTAs in 32-element blocks; only read-only data (factors, rhs, coupling
// matrices) is read from global memory, and each slab's solution is written
// back once.  The level barrier then never waits on global stores.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

struct Dsm {
  double *rb[16];
  int cmask, shift;
  __device__ __forceinline__ double *at(int64_t e) const {
    return rb[(e >> 5) & cmask] + (((e >> shift) << 5) | (e & 31));
  }
};

// sum_c coef_c (C_c x_{k-lag_c})[pr] with the x ring in distributed shared memory
__device__ __forceinline__ double coupling_row(const SweepArgs &a, const Dsm &dm, int k, int64_t pr) {
  const int64_t n = a.n;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (c >= a.ncpl) break;
    const SweepCpl &cp = a.cpl[c];
    const int kp = k - cp.lag;
    if (kp < 0) continue;
    const int64_t xl = (int64_t)(kp % 3) * n;
    const double *cv = cp.val + (k - cp.val_shift) * cp.val_stride;
    double part = 0.0;
    for (int j0 = 0; j0 < cp.width; j0 += 8) {
      int ci[8], ei[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool ok = j0 + q < cp.width;
        ci[q] = ok ? cp.colp[(int64_t)(j0 + q) * n + pr] : -1;
        ei[q] = ok ? cp.eidx[(int64_t)(j0 + q) * n + pr] : 0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (ci[q] >= 0) part += cv[ei[q]] * *dm.at(xl + ci[q]);
    }
    acc += cp.coef * part;
  }
  return acc;
}

__global__ void __launch_bounds__(512, 1) nd_sweep_dsm_kernel(SweepArgs a) {
  extern __shared__ double sm[];
  __shared__ Dsm D;
  cg::cluster_group cl = cg::this_cluster();
  double *local = sm;
  if (threadIdx.x < a.ncta) D.rb[threadIdx.x] = cl.map_shared_rank(local, (int)threadIdx.x);
  if (threadIdx.x == 0) {
    D.cmask = a.ncta - 1;
    D.shift = 5 + a.lc;
  }
  const int lane = threadIdx.x & 31;
  const int gw = (threadIdx.x >> 5) * gridDim.x + blockIdx.x;
  double *v = sm + a.dsm_local + (threadIdx.x >> 5) * a.vstride;
  const int64_t n = a.n;
  const int64_t XR = 0, Y = 3 * n, RF = 4 * n, CB = 5 * n;
  cl.sync();
  const Dsm &dm = D;  // remote bases stay in shared memory (no local-memory copy)
  int step = 0;
  sweep_trace(a, step);
  const int64_t nth = (int64_t)a.nw * 32;
  const int64_t tid = (int64_t)gw * 32 + lane;
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
    const int64_t xs = XR + (int64_t)(k % 3) * n;
    const bool coupled = k > 0 && a.ncpl;
    const double *F = a.factors + (int64_t)k * a.fstride;
    for (int l = 0; l < a.nlevels; ++l) {
      if (l == 0 && k > 0) {
        // previous slab's solution to global memory; coupling rows of the
        // separators (leaves compute their own rows' coupling in their gather)
        const int64_t xprev = XR + (int64_t)((k - 1) % 3) * n;
        double *xout = a.xp + (int64_t)(k - 1) * n;
        for (int64_t pr = tid; pr < n; pr += nth) xout[pr] = *dm.at(xprev + pr);
        if (coupled)
          for (int64_t q = tid; q < a.nsep; q += nth) {
            const int64_t pr = a.seprows[q];
            *dm.at(RF + pr) = rhs[pr] + coupling_row(a, dm, k, pr);
          }
      }
      const int *wp = a.fwptr + (int64_t)l * a.nw;
      const int t0 = wp[gw], t1 = wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        const SweepTask tk = a.ftask[ti];
        const int4 *g = a.g3p + tk.goff;
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int4 gg[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) gg[q] = (b0 + 32 * q < tk.f) ? g[b0 + 32 * q] : make_int4(-1, -1, -1, 0);
          double vv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            double r = 0.0;
            if (gg[q].x >= 0) {
              if (!coupled) r = rhs[gg[q].x];
              else if (l == 0) r = rhs[gg[q].x] + coupling_row(a, dm, k, gg[q].x);
              else r = *dm.at(RF + gg[q].x);
            }
            const double c1 = gg[q].y >= 0 ? *dm.at(CB + gg[q].y) : 0.0;
            const double c2 = gg[q].z >= 0 ? *dm.at(CB + gg[q].z) : 0.0;
            vv[q] = (r + c1) + c2;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (b0 + 32 * q < tk.f) v[b0 + 32 * q] = vv[q];
        }
        __syncwarp();
        const int kl = tk.kl, kq = lane % kl, R = 32 / kl;
        const double *FLT = F + tk.foff;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int r = c * R + lane / kl;
          const bool act = r < tk.rows;
          const double out = sweep_gemv(FLT, tk.f, tk.ns, v, r, kl, kq, act);
          if (act && kq == 0) {
            if (r < tk.ns) *dm.at(Y + tk.first + r) = out;
            else *dm.at(CB + tk.cboff + r - tk.ns) = v[r] - out;
          }
        }
        __syncwarp();
      }
      cl.sync();
      sweep_trace(a, step);
    }
    for (int l = a.nlevels - 1; l >= 0; --l) {
      const int *wp = a.bwptr + (int64_t)l * a.nw;
      const int t0 = wp[gw], t1 = wp[gw + 1];
      for (int ti = t0; ti < t1; ++ti) {
        const SweepTask tk = a.btask[ti];
        const int *bp = a.bpos + tk.goff;
        for (int b0 = lane; b0 < tk.f; b0 += 256) {
          int ii[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = b0 + 32 * q;
            ii[q] = (t >= tk.ns && t < tk.f) ? bp[t] : -1;
          }
          double vv[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int t = b0 + 32 * q;
            vv[q] = t < tk.ns ? *dm.at(Y + tk.first + t) : (ii[q] >= 0 ? *dm.at(xs + ii[q]) : 0.0);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (b0 + 32 * q < tk.f) v[b0 + 32 * q] = vv[q];
        }
        __syncwarp();
        const int kl = tk.kl, kq = lane % kl, R = 32 / kl;
        const double *FUT = F + tk.foff;
        for (int c = tk.c0; c < tk.c1; ++c) {
          const int r = c * R + lane / kl;
          const bool act = r < tk.rows;
          const double out = sweep_gemv(FUT, tk.ns, tk.f, v, r, kl, kq, act);
          if (act && kq == 0) *dm.at(xs + tk.first + r) = out;
        }
        __syncwarp();
      }
      cl.sync();
      sweep_trace(a, step);
    }
  }
  // last slab's solution
  {
    const int k = a.nslab - 1;
    const int64_t xs = XR + (int64_t)(k % 3) * n;
    double *xout = a.xp + (int64_t)k * n;
    for (int64_t pr = tid; pr < n; pr += nth) xout[pr] = *dm.at(xs + pr);
  }
  cl.sync();  // keep every CTA's shared memory alive until all remote reads are done
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

__global__ void perm_cols_kernel(const int *col, int64_t nnz, const int *pos, int *colp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    colp[e] = pos[col[e]];
}

static int env_int2(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Coupling matrix re-indexed to the elimination order (rows and columns),
// cached in the sweep plan: {rowptr_p (n+1), colp (nnz), eidx (nnz)}.
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
  // ELL in elimination order, entry slot j of row q at [j*n + q]; padding: col -1
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
  // scratch: rhs_p, x_p (nrhs*n), reff, ybuf (n), cbv (cbv_size)
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
  a.iperm = sp.iperm.as<int>();
  a.nlevels = p.nlevels;
  a.nw = cluster * warps;
  a.n = n;
  a.factors = fac.factors.as<double>();
  a.fstride = fac.nbatch == 1 ? 0 : p.factor_size;
  if (env_int2("STMHD_SWEEP_SAMEFACTOR", 0)) a.fstride = 0;  // diagnostics only
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
  a.vstride = std::max(dev.max_front, 1) + 8;
  static const int prefetch = env_int2("STMHD_SWEEP_PREFETCH", 1);
  a.prefetch = prefetch;
  const int threads = warps * 32;
  // distributed vectors: x ring (3n) + y (n) + rhs_eff (n) + update vectors
  a.ncta = cluster;
  a.lc = 0;
  while ((1 << a.lc) < cluster) ++a.lc;
  const int64_t V = 5 * n + p.cbv_size;
  const int64_t blocks = (V + 32 * cluster - 1) / (32 * cluster);
  a.dsm_local = blocks * 32;
  a.seprows = sp.seprows.as<int>();
  a.nsep = sp.nsep;
  size_t smem = (size_t)warps * a.vstride * sizeof(double);
  static const int dsm_env = env_int2("STMHD_SWEEP_DSMEM", 0);
  const bool use_dsm = dsm_env && (cluster & (cluster - 1)) == 0 &&
                       smem + a.dsm_local * sizeof(double) + 1024 <= 226 * 1024;
  if (use_dsm) smem += a.dsm_local * sizeof(double);
  require(smem <= 227 * 1024, "nd sweep: front too large for shared memory");
  const void *kern = use_dsm ? (const void *)nd_sweep_dsm_kernel : (const void *)nd_sweep_kernel;
  static bool attr = false;
  if (!attr) {
    for (const void *kf : {(const void *)nd_sweep_kernel, (const void *)nd_sweep_dsm_kernel}) {
      cudaFuncAttributes fa{};
      STMHD_CUDA_CHECK(cudaFuncGetAttributes(&fa, kf));
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(227 * 1024 - fa.sharedSizeBytes)));
    }
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
  DevBuf wtr;
  if (trace_on) {
    wtr.alloc((size_t)nsteps * a.nw * 3 * 8);
    STMHD_CUDA_CHECK(cudaMemsetAsync(wtr.ptr, 0, wtr.bytes, s));
    a.wtrace = wtr.as<unsigned long long>();
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
  STMHD_CUDA_CHECK(cudaLaunchKernelExC(&cfg, kern, args));
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
    std::vector<unsigned long long> w((size_t)nsteps * a.nw * 3);
    STMHD_CUDA_CHECK(cudaMemcpy(w.data(), wtr.ptr, w.size() * 8, cudaMemcpyDeviceToHost));
    {
      int last = 0;
      for (int i = 0; i < nsteps; ++i)
        if (h[i]) last = i;
      fprintf(stderr, "[sweep] SM clock during sweep: %.0f MHz\n", 1e3 * (double)(w[last] - w[0]) / (double)(h[last] - h[0]));
    }
    fprintf(stderr, "[sweep] fwd levels slab1, slowest warp cycles {task,gather,gemv} (busy):");
    for (int l = 0; l < p.nlevels; ++l) {
      int st = base - 1 + l;  // forward level l of slab 1 ran with step index base-1+l
      unsigned long long best[3] = {0, 0, 0};
      int busy = 0;
      for (int q = 0; q < a.nw; ++q) {
        const unsigned long long *x = &w[((size_t)st * a.nw + q) * 3];
        if (x[0] + x[1] + x[2]) ++busy;
        if (x[0] + x[1] + x[2] > best[0] + best[1] + best[2]) { best[0] = x[0]; best[1] = x[1]; best[2] = x[2]; }
      }
      fprintf(stderr, " [%llu,%llu,%llu x%d]", best[0], best[1], best[2], busy);
    }
    fprintf(stderr, "\n");
  }
}

}  // namespace stmhd
