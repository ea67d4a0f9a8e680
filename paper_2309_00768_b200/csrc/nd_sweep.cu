// Cluster-resident sequential time sweep through a batch of supernodal LU
// factors (reference: solve_velocity / solve_wave / solve_potential /
// solve_pressure_cd, pkg/src/stmhd/precond.py:122-205):
//
//   x_k = A_k^{-1} ( rhs_k + sum_c coef_c C_c src_c ),  k = 0..nt-1,
//
// src_c = x_{k-lag} (lag 1, 2) or another sweep's x_k (pipelined launch).
// The slabs are strictly sequential, so the sweep is latency bound.  One
// 16-CTA thread-block cluster runs a whole sweep in one launch (hardware cluster
// barrier; a software grid barrier costs 2.3 us, tools/bench_barrier.py).  Per slab:
//  1. coupling program (CTA-local): the coupled rhs of this CTA's rows, all loads
//     of a row batch in flight (sources through a shared-memory pointer table);
//  2. subtree forward: the bottom of the nested-dissection tree is cut into <= 16
//     balanced subtrees, one per CTA; their levels are separated by __syncthreads
//     and their vectors live in that CTA's shared memory;
//  3. dense top: x_T = K z_T, K = (A^{-1})_TT built once per factorisation
//     (topk_kernel), one GEMV step instead of 2 * (top levels) cluster steps;
//  4. subtree backward (CTA-local);  5. (pipelined launch) post-slab program and
//     per-slab release flag for the consuming sweep.
// Every warp walks a static item sequence (front tables, factor chunks, K rows)
// held in shared memory; a TMA ring (cp.async.bulk + mbarrier, two slots) keeps
// its next items in flight across task, level and slab boundaries.  Vectors run in
// the nested-dissection ordering, permuted in and out around the launch.
#include <algorithm>
#include <array>
#include <climits>
#include <cstdlib>
#include <map>

#include "nd.hpp"

namespace stmhd {

// TMA ring slots per warp (compile-time: -DSTMHD_RING=n)
#ifndef STMHD_RING
#define STMHD_RING 2
#endif
constexpr int kRing = STMHD_RING;

static int env_int2(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}

// Top supernode for the dense-top construction (postorder).
struct TopSN {
  int ns, nb, first, goff;  // columns, boundary, first position, front table offset
  int fl_off, fu_off, rf, rb, bszf, bszb;  // chunk layout of FL (f x ns) and FU (ns x f)
  int tcb_off;              // offset of its update block in the construction scratch
  int nchild, child0;       // top children in tchild[child0 .. child0 + nchild)
  int pad[3];
};

// Shared memory per warp: gather buffer (largest front it gathers, rounded to 16
// doubles) + two TMA slots of the largest ring item.
static int sweep_slot(const NDPlan &p) {
  int64_t maxb = 2;
  for (int sn = 0; sn < p.nsn; ++sn) maxb = std::max({maxb, p.bsz_f[sn], p.bsz_b[sn]});
  return (int)((maxb + 15) / 16 * 16);
}

// mode ladder (first that fits shared memory wins): 0 subtrees + dense top + resident
// subtree tables, 1 subtrees + dense top, 2 subtrees + tree top, 3 all levels cluster-wide
const NDSweepPlan &NDDevice::get_sweep_plan(int ncta, int warps, int64_t smem_budget, cudaStream_t s,
                                            int mode) const {
  const bool flat = mode >= 3;
  const int slot_sz = sweep_slot(*plan);
  const int64_t vstride_max = (std::max(max_front, 1) + 15) / 16 * 16 + kRing * slot_sz;
  const int64_t sub_budget = smem_budget - (int64_t)warps * vstride_max;  // conservative (largest front)
  for (const auto &c : sweep_plans)
    if (c->ncta == ncta && c->warps == warps) return *c;
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
  // child update slots per front position: children 0, 1 -> y, z; children 2, 3 of an
  // amalgamated (wide) supernode -> w and the parallel table g4
  std::vector<int4> g3(p.idx.size(), make_int4(-1, -1, -1, -1));
  std::vector<int> g4(std::max<size_t>(p.idx.size(), 1), -1);
  std::vector<int> bpos(p.idx.size());
  for (int sn = 0; sn < p.nsn; ++sn) {
    int64_t o = p.idx_off[sn];
    int f = p.ns[sn] + p.nb[sn];
    for (int t = 0; t < f; ++t) bpos[o + t] = pos[p.idx[o + t]];
    for (int t = 0; t < p.ns[sn]; ++t) g3[o + t].x = (int)(p.first[sn] + t);
    int which = 0;
    for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci, ++which) {
      int c = p.child_list[ci];
      require(which < 4, "nd sweep: supernode with more than four children");
      for (int a = 0; a < p.nb[c]; ++a) {
        int ps = p.emap[p.emap_off[c] + a];
        int src = (int)(p.cbv_off[c] + a);
        if (which == 0) g3[o + ps].y = src;
        else if (which == 1) g3[o + ps].z = src;
        else if (which == 2) g3[o + ps].w = src;
        else g4[o + ps] = src;
      }
    }
  }

  // ---- split the tree: a frontier of <= ncta subtrees (one per CTA) + the top ----
  // Greedy: start from the tree roots and keep splitting the frontier node with the
  // most subtree work (factor doubles) while the frontier still fits the CTAs, so
  // the subtrees are balanced even when the tree is not.
  std::vector<double> swork(p.nsn, 0.0);
  for (int sn = 0; sn < p.nsn; ++sn) {  // postorder: children first
    swork[sn] += 2.0 * (double)(p.ns[sn] + p.nb[sn]) * p.ns[sn] + 64.0;
    if (p.parent[sn] >= 0) swork[p.parent[sn]] += swork[sn];
  }
  static const int sub_env = [] {
    const char *e = getenv("STMHD_SWEEP_SUBTREES");
    return e ? atoi(e) : 1;
  }();
  int D = (sub_env && !flat) ? 1 : 0;  // 1: subtree phase in use
  // subtrees per sweep: one per CTA in cluster mode; in grid mode (ncta > 16) fewer
  // subtrees than CTAs keep the top small enough for the dense K (all CTAs stream K
  // and the coupling; CTAs without a subtree idle through the subtree phases)
  // (STMHD_SWEEP_GRID_SUBTREES; default: 64 for a stage of the grid-family pipelined
  // launch -- two more CTA-local levels and two fewer grid-wide band levels per
  // direction than one subtree per CTA, C4/C3 P_T^-1 -8 % -- and one per CTA for a
  // whole-GPU single sweep, where 64 measured 30 % slower on C5)
  static const int maxsub_env = env_int2("STMHD_SWEEP_GRID_SUBTREES", 0);
  // the largest power of two <= the CTA count (a balanced frontier of the
  // nested-dissection tree; 96 or 112 subtrees split it unevenly and measured 30 %
  // slower): 64 for a 116-CTA stage of the pipelined launch, 128 for a whole-GPU sweep
  int pow2 = 1;
  while (pow2 * 2 <= ncta) pow2 *= 2;
  const int maxsub_dflt = pow2;
  const int max_sub = ncta > 16 ? std::min(maxsub_env > 0 ? maxsub_env : maxsub_dflt, ncta) : ncta;
  std::vector<int> frontier, uniform;
  if (D) {
    for (int sn = 0; sn < p.nsn; ++sn)
      if (p.parent[sn] < 0) frontier.push_back(sn);
    for (;;) {
      int best = -1;
      for (int i = 0; i < (int)frontier.size(); ++i) {
        const int sn = frontier[i];
        const int nc = p.child_ptr[sn + 1] - p.child_ptr[sn];
        if (nc == 0 || (int)frontier.size() - 1 + nc > max_sub) continue;
        if (best < 0 || swork[sn] > swork[frontier[best]]) best = i;
      }
      if (best < 0) break;
      const int sn = frontier[best];
      frontier.erase(frontier.begin() + best);
      for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci) frontier.push_back(p.child_list[ci]);
      bool same = true;
      for (int f : frontier) same = same && p.level[f] == p.level[frontier[0]];
      if (same) uniform = frontier;
    }
    // amalgamated trees widen by four per level in places: a frontier that ends between
    // two levels has subtrees of different depths, and the slab time is the deepest
    // one's -- keep the last frontier whose subtrees all have the same height
    if (p.nwide > 0 && uniform.size() > 1) frontier = uniform;
    if ((int)frontier.size() > ncta || frontier.size() <= 1) D = 0;
    std::sort(frontier.begin(), frontier.end());
  }
  // subtree membership (owner CTA; -1 = top); falls back to an all-top schedule
  // when the subtree vectors exceed shared memory
  std::vector<int> owner, roots;
  std::vector<int64_t> info;
  int64_t maxlen = 0, maxcb = 0;
  for (;;) {
    owner.assign(p.nsn, -1);
    roots.clear();
    info.assign(4 * (size_t)ncta, 0);
    maxlen = maxcb = 0;
    if (D > 0) {
      roots = frontier;
      for (int r = 0; r < (int)roots.size(); ++r) owner[roots[r]] = r;
      for (int sn = p.nsn - 1; sn >= 0; --sn)  // parents first
        if (owner[sn] < 0 && p.parent[sn] >= 0 && owner[p.parent[sn]] >= 0) owner[sn] = owner[p.parent[sn]];
    }
    // per-CTA subtree ranges (a subtree is contiguous in postorder/elimination order)
    std::vector<int64_t> lo(roots.size(), INT64_MAX), hi(roots.size(), 0), cblo(roots.size(), INT64_MAX),
        cbhi(roots.size(), 0);
    for (int sn = 0; sn < p.nsn; ++sn) {
      int o = owner[sn];
      if (o < 0) continue;
      lo[o] = std::min(lo[o], p.first[sn]);
      hi[o] = std::max(hi[o], p.first[sn] + p.ns[sn]);
      if (sn != roots[o] && p.nb[sn] > 0) {
        cblo[o] = std::min(cblo[o], p.cbv_off[sn]);
        cbhi[o] = std::max(cbhi[o], p.cbv_off[sn] + p.nb[sn]);
      }
    }
    for (int r = 0; r < (int)roots.size(); ++r) {
      if (cblo[r] == INT64_MAX) cblo[r] = cbhi[r] = 0;
      info[4 * r + 0] = lo[r];
      info[4 * r + 1] = hi[r] - lo[r];
      info[4 * r + 2] = cblo[r];
      info[4 * r + 3] = cbhi[r] - cblo[r];
      maxlen = std::max(maxlen, hi[r] - lo[r]);
      maxcb = std::max(maxcb, cbhi[r] - cblo[r]);
    }
    if (D == 0 || 3 * maxlen + maxcb <= sub_budget) break;  // ys, xs, rhs_s + cbs
    D = 0;
  }
  if (D == 0) maxlen = maxcb = 0;

  struct SN {
    int s, rows, K, R, m;
    double cg, cc;
  };
  auto make_sn = [&](int sn, bool fwd, SN &x) {
    int f = p.ns[sn] + p.nb[sn];
    int rows = fwd ? f : p.ns[sn];
    if (rows == 0) return false;
    int K = fwd ? p.ns[sn] : f;
    int R = fwd ? p.rf[sn] : p.rb[sn];
    x = {sn, rows, K, R, (rows + R - 1) / R, 2.0, 1.0 + (double)((K + 16 * (32 / R) - 1) / (16 * (32 / R)))};
    return true;
  };
  // front tables as TMA ring items: forward g3 (int4 per entry, 16-byte aligned at
  // idx_off) and a 16-byte aligned copy of bpos per supernode; a table rides in the
  // ring ahead of its task's chunks when it fits a slot (slot = largest chunk block)
  int64_t slot_dbl = 2;
  for (int sn = 0; sn < p.nsn; ++sn) slot_dbl = std::max({slot_dbl, p.bsz_f[sn], p.bsz_b[sn]});
  slot_dbl = (slot_dbl + 15) / 16 * 16;
  static const int tables_env = env_int2("STMHD_SWEEP_TABLES", 1);
  std::vector<int> boff(p.nsn), bpos4;
  for (int sn = 0; sn < p.nsn; ++sn) {
    const int f = p.ns[sn] + p.nb[sn];
    boff[sn] = (int)bpos4.size();
    bpos4.insert(bpos4.end(), bpos.begin() + p.idx_off[sn], bpos.begin() + p.idx_off[sn] + f);
    while (bpos4.size() % 4) bpos4.push_back(0);
  }
  if (bpos4.empty()) bpos4.push_back(0);
  auto make_task = [&](const SN &x, int c0, int c1, bool fwd, bool cb_global) {
    const int64_t foff = fwd ? p.fl_off[x.s] : p.fu_off[x.s];
    const int f = p.ns[x.s] + p.nb[x.s];
    require(foff + (int64_t)x.m * (fwd ? p.bsz_f[x.s] : p.bsz_b[x.s]) < INT32_MAX && p.idx_off[x.s] < INT32_MAX &&
                p.cbv_off[x.s] < INT32_MAX && f < 32768 && x.m < 32768,
            "nd sweep: factor too large for the compact task layout");
    SweepTask t{};
    t.foff = (int)foff;
    t.goff = (int)p.idx_off[x.s];
    t.first = (int)p.first[x.s];
    t.cboff = (int)p.cbv_off[x.s];
    t.c0 = (short)c0;
    t.c1 = (short)c1;
    t.ns = (short)p.ns[x.s];
    t.f = (short)f;
    t.rows = (short)x.rows;
    t.R = (unsigned char)x.R;
    t.flags = cb_global ? 1 : 0;
    if (fwd && p.wide(x.s)) t.flags |= 64;  // gather with the two extra child slots
    t.bsz = (int)(fwd ? p.bsz_f[x.s] : p.bsz_b[x.s]);
    const int64_t tbl_dbl = fwd ? 2LL * f : ((int64_t)f + 3) / 4 * 2;  // table size in doubles
    if (tables_env && tbl_dbl <= slot_dbl) t.flags |= fwd ? 4 : (4 | 8);
    if (!fwd) t.cboff = boff[x.s];  // backward tasks: offset of the aligned bpos copy
    return t;
  };
  // LPT of a set of supernodes onto `nw` warps; pieces split big supernodes
  auto schedule = [&](const std::vector<SN> &sns, int nw, bool fwd, std::vector<std::vector<SweepTask>> &per,
                      const std::vector<char> &cbg) {
    per.assign(nw, {});
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
      if ((int)sns.size() < nw) np = std::max(1, std::min(x.m, (int)(nw * c / total)));
      for (int q = 0; q < np; ++q) {
        int c0 = (int)((int64_t)x.m * q / np), c1 = (int)((int64_t)x.m * (q + 1) / np);
        if (c1 > c0) pieces.push_back({i, c0, c1, x.cg + (c1 - c0) * x.cc});
      }
    }
    std::sort(pieces.begin(), pieces.end(), [](const Piece &a, const Piece &b) { return a.cost > b.cost; });
    std::vector<double> load(nw, 0.0);
    for (auto &pc : pieces) {
      int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      per[w].push_back(make_task(sns[pc.idx], pc.c0, pc.c1, fwd, cbg[pc.idx]));
      load[w] += pc.cost;
    }
  };
  // top part: levels (heights) that contain top supernodes, ascending
  // top nodes scheduled by their height within the top tree (frontier subtrees
  // are complete before the top phase starts)
  std::vector<int> th(p.nsn, -1);
  int ntop = 0;
  for (int sn = 0; sn < p.nsn; ++sn) {  // postorder: children first
    if (owner[sn] >= 0) continue;
    int h = 0;
    for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci) {
      const int c = p.child_list[ci];
      if (owner[c] < 0) h = std::max(h, th[c] + 1);
    }
    th[sn] = h;
    ntop = std::max(ntop, h + 1);
  }
  int nsub = 0;
  for (int r = 0; r < (int)roots.size(); ++r) nsub = std::max(nsub, p.level[roots[r]] + 1);
  sp->nsub = roots.empty() ? 0 : nsub;
  sp->sub_len = maxlen;
  sp->sub_cb = maxcb;
  // ---- dense top: one GEMV with K = (A^{-1})_TT replaces the top tree levels ----
  // K covers the top `kl` heights of the top tree (the K region: those supernodes and
  // all their ancestors); the heights below it (the band) stay tree levels, run
  // cluster/grid-wide between the subtree phase and the dense step.  kl = ntop: the
  // whole top is dense (no band).  The largest kl whose K fits the size rule wins.
  static const int dense_env = env_int2("STMHD_SWEEP_DENSE_TOP", 1);
  static const int klev_env = env_int2("STMHD_SWEEP_KLEVELS", -1);  // force kl (0: no dense top)
  static const int kmax_env = env_int2("STMHD_SWEEP_KMAX", 1600);   // largest K order with a band
  std::vector<char> isK(p.nsn, 0);
  int kl = 0;
  std::vector<int> tpos, tidx_h(p.n, -1);
  std::vector<int4> ztab;
  if (dense_env && mode <= 1 && sp->nsub > 0 && ntop > 0) {
    std::vector<int64_t> tcount(ntop + 1, 0);  // unknowns of the top kl heights
    for (int sn = 0; sn < p.nsn; ++sn)
      if (owner[sn] < 0) tcount[ntop - th[sn]] += p.ns[sn];
    for (int d = 1; d <= ntop; ++d) tcount[d] += tcount[d - 1];
    auto fits = [&](int d) {
      const int64_t nT = tcount[d];
      if (nT <= 0 || nT > 4096) return false;
      if (d == ntop)  // whole top: K (nT^2 per slab) may not outgrow the factor itself
        return nT * nT * (ncta <= 48 ? 1 : (max_sub < ncta ? 2 : 8)) <= p.factor_size;
      return nT <= kmax_env && 2 * nT * nT <= p.factor_size;
    };
    if (klev_env >= 0) kl = std::min(klev_env, ntop);
    else
      for (int d = ntop; d >= 1 && !kl; --d)
        if (fits(d)) kl = d;
    if (kl > 0 && tcount[kl] > 4096) kl = 0;
  }
  for (int sn = 0; sn < p.nsn; ++sn)
    if (owner[sn] < 0 && th[sn] >= ntop - kl) isK[sn] = 1;
  const int nband = ntop - kl;
  std::vector<std::vector<int>> top_sn(nband);
  for (int sn = 0; sn < p.nsn; ++sn)
    if (owner[sn] < 0 && !isK[sn]) top_sn[th[sn]].push_back(sn);
  sp->ntop = nband;
  if (kl > 0) {
    for (int sn = 0; sn < p.nsn; ++sn)  // K unknowns in elimination order
      if (isK[sn])
        for (int t = 0; t < p.ns[sn]; ++t) {
          const int q = (int)(p.first[sn] + t);
          tidx_h[q] = (int)tpos.size();
          tpos.push_back(q);
        }
    const int nT = (int)tpos.size();
    std::vector<std::array<int, 4>> zc(nT, {-1, -1, -1, -1});
    bool ok = nT > 0;
    // updates of the K region's children outside it (band nodes or subtree roots; they
    // write their update vectors to global memory) land on K unknowns: z_T inputs
    for (int sn = 0; sn < p.nsn && ok; ++sn) {
      if (!isK[sn]) continue;
      for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1] && ok; ++ci) {
        const int r = p.child_list[ci];
        if (isK[r]) continue;
        for (int a = 0; a < p.nb[r]; ++a) {
          const int tgt = bpos[p.idx_off[r] + p.ns[r] + a];
          const int i = tgt >= 0 ? tidx_h[tgt] : -1;
          if (i < 0) {
            ok = false;
            break;
          }
          int sl = 0;
          while (sl < 4 && zc[i][sl] >= 0) ++sl;
          if (sl == 4) {
            ok = false;
            break;
          }
          zc[i][sl] = (int)(p.cbv_off[r] + a);
        }
      }
    }
    if (ok) {
      sp->dense = 1;
      sp->ntT = nT;
      // row groups of kr rows x kc columns per ring item (<= one slot); kc even keeps
      // the items 16-byte aligned
      static const int kr_env = env_int2("STMHD_SWEEP_DENSE_R", 4);
      sp->kr = (kr_env == 1 || kr_env == 2 || kr_env == 4 || kr_env == 8) ? kr_env : 4;
      const int kcmax = (int)(slot_dbl / sp->kr) & ~1;
      sp->nch = (nT + kcmax - 1) / kcmax;
      sp->kc = ((nT + sp->nch - 1) / sp->nch + 1) / 2 * 2;
      sp->kpad = sp->nch * sp->kc;
      for (int i = 0; i < nT; ++i) {
        ztab.push_back(make_int4(tpos[i], zc[i][0], zc[i][1], zc[i][2]));
        ztab.push_back(make_int4(zc[i][3], -1, -1, -1));
      }
    } else {  // no dense top: the whole top runs as tree levels
      std::fill(isK.begin(), isK.end(), 0);
      std::fill(tidx_h.begin(), tidx_h.end(), -1);
      tpos.clear();
      top_sn.assign(ntop, {});
      for (int sn = 0; sn < p.nsn; ++sn)
        if (owner[sn] < 0) top_sn[th[sn]].push_back(sn);
      sp->ntop = ntop;
    }
  }
  // ---- subtree front tables resident in shared memory (dense mode) ----
  // forward (internal subtree supernodes only; leaves gather rhs rows alone): int32
  // per front entry = child update indices (y, z) relative to the CTA's update block
  // as two int16; backward (every subtree supernode, boundary entries t >= ns): uint16
  // = own-subtree index, 0x8000 | K index (x_T is staged in shared memory), or, with
  // band levels between the subtrees and the K region, 0xC000 | index into the CTA's
  // list of band positions (x read from global memory after the band levels).
  static const int stab_env = env_int2("STMHD_SWEEP_SMEM_TABLES", 1);
  std::vector<int> ftab_off(p.nsn, -1), btab_off(p.nsn, -1), sn_of_first(p.n, -1);
  std::vector<int> tab_all, tab_ptr(ncta + 1, 0), tab_nf(ncta, 0), tab_band, tab_band_ptr(ncta + 1, 0);
  bool stab = stab_env && mode == 0 && sp->dense && sp->nsub > 0 && maxlen < 32768 && maxcb < 32768 &&
              sp->ntT < 0x4000;
  // with resident tables the CTA's update block is compact: an update vector written at
  // subtree level h is read at level h + 1 only, so even and odd levels alternate between
  // two regions (each as large as its fullest level) instead of every supernode keeping
  // its own range -- about half the shared memory (C4 64-subtree plan: 1344 -> ~700 doubles)
  std::vector<int> cbloc(p.nsn, -1);
  if (stab) {
    int64_t maxcb2 = 0;
    for (int c = 0; c < ncta && c < (int)roots.size(); ++c) {
      std::vector<int64_t> lsum(sp->nsub + 1, 0);
      for (int sn = 0; sn < p.nsn; ++sn)
        if (owner[sn] == c && sn != roots[c]) lsum[p.level[sn]] += p.nb[sn];
      int64_t size[2] = {0, 0};
      for (int h = 0; h <= sp->nsub; ++h) size[h & 1] = std::max(size[h & 1], lsum[h]);
      std::vector<int64_t> cur(sp->nsub + 1);
      for (int h = 0; h <= sp->nsub; ++h) cur[h] = (h & 1) ? size[0] : 0;
      for (int sn = 0; sn < p.nsn; ++sn)
        if (owner[sn] == c && sn != roots[c]) {
          cbloc[sn] = (int)cur[p.level[sn]];
          cur[p.level[sn]] += p.nb[sn];
        }
      maxcb2 = std::max(maxcb2, size[0] + size[1]);
    }
    maxcb = maxcb2;
    sp->sub_cb = maxcb2;
  }
  if (stab) {
    for (int sn = 0; sn < p.nsn; ++sn) sn_of_first[p.first[sn]] = sn;
    for (int c = 0; c < ncta && c < (int)roots.size(); ++c) {
      const int64_t sf = info[4 * c];
      std::vector<int> fw;
      std::vector<unsigned short> bw;
      for (int sn = 0; sn < p.nsn; ++sn) {
        if (owner[sn] != c) continue;
        const int f = p.ns[sn] + p.nb[sn];
        const int64_t o = p.idx_off[sn];
        if (p.child_ptr[sn + 1] > p.child_ptr[sn]) {
          ftab_off[sn] = (int)fw.size();
          std::vector<int> yz[4] = {std::vector<int>(f, -1), std::vector<int>(f, -1), std::vector<int>(f, -1),
                                    std::vector<int>(f, -1)};
          int which = 0;
          for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci, ++which) {
            const int ch = p.child_list[ci];
            require(which < 4 && cbloc[ch] >= 0, "nd sweep: subtree supernode with an unexpected child");
            for (int a = 0; a < p.nb[ch]; ++a) yz[which][p.emap[p.emap_off[ch] + a]] = cbloc[ch] + a;
          }
          // (an amalgamated supernode has two table words per entry: children 0, 1 and 2, 3)
          for (int t = 0; t < f; ++t) {
            fw.push_back((int)((unsigned)(yz[0][t] & 0xffff) | ((unsigned)(yz[1][t] & 0xffff) << 16)));
            if (p.wide(sn)) fw.push_back((int)((unsigned)(yz[2][t] & 0xffff) | ((unsigned)(yz[3][t] & 0xffff) << 16)));
          }
        }
        btab_off[sn] = (int)bw.size();
        for (int t = p.ns[sn]; t < f; ++t) {
          const int q = bpos[o + t];
          const int64_t rel = q - sf;
          if (rel >= 0 && rel < info[4 * c + 1]) bw.push_back((unsigned short)rel);
          else if (tidx_h[q] >= 0) {
            bw.push_back((unsigned short)(0x8000 | tidx_h[q]));
          } else {  // band node
            int bi = -1;
            for (int i = tab_band_ptr[c]; i < (int)tab_band.size(); ++i)
              if (tab_band[i] == q) bi = i - tab_band_ptr[c];
            if (bi < 0) {
              bi = (int)tab_band.size() - tab_band_ptr[c];
              tab_band.push_back(q);
            }
            require(bi < 0x4000, "nd sweep: too many band boundary entries for the subtree tables");
            bw.push_back((unsigned short)(0xC000 | bi));
          }
        }
      }
      tab_band_ptr[c + 1] = (int)tab_band.size();
      while (bw.size() % 8) bw.push_back(0);  // 16-byte blocks
      tab_nf[c] = (int)fw.size();
      while (fw.size() % 4) fw.push_back(0);
      // block layout (ints): fwd entries, then the uint16 backward entries packed in pairs
      const size_t base = tab_all.size();
      tab_all.insert(tab_all.end(), fw.begin(), fw.end());
      for (size_t i = 0; i < bw.size(); i += 2) tab_all.push_back((int)((unsigned)bw[i] | ((unsigned)bw[i + 1] << 16)));
      tab_ptr[c + 1] = (int)tab_all.size();
      tab_nf[c] = (int)fw.size();  // padded forward length (start of the backward entries)
      static_cast<void>(base);
    }
    for (int c = (int)roots.size(); c < ncta; ++c) {
      tab_ptr[c + 1] = tab_ptr[c];
      tab_band_ptr[c + 1] = tab_band_ptr[c];
    }
    int maxtab = 0;
    for (int c = 0; c < ncta; ++c) maxtab = std::max(maxtab, tab_ptr[c + 1] - tab_ptr[c]);
    sp->tab_ints = (maxtab + 3) / 4 * 4;
  }
  // per direction: top tasks per [top level][global warp], subtree tasks per
  // [cta][local level][warp]
  std::vector<std::vector<SweepTask>> top_t[2], sub_t[2];
  auto build_dir = [&](bool fwd) {
    auto &tt = top_t[fwd];
    auto &st = sub_t[fwd];
    tt.assign((size_t)sp->ntop * W, {});
    st.assign((size_t)ncta * sp->nsub * warps, {});
    for (int t = 0; t < sp->ntop; ++t) {
      std::vector<SN> sns;
      std::vector<char> cbg;
      for (int sn : top_sn[t]) {
        SN x;
        if (make_sn(sn, fwd, x)) {
          sns.push_back(x);
          cbg.push_back(1);
        }
      }
      std::vector<std::vector<SweepTask>> per;
      schedule(sns, W, fwd, per, cbg);
      for (int w = 0; w < W; ++w) tt[(size_t)t * W + w] = std::move(per[w]);
    }
    for (int c = 0; c < ncta; ++c)
      for (int h = 0; h < sp->nsub; ++h) {
        std::vector<SN> sns;
        std::vector<char> cbg;
        if (c < (int)roots.size())
          for (int sn : p.level_sn[h]) {
            SN x;
            if (owner[sn] == c && make_sn(sn, fwd, x)) {
              sns.push_back(x);
              cbg.push_back(sn == roots[c]);
            }
          }
        std::vector<std::vector<SweepTask>> per;
        schedule(sns, warps, fwd, per, cbg);
        if (stab)  // tables in shared memory (flags 16: leaf, no forward table; 32: shared table)
          for (auto &pw : per)
            for (SweepTask &t : pw) {
              const int sn = sn_of_first[t.first];
              t.flags &= (unsigned char)~(4 | 8);
              if (fwd) {
                // compact update block: the kernel adds cboff to cbs - cbfirst
                if (!(t.flags & 1)) t.cboff = (int)(info[4 * c + 2] + cbloc[sn]);
                if (ftab_off[sn] < 0) t.flags |= 16;
                else {
                  t.flags |= 32;
                  t.goff = ftab_off[sn];
                }
              } else {
                t.flags |= 32;
                t.cboff = btab_off[sn];
              }
            }
        for (int w = 0; w < warps; ++w) st[((size_t)c * sp->nsub + h) * warps + w] = std::move(per[w]);
      }
  };
  build_dir(true);
  build_dir(false);
  // per physical warp (cta c, warp w; top-phase global warp id w * ncta + c): its
  // list in kernel order and the bound of every phase level
  // dense top: one phase level of row tasks (row i of K: nch column chunks of kc)
  std::vector<std::vector<SweepTask>> dense_t(W);  // by global warp w * ncta + c
  if (sp->dense) {
    const int ng = (sp->ntT + sp->kr - 1) / sp->kr;
    static const int dsplit_env = env_int2("STMHD_SWEEP_DENSE_SPLIT", 1);
    static const int dpc_env = env_int2("STMHD_SWEEP_DENSE_PC", 0);  // force chunks per piece
    int npc = dsplit_env ? std::max(1, std::min(sp->nch, (W + ng - 1) / ng)) : 1;
    if (dpc_env > 0) npc = (sp->nch + dpc_env - 1) / dpc_env;
    const int pc = (sp->nch + npc - 1) / npc;  // chunks per piece
    npc = (sp->nch + pc - 1) / pc;
    sp->dpieces = npc;
    sp->dgroups = (ng + ncta - 1) / ncta;
    for (int c = 0; c < ncta; ++c) {
      std::vector<std::pair<int, SweepTask>> items;  // (chunks, task)
      for (int g = c, j = 0; g < ng; g += ncta, ++j)
        for (int q = 0; q < npc; ++q) {
          const int c0 = q * pc, c1 = std::min(sp->nch, (q + 1) * pc);
          if (c1 <= c0) continue;
          SweepTask t{};
          t.foff = g * sp->kr * sp->kpad;
          t.goff = 0;
          t.first = g * sp->kr;  // first row of the group (top index; positions via ztab)
          t.cboff = j * npc + q;  // partial-sum slot in the CTA's dred
          t.c0 = (short)c0;
          t.c1 = (short)c1;
          t.ns = (short)sp->kc;
          t.f = (short)sp->kc;
          t.rows = (short)sp->kr;
          t.R = (unsigned char)sp->kr;
          t.flags = 2;
          t.bsz = sp->kr * sp->kc;
          items.push_back({c1 - c0, t});
        }
      std::stable_sort(items.begin(), items.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
      std::vector<int> load(warps, 0);
      for (auto &it : items) {
        const int w = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        dense_t[(size_t)w * ncta + c].push_back(it.second);
        load[w] += it.first;
      }
      if (c == 0 && getenv("STMHD_SWEEP_PLAN_INFO"))
        fprintf(stderr, "[sweep-plan] dense: nT %d kc %d nch %d groups %d pieces %d x %d chunks, CTA 0: %zu items, max chunks per warp %d\n",
                sp->ntT, sp->kc, sp->nch, ng, npc, pc, items.size(), *std::max_element(load.begin(), load.end()));
    }
  }
  sp->nl = 2 * sp->nsub + 2 * sp->ntop + (sp->dense ? 1 : 0);
  {
    std::vector<SweepTask> all;
    std::vector<int> off, bnd;
    int maxw = 0;
    for (int c = 0; c < ncta; ++c)
      for (int w = 0; w < warps; ++w) {
        off.push_back((int)all.size());
        const size_t o = all.size();
        auto add = [&](const std::vector<SweepTask> &v) {
          bnd.push_back((int)(all.size() - o));
          all.insert(all.end(), v.begin(), v.end());
        };
        for (int h = 0; h < sp->nsub; ++h) add(sub_t[1][((size_t)c * sp->nsub + h) * warps + w]);
        for (int t = 0; t < sp->ntop; ++t) add(top_t[1][(size_t)t * W + w * ncta + c]);  // band forward
        if (sp->dense) add(dense_t[w * ncta + c]);
        for (int t = sp->ntop - 1; t >= 0; --t) add(top_t[0][(size_t)t * W + w * ncta + c]);  // band backward
        for (int h = sp->nsub - 1; h >= 0; --h) add(sub_t[0][((size_t)c * sp->nsub + h) * warps + w]);
        bnd.push_back((int)(all.size() - o));
        maxw = std::max(maxw, (int)(all.size() - o));
      }
    off.push_back((int)all.size());
    if (all.empty()) all.push_back(SweepTask{});
    sp->max_wtasks = maxw;
    if (getenv("STMHD_SWEEP_TRACE") || getenv("STMHD_SWEEP_PLAN_INFO")) {
      std::vector<int64_t> fsum(ncta, 0), nbsum(ncta, 0);
      for (int sn = 0; sn < p.nsn; ++sn)
        if (owner[sn] >= 0) {
          fsum[owner[sn]] += p.ns[sn] + p.nb[sn];
          nbsum[owner[sn]] += p.nb[sn];
        }
      fprintf(stderr, "[sweep-plan] n=%lld D=%d band=%d dense=%d (K levels %d, nT %d) nsub=%d max_wtasks=%d max sub front entries %lld (nb %lld)\n",
              (long long)p.n, D, sp->ntop, sp->dense, kl, sp->ntT, sp->nsub, maxw, (long long)*std::max_element(fsum.begin(), fsum.end()),
              (long long)*std::max_element(nbsum.begin(), nbsum.end()));
    }
    // shared memory: subtree vectors + per-warp task lists must fit next to the
    // per-warp gather buffers; otherwise fall back to an all-top schedule
    const int64_t tdoubles = (int64_t)warps * (((sp->nl + 1 + 3) / 4) * 16 + (int64_t)maxw * 32) / 8;
    // gather buffer: in dense mode only subtree fronts are gathered
    int fmax = 1;
    for (int sn = 0; sn < p.nsn; ++sn)
      if (!isK[sn]) fmax = std::max(fmax, p.ns[sn] + p.nb[sn]);
    sp->vstride = (int)((fmax + 15) / 16 * 16 + kRing * slot_sz);
    const int64_t need = (int64_t)warps * sp->vstride + 3 * maxlen + maxcb + tdoubles + sp->zlen() + sp->tab_ints / 2 + 4;
    if (!flat && D > 0 && need > smem_budget) {
      const int next = sp->tab_ints ? 1 : (sp->dense ? 2 : 3);
      return get_sweep_plan(ncta, warps, smem_budget, s, next);
    }
    sp->wl_tasks = upload_vec(all, s);
    sp->wl_off = upload_vec(off, s);
    sp->wl_bnd = upload_vec(bnd, s);
  }
  sp->sub_info = upload_vec(info, s);
  if (sp->dense) {
    sp->ztab = upload_vec(ztab, s);
    sp->tidx = upload_vec(tidx_h, s);
    std::vector<int> tsn_index(p.nsn, -1);
    std::vector<TopSN> tsn;
    std::vector<int4> tch;
    int64_t tcb = 0;
    for (int sn = 0; sn < p.nsn; ++sn) {
      if (!isK[sn]) continue;
      require(p.fl_off[sn] < INT32_MAX && p.fu_off[sn] < INT32_MAX && p.idx_off[sn] < INT32_MAX,
              "nd sweep: factor too large for the dense-top construction");
      TopSN t{};
      t.ns = p.ns[sn];
      t.nb = p.nb[sn];
      t.first = (int)p.first[sn];
      t.goff = (int)p.idx_off[sn];
      t.fl_off = (int)p.fl_off[sn];
      t.fu_off = (int)p.fu_off[sn];
      t.rf = p.rf[sn];
      t.rb = p.rb[sn];
      t.bszf = (int)p.bsz_f[sn];
      t.bszb = (int)p.bsz_b[sn];
      t.tcb_off = (int)tcb;
      tcb += p.nb[sn];
      t.child0 = (int)tch.size();
      for (int ci = p.child_ptr[sn]; ci < p.child_ptr[sn + 1]; ++ci) {
        const int c = p.child_list[ci];
        if (!isK[c]) continue;  // band nodes / subtree roots: their updates are inputs (z_T)
        require(tsn_index[c] >= 0, "nd sweep: top tree not in postorder");
        tch.push_back(make_int4(tsn_index[c], (int)p.emap_off[c], p.nb[c], 0));
      }
      t.nchild = (int)tch.size() - t.child0;
      tsn_index[sn] = (int)tsn.size();
      tsn.push_back(t);
    }
    if (tch.empty()) tch.push_back(make_int4(0, 0, 0, 0));
    sp->ntsn = (int)tsn.size();
    sp->tcb_total = tcb;
    sp->kfmax = 1;
    for (const TopSN &t : tsn) sp->kfmax = std::max(sp->kfmax, t.ns + t.nb);
    sp->tsn = upload_vec(tsn, s);
    sp->tchild = upload_vec(tch, s);
  }
  sp->sub_info_h = info;
  sp->pos_h = pos;
  sp->iperm_h = iperm;
  sp->g3p = upload_vec(g3, s);
  sp->g4p = upload_vec(g4, s);
  sp->bpos = upload_vec(bpos, s);
  sp->bpos4 = upload_vec(bpos4, s);
  if (stab) {
    if (tab_all.empty()) tab_all.push_back(0);
    sp->tab = upload_vec(tab_all, s);
    sp->tab_ptr = upload_vec(tab_ptr, s);
    sp->tab_nf = upload_vec(tab_nf, s);
    if (tab_band.empty()) tab_band.push_back(0);
    sp->tab_band = upload_vec(tab_band, s);
    sp->tab_band_ptr = upload_vec(tab_band_ptr, s);
  }
  sp->pos = upload_vec(pos, s);
  sp->iperm = upload_vec(iperm, s);
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  sweep_plans.push_back(std::move(sp));
  return *sweep_plans.back();
}

struct SweepArgs {
  // per physical warp task lists (NDSweepPlan::wl_*), copied to shared memory
  const SweepTask *wl_tasks;
  const int *wl_off, *wl_bnd;
  int nl, tstride;             // phase levels; bytes of shared memory per warp list
  const int64_t *sub_info;     // per CTA {first col, ncols, first cb, ncb}
  int ntop, nsub, warps;
  int64_t sub_len, sub_cb;     // shared-memory sizes of the subtree vectors
  // fused slab coupling (CplProgram): per-CTA items computed at the start of a slab
  const int4 *prog_hdr;
  const int2 *prog_items;
  const int *prog_ecol;
  const double *prog_vals;     // [slab or 0][entry]: coef * coupling value
  int64_t prog_nent;
  int prog_per_slab;
  double *tbuf;                // coupled right-hand side of the top rows
  // per-CTA subtree front tables resident in shared memory (NDSweepPlan::tab)
  const int *tab, *tab_ptr, *tab_nf;
  const int *tab_band, *tab_band_ptr;  // per-CTA band positions of the backward tables
  int tab_ints;
  // dense top (NDSweepPlan::dense): z_T gather table and K = (A^{-1})_TT per slab
  int dense, ntT, kpad, zlen;  // zlen: shared doubles of z_T + the dense partial sums
  int dpieces, dgroups, kr;
  const int4 *ztab;
  const double *ktop;
  int64_t kstride;             // doubles per slab of ktop (0: one K for all slabs)
  // post-slab program (pipelined launch): after slab k, post_out[k] += C x(k)
  const int4 *post_hdr;
  const int2 *post_items;
  const int *post_ecol;
  const double *post_vals;
  int64_t post_nent, post_n;
  int post_per_slab;
  double *post_out;            // another stage's permuted right-hand sides (nslab x post_n)
  const int4 *g3p;
  const int *g4p;  // fourth child update slot of wide supernodes (task flag 64)
  const int *bpos;
  const int *bpos4;            // 16-byte aligned bpos copy (ring table items)
  int nlevels, nw;
  int64_t n;
  const double *factors;
  int64_t fstride;
  const double *rhsp;  // nslab x n (permuted)
  double *xp;          // nslab x n (permuted)
  double *ybuf, *cbv;
  const double *zero;  // n zeros (sources that do not exist yet read from here)
  int nslab, ncta;
  // pipelined launch: external sources (other stages' permuted outputs) and flags
  const double *ext_xp[2];
  int64_t ext_n[2];
  const int *flag_in[2];  // per producer: [slab][cta] = epoch once slab written
  int ext_ncta[2];        // per producer: its CTA count
  int nwait;
  int *flag_out;          // this stage's flags (null: not consumed and not early coupling)
  // early coupling (grid mode with CTAs that own no subtree): a subtree CTA computes the
  // coupled right-hand side of its own rows for slab k+1 right after its subtree
  // backward of slab k (its rows couple only to its own subtree and to separator
  // nodes, all final by then), with no grid barrier at the slab end; the CTAs without
  // a subtree compute the top rows after the subtree CTAs published slab k
  int early_cpl, nroots;
  int epoch;
  int vstride;  // doubles per warp: gather buffer + 2 TMA slots
  int slot;     // doubles per TMA slot (largest chunk block)
  int null_work;  // diagnostics: skip all task work (barrier/loop floor)
  unsigned *gbar;  // grid mode (one CTA per SM, cooperative launch): software grid barrier word
  int cpl16;       // coupling program: 16 entries per step when a CTA has one item per thread
  int kpref;       // L2 prefetch of the slab's dense-top rows at the slab start
  unsigned long long *progress;  // L2 prefetch cluster: (epoch << 32) | slab in progress (CTA 0)
  int ldgsts;      // ring items by warp-wide cp.async (16 B per lane) instead of one cp.async.bulk
  int *fault;       // device word: a consumer gave up waiting for a producer (timeout)
  int *fault_host;  // host-mapped copy of the fault word, read by the host after the launch
  unsigned long long *trace;
  unsigned long long *prof;  // PROF instantiation: 6 counters per warp
  unsigned long long *tline; // PROF instantiation: per-warp event timeline of slab 1, CTA 0 (128 per warp)
  unsigned long long *pcta;  // PROF instantiation: per CTA, slab 1: subtree forward / backward durations (ns)
};

__device__ __forceinline__ void sweep_barrier(const SweepArgs &a, int crank, unsigned &gphase) {
  if (a.gbar) {
    // software barrier over the stage's a.ncta CTAs (cooperative-groups arrival
    // scheme: every CTA adds 1, rank 0 adds 2^31 - (n - 1), so the top bit flips once
    // all arrived).  The arrival is a fire-and-forget release reduction; each CTA
    // tracks the expected top bit itself (gphase, read once per launch), so only the
    // polling loads are round trips.
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned nb = crank == 0 ? 0x80000000u - (unsigned)(a.ncta - 1) : 1u;
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a.gbar), "r"(nb) : "memory");
      gphase ^= 0x80000000u;
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(a.gbar) : "memory");
      } while ((cur & 0x80000000u) != gphase);
    }
    __syncthreads();
    return;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned cluster_index() {
  unsigned r;
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void sweep_trace(const SweepArgs &a, int &step, int crank) {
  if (a.trace && threadIdx.x == 0 && crank == 0) {
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
  // no cross-proxy fence: the slot's previous contents were only READ through the
  // generic proxy, and those loads completed (their values were consumed before the
  // __syncwarp that precedes every issue)
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

// This CTA's band positions (global; 0xC000 backward-table codes).  Kept in shared
// memory, not in SubView: the sweep kernel sits at its register cap and every pointer
// held across the slab loop spills.
__shared__ const int *s_bband;

// Per-CTA view of the subtree vectors kept in shared memory.
struct SubView {
  double *ys, *xs, *cbs, *rhs_s;  // rhs_s: coupled right-hand side of the subtree rows (fused mode)
  double *zs;                     // dense top: z_T (kpad doubles); x_T during the subtree backward
  const int *ftab;                // subtree forward tables (shared memory) or null
  const unsigned short *btab;     // subtree backward tables
  int64_t first, len, cbfirst;
};

struct WarpCtx {
  int lane, wl;
  double *v;
  double *slot0;  // two TMA slots: slot0, slot0 + slotsz
  int slotsz;
  // this warp's task list for one slab (shared memory; repeated for every slab)
  const SweepTask *tl;
  const int *bnd;  // start of every phase level in tl (nl + 1 entries)
  int nt;
  int jc;                       // chunks consumed (slot jc % kRing, mbarrier parity (jc / kRing) & 1)
  int icount, rt, rc, rslab;    // TMA ring cursor (lane 0): two chunks ahead of jc
  // PROF instantiation: cycles in gather / TMA wait / GEMV+store / barriers, tasks, chunks
  long long acc[10];  // PROF: 8 issue cycles (ring_issue after a chunk)
  unsigned long long *tl_out;  // timeline (PROF, slab 1 of CTA 0) or null
  int tl_n;
};

__device__ __forceinline__ void tl_mark(WarpCtx &w, unsigned code) {
  if (w.tl_out && w.lane == 0 && w.tl_n < 128) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    w.tl_out[w.tl_n++] = ((unsigned long long)code << 56) | (t & ((1ull << 56) - 1));
  }
}

template <bool PROF>
__device__ __forceinline__ long long pclock() {
  if constexpr (PROF) return clock64();
  else return 0;
}

// First ring item of a task: its front table (flags & 4) or its first chunk.
__device__ __forceinline__ int first_item(const SweepTask &t) { return (t.flags & 4) ? t.c0 - 1 : t.c0; }

// Global source and size (doubles) of ring item (task t, index c, slab) -- the
// task's front table (c < c0) or one of its chunks.
__device__ __forceinline__ const double *item_src(const SweepArgs &a, const SweepTask &t, int c, int slab,
                                                  int &dbl) {
  if (c < t.c0) {
    if (t.flags & 8) {
      dbl = (t.f + 3) / 4 * 2;
      return reinterpret_cast<const double *>(a.bpos4 + t.cboff);
    }
    dbl = 2 * t.f;
    return reinterpret_cast<const double *>(a.g3p + t.goff);
  }
  dbl = t.bsz;
  const double *base = (t.flags & 2) ? a.ktop + (int64_t)slab * a.kstride  // dense-top row chunk
                                     : a.factors + (int64_t)slab * a.fstride;
  return base + t.foff + (int64_t)c * t.bsz;
}

// Advance a (task, item, slab) cursor along the warp's item sequence.
__device__ __forceinline__ void item_next(const WarpCtx &w, int &t, int &c, int &slab) {
  if (++c == w.tl[t].c1) {
    if (++t == w.nt) {
      t = 0;
      ++slab;
    }
    c = first_item(w.tl[t]);
  }
}

// Issue the next item of the warp's sequence into the free slot (lane 0).  The ring
// runs across task, level and slab boundaries (factors do not depend on the data),
// so a warp's next items are in flight while it waits at a barrier.  (An L2 bulk
// prefetch cursor further ahead along the same sequence was measured slower.)
__device__ __forceinline__ void ring_issue(const SweepArgs &a, WarpCtx &w, unsigned long long (*mbar)[kRing]) {
  if (w.rslab < a.nslab && w.nt > 0) {
    const int sl = w.icount % kRing;
    int dbl;
    const double *src = item_src(a, w.tl[w.rt], w.rc, w.rslab, dbl);
    tma_load(w.slot0 + sl * w.slotsz, src, dbl, &mbar[w.wl][sl]);
    ++w.icount;
    item_next(w, w.rt, w.rc, w.rslab);
  }
}

// Warp-wide variant (a.ldgsts, every lane calls it): 16-byte cp.async per lane, the
// slot's mbarrier (expected count 32) completes once every lane's copies landed.  A
// cp.async.bulk issue blocks the issuing warp ~350-430 cycles (tools/tma_ring_probe.cu),
// on the critical path after every chunk; the per-lane copies issue in ~10 cycles each.
__device__ __forceinline__ void ring_issue_warp(const SweepArgs &a, WarpCtx &w, unsigned long long (*mbar)[kRing]) {
  if (w.rslab < a.nslab && w.nt > 0) {
    const int sl = w.icount % kRing;
    int dbl;
    const double *src = item_src(a, w.tl[w.rt], w.rc, w.rslab, dbl);
    double *dst = w.slot0 + sl * w.slotsz;
    for (int i = 2 * w.lane; i < dbl; i += 64)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst + i)), "l"(src + i) : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar[w.wl][sl])) : "memory");
    ++w.icount;
    item_next(w, w.rt, w.rc, w.rslab);
  }
}

// Refill the ring after a consumed item (call from every lane, after the __syncwarp
// that ends the item's reads).
__device__ __forceinline__ void ring_next(const SweepArgs &a, WarpCtx &w, unsigned long long (*mbar)[kRing]) {
  if (a.ldgsts) ring_issue_warp(a, w, mbar);
  else if (w.lane == 0) ring_issue(a, w, mbar);
}

// GEMV of one shared-memory chunk block [K][R] (R a power of two, lane = kq*R + rl):
// element (kq + q*kl, rl) sits at blk[lane + 32 q], so the block is walked with
// immediate offsets and one predicate per step.  Returns row rl's dot product
// (reduced over the kl lanes sharing rl).
__device__ __forceinline__ double chunk_gemv_smem(const double *blk, int KR, int kl, int kq, int R,
                                                  const double *v, int lane) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const double *b = blk + lane;
  const double *vv = v + kq;
  for (int base = 0; base < KR; base += 640) {
    const int rem = KR - base - lane;
#pragma unroll
    for (int q = 0; q < 20; ++q)
      if (32 * q < rem) acc[q & 3] = fma(b[32 * q], vv[q * kl], acc[q & 3]);
    b += 640;
    vv += 20 * kl;
  }
  double out = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (int o = R; o < 32; o <<= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
  return out;
}

// Forward (L) step of one task: gather the front, stream its factor chunks, GEMV.
template <bool SUB, bool PROF>
__device__ __forceinline__ void forward_task(const SweepArgs &a, const SweepTask &tk, const double *F,
                                             const double *rhs, const SubView &sv, WarpCtx &w,
                                             unsigned long long (*mbar)[kRing]) {
  const int lane = w.lane;
  long long t0 = pclock<PROF>();
  const int4 *g = a.g3p + tk.goff;
  if (tk.flags & 4) {  // front table arrived through the ring
    mbar_wait(&mbar[w.wl][w.jc % kRing], (unsigned)(w.jc / kRing) & 1u);
    g = reinterpret_cast<const int4 *>(w.slot0 + (w.jc % kRing) * w.slotsz);
  }
  const double *cbsrc = SUB ? sv.cbs - sv.cbfirst : a.cbv;
  // fused coupling: subtree rows come from shared memory, top rows from tbuf
  const bool fused = a.prog_hdr != nullptr;
  const double *rsrc = (SUB && fused) ? sv.rhs_s - sv.first : (fused ? a.tbuf : rhs);
  if (SUB && (tk.flags & (16 | 32))) {
    // shared-memory front: a leaf gathers its rhs rows only; an internal node adds
    // its children's updates through the resident table
    const int *ft = sv.ftab + tk.goff;
    const bool leaf = tk.flags & 16;
    if (tk.flags & 64) {  // amalgamated supernode: two table words per entry (four children)
      for (int t = lane; t < tk.f; t += 32) {
        double v = t < tk.ns ? rsrc[tk.first + t] : 0.0;
        const int e = ft[2 * t], e2 = ft[2 * t + 1];
        const int y = (short)(e & 0xffff), z = (short)(e >> 16), y2 = (short)(e2 & 0xffff), z2 = (short)(e2 >> 16);
        v = ((v + (y >= 0 ? sv.cbs[y] : 0.0)) + (z >= 0 ? sv.cbs[z] : 0.0)) +
            ((y2 >= 0 ? sv.cbs[y2] : 0.0) + (z2 >= 0 ? sv.cbs[z2] : 0.0));
        w.v[t] = v;
      }
    } else
    for (int t = lane; t < tk.f; t += 32) {
      double v = t < tk.ns ? rsrc[tk.first + t] : 0.0;
      if (!leaf) {
        const int e = ft[t];
        const int y = (short)(e & 0xffff), z = (short)(e >> 16);
        v = (v + (y >= 0 ? sv.cbs[y] : 0.0)) + (z >= 0 ? sv.cbs[z] : 0.0);
      }
      w.v[t] = v;
    }
  } else if (!SUB) {
    // top-level task: the GEMV reads the ns column entries and the update needs the
    // task's own rows beyond them, so only those front entries are gathered
    // (entry tt of the list is front position tt < ns ? tt : rlo + tt - ns).
    const int rlo = max((int)tk.ns, tk.c0 * (int)tk.R), rhi = min((int)tk.f, tk.c1 * (int)tk.R);
    const int ng = tk.ns + max(0, rhi - rlo), sh = rlo - tk.ns;
    if (tk.flags & 64) {
      // amalgamated supernode: up to four child updates per entry (slot w of the table
      // and the parallel g4 table); five entries per lane and pass
      const int *g4 = a.g4p + tk.goff;
      for (int b0 = lane; b0 < ng; b0 += 160) {
        int4 gg[5];
        int g5[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          const int tt = b0 + 32 * q, te = tt < tk.ns ? tt : tt + sh;
          gg[q] = tt < ng ? g[te] : make_int4(-1, -1, -1, -1);
          g5[q] = tt < ng ? g4[te] : -1;
        }
        double vv[5];
#pragma unroll
        for (int q = 0; q < 5; ++q)
          vv[q] = (((gg[q].x >= 0 ? rsrc[gg[q].x] : 0.0) + (gg[q].y >= 0 ? cbsrc[gg[q].y] : 0.0)) +
                   (gg[q].z >= 0 ? cbsrc[gg[q].z] : 0.0)) +
                  ((gg[q].w >= 0 ? cbsrc[gg[q].w] : 0.0) + (g5[q] >= 0 ? cbsrc[g5[q]] : 0.0));
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          const int tt = b0 + 32 * q;
          if (tt < ng) w.v[tt < tk.ns ? tt : tt + sh] = vv[q];
        }
      }
    } else {
      for (int b0 = lane; b0 < ng; b0 += 256) {
        int4 gg[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int tt = b0 + 32 * q;
          gg[q] = tt < ng ? g[tt < tk.ns ? tt : tt + sh] : make_int4(-1, -1, -1, -1);
        }
        double vv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          vv[q] = ((gg[q].x >= 0 ? rsrc[gg[q].x] : 0.0) + (gg[q].y >= 0 ? cbsrc[gg[q].y] : 0.0)) +
                  (gg[q].z >= 0 ? cbsrc[gg[q].z] : 0.0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int tt = b0 + 32 * q;
          if (tt < ng) w.v[tt < tk.ns ? tt : tt + sh] = vv[q];
        }
      }
    }
  } else
  for (int b0 = lane; b0 < tk.f; b0 += 256) {
    int4 gg[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) gg[q] = (b0 + 32 * q < tk.f) ? g[b0 + 32 * q] : make_int4(-1, -1, -1, -1);
    double vv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      vv[q] = ((gg[q].x >= 0 ? rsrc[gg[q].x] : 0.0) + (gg[q].y >= 0 ? cbsrc[gg[q].y] : 0.0)) +
              (gg[q].z >= 0 ? cbsrc[gg[q].z] : 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b0 + 32 * q < tk.f) w.v[b0 + 32 * q] = vv[q];
  }
  if (SUB && (tk.flags & 64) && !(tk.flags & (16 | 32))) {
    // amalgamated supernode on the table path of a subtree (no resident tables):
    // children 2 and 3 (each lane revisits its own entries)
    const double *cb2 = sv.cbs - sv.cbfirst;
    const int *g4 = a.g4p + tk.goff;
    for (int t = lane; t < tk.f; t += 32) {
      const int gw = g[t].w, g5 = g4[t];
      w.v[t] += (gw >= 0 ? cb2[gw] : 0.0) + (g5 >= 0 ? cb2[g5] : 0.0);
    }
  }
  __syncwarp();
  if (PROF) tl_mark(w, 2);
  if (tk.flags & 4) {  // table consumed: its slot goes back to the ring
    ++w.jc;
    ring_next(a, w, mbar);
  }
  if (PROF) {
    const long long t1 = pclock<PROF>();
    w.acc[0] += t1 - t0;
    w.acc[4] += 1;
    w.acc[5] += tk.c1 - tk.c0;
    t0 = t1;
  }
  const int R = tk.R, lgR = __ffs(R) - 1, kl = 32 >> lgR, kq = lane >> lgR;
  double *ydst = SUB ? sv.ys - sv.first : a.ybuf;
  double *cbdst = (!SUB || (tk.flags & 1)) ? a.cbv : sv.cbs - sv.cbfirst;
  for (int c = tk.c0; c < tk.c1; ++c) {
    const int sl = w.jc % kRing;
    mbar_wait(&mbar[w.wl][sl], (unsigned)(w.jc / kRing) & 1u);
    const double *blk = w.slot0 + sl * w.slotsz;
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[1] += t1 - t0;
      t0 = t1;
    }
    const double out = chunk_gemv_smem(blk, tk.ns * R, kl, kq, R, w.v, lane);
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[6] += t1 - t0;
      t0 = t1;
    }
    const int r = c * R + (lane & (R - 1));
    if (lane < R && r < tk.rows) {
      if (r < tk.ns) ydst[tk.first + r] = out;
      else cbdst[tk.cboff + r - tk.ns] = w.v[r] - out;
    }
    __syncwarp();
    ++w.jc;
    long long ti0 = pclock<PROF>();
    ring_next(a, w, mbar);
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[8] += t1 - ti0;
      w.acc[2] += t1 - t0;
      t0 = t1;
      tl_mark(w, 3);
    }
  }
  __syncwarp();
}

// Backward (U) step of one task.
template <bool SUB, bool PROF>
__device__ __forceinline__ void backward_task(const SweepArgs &a, const SweepTask &tk, const double *F, double *x,
                                              const SubView &sv, WarpCtx &w, unsigned long long (*mbar)[kRing]) {
  const int lane = w.lane;
  long long t0 = pclock<PROF>();
  if (SUB && (tk.flags & 32)) {
    // shared-memory front: own y, own-subtree x (xs) or top x (staged in zs)
    const unsigned short *bt = sv.btab + tk.cboff - tk.ns;
    const double *ys = sv.ys - sv.first + tk.first;
    if (a.ntop == 0) {  // no band levels: own subtree or K only (keeps this loop lean)
      for (int t = lane; t < tk.f; t += 32) {
        double v;
        if (t < tk.ns) v = ys[t];
        else {
          const unsigned code = bt[t];
          v = (code & 0x8000u) ? sv.zs[code & 0x3fffu] : sv.xs[code];
        }
        w.v[t] = v;
      }
    } else {
      for (int t = lane; t < tk.f; t += 32) {
        double v;
        if (t < tk.ns) v = ys[t];
        else {
          const unsigned code = bt[t];
          v = (code & 0x8000u) ? ((code & 0x4000u) ? x[s_bband[code & 0x3fffu]] : sv.zs[code & 0x3fffu])
                               : sv.xs[code];
        }
        w.v[t] = v;
      }
    }
    __syncwarp();
  }
  const int *bp = a.bpos + tk.goff;
  if (tk.flags & 4) {  // front table arrived through the ring
    mbar_wait(&mbar[w.wl][w.jc % kRing], (unsigned)(w.jc / kRing) & 1u);
    bp = reinterpret_cast<const int *>(w.slot0 + (w.jc % kRing) * w.slotsz);
  }
  const double *y = (SUB ? sv.ys - sv.first : a.ybuf) + tk.first;
  if (!(SUB && (tk.flags & 32)))
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
      // one (generic) load per entry: own subtree from shared memory, else global
      const int64_t off = ii[q] - sv.first;
      const double *src = (SUB && (uint64_t)off < (uint64_t)sv.len) ? sv.xs + off : x + ii[q];
      if (ii[q] < 0) src = y + (t < tk.ns ? t : 0);  // t >= f: any valid address (unused)
      vv[q] = *src;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (b0 + 32 * q < tk.f) w.v[b0 + 32 * q] = vv[q];
  }
  __syncwarp();
  if (PROF) tl_mark(w, 2);
  if (tk.flags & 4) {
    ++w.jc;
    ring_next(a, w, mbar);
  }
  if (PROF) {
    const long long t1 = pclock<PROF>();
    w.acc[0] += t1 - t0;
    w.acc[4] += 1;
    w.acc[5] += tk.c1 - tk.c0;
    t0 = t1;
  }
  const int R = tk.R, lgR = __ffs(R) - 1, kl = 32 >> lgR, kq = lane >> lgR;
  for (int c = tk.c0; c < tk.c1; ++c) {
    const int sl = w.jc % kRing;
    mbar_wait(&mbar[w.wl][sl], (unsigned)(w.jc / kRing) & 1u);
    const double *blk = w.slot0 + sl * w.slotsz;
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[1] += t1 - t0;
      t0 = t1;
    }
    const double out = chunk_gemv_smem(blk, tk.f * R, kl, kq, R, w.v, lane);
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[7] += t1 - t0;
      t0 = t1;
    }
    const int r = c * R + (lane & (R - 1));
    if (lane < R && r < tk.rows) {
      x[tk.first + r] = out;
      if (SUB) sv.xs[tk.first + r - sv.first] = out;
    }
    __syncwarp();
    ++w.jc;
    long long ti0 = pclock<PROF>();
    ring_next(a, w, mbar);
    if (PROF) {
      const long long t1 = pclock<PROF>();
      w.acc[8] += t1 - ti0;
      w.acc[2] += t1 - t0;
      t0 = t1;
      tl_mark(w, 3);
    }
  }
  __syncwarp();
}

// Dense-top row-group task: x[pos(first + r)] = K[first + r] . z_T for the group's R
// rows, streamed as nch column chunks ([kc][R] blocks) through the warp's TMA ring
// (lane = kq * R + r covers columns kq + (32 / R) q of row r).
template <bool PROF>
__device__ __forceinline__ void dense_task(const SweepArgs &a, const SweepTask &tk, const double *zs, double *dred,
                                           WarpCtx &w, unsigned long long (*mbar)[kRing]) {
  const int lane = w.lane;
  const int R = tk.R, kl = 32 / R;
  double acc = 0.0;
  for (int c = tk.c0; c < tk.c1; ++c) {
    const int sl = w.jc % kRing;
    mbar_wait(&mbar[w.wl][sl], (unsigned)(w.jc / kRing) & 1u);
    acc += chunk_gemv_smem(w.slot0 + sl * w.slotsz, R * tk.ns, kl, lane / R, R, zs + (int64_t)c * tk.ns, lane);
    __syncwarp();
    ++w.jc;
    ring_next(a, w, mbar);
    if (PROF) tl_mark(w, 3);
  }
  if (PROF) {
    w.acc[4] += 1;
    w.acc[5] += tk.c1 - tk.c0;
  }
  if (lane < R) dred[tk.cboff * R + lane] = acc;  // partial of rows first + lane over the piece's columns
}

// Run this CTA's items of a coupling program.  MODE 0 (slab start): rhs rows, item
// dst kind 0 -> the subtree's shared rhs_s, kind 1 -> tbuf.  MODE 1 (after a slab):
// out[dst] += sum, the rows of another stage's right-hand side.  srcs: source table.
template <int MODE>
__device__ __forceinline__ void run_program(const int4 hd, const int2 *items, const int *ecol, const double *vk,
                                            const double *rhs, double *out, const SubView &sv, double *tbuf,
                                            const double *const *srcs, bool wide16 = false) {
  const int nth = blockDim.x;
  constexpr int kIdx = (1 << 28) - 1;
  // threads per item: spread an item's entries over tpi lanes when there are few
  // items (so every load of the step is in flight at once)
  int tpi = 1;
  while (tpi < 32 && hd.y * tpi * 2 <= nth) tpi *= 2;
  if (tpi == 1 && hd.y <= nth && wide16) {
    // one item per thread (a subtree CTA's rows): 16 entries per step -- the step is a
    // chain of two memory round trips (entry table, then sources), so a 19-entry mass
    // matrix row takes two steps instead of three; same accumulation order
    const int it = threadIdx.x;
    const bool live = it < hd.y;
    const int2 io = live ? items[hd.x + it] : make_int2(0, -1);
    double acc = io.y >= 0 ? rhs[io.y] : 0.0;
    for (int s0 = 0; s0 < hd.w; s0 += 16) {
      int cc[16];
      double vv[16], xv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int64_t id = hd.z + (int64_t)(s0 + q) * hd.y + it;
        const bool ok = live && s0 + q < hd.w;
        cc[q] = ok ? __ldg(ecol + id) : 0;
        vv[q] = ok ? __ldg(vk + id) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) xv[q] = srcs[cc[q] >> 28][cc[q] & kIdx];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc = fma(vv[q], xv[q], acc);
    }
    if (live) {
      const int kind = io.x >> 29, di = io.x & ((1 << 29) - 1);
      if (MODE == 1) out[io.x] += acc;
      else if (kind == 0) sv.rhs_s[di] = acc;
      else tbuf[di] = acc;
    }
  } else if (tpi == 1) {
    for (int i0 = threadIdx.x; i0 < hd.y; i0 += 2 * nth) {
      const int it[2] = {i0, i0 + nth};
      const bool live[2] = {true, i0 + nth < hd.y};
      double acc[2];
      int2 io[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        io[r] = live[r] ? items[hd.x + it[r]] : make_int2(0, -1);
        acc[r] = io[r].y >= 0 ? rhs[io[r].y] : 0.0;
      }
      for (int s0 = 0; s0 < hd.w; s0 += 8) {
        int cc[2][8];
        double vv[2][8];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int64_t id = hd.z + (int64_t)(s0 + q) * hd.y + it[r];
            const bool ok = live[r] && s0 + q < hd.w;
            cc[r][q] = ok ? __ldg(ecol + id) : 0;
            vv[r][q] = ok ? __ldg(vk + id) : 0.0;
          }
        double xv[2][8];  // all 16 loads in flight together
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) xv[r][q] = srcs[cc[r][q] >> 28][cc[r][q] & kIdx];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[r] = fma(vv[r][q], xv[r][q], acc[r]);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!live[r]) continue;
        const int kind = io[r].x >> 29, di = io[r].x & ((1 << 29) - 1);
        if (MODE == 1) out[io[r].x] += acc[r];
        else if (kind == 0) sv.rhs_s[di] = acc[r];
        else tbuf[di] = acc[r];
      }
    }
  } else {
    const int g = threadIdx.x / tpi, part = threadIdx.x & (tpi - 1), ng = nth / tpi;
    for (int base = 0; base < hd.y; base += ng) {  // uniform trip count per warp
      const int it = base + g;
      const bool live = it < hd.y;
      const int2 io = live ? items[hd.x + it] : make_int2(0, -1);
      double acc = 0.0;
      for (int s0 = part; s0 < hd.w; s0 += 16 * tpi) {
        int cc[16];
        double vv[16], xv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int sl = s0 + q * tpi;
          const bool ok = live && sl < hd.w;
          const int64_t id = hd.z + (int64_t)sl * hd.y + it;
          cc[q] = ok ? __ldg(ecol + id) : 0;
          vv[q] = ok ? __ldg(vk + id) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) xv[q] = srcs[cc[q] >> 28][cc[q] & kIdx];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = fma(vv[q], xv[q], acc);
      }
      for (int o = 1; o < tpi; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (live && part == 0) {
        acc += io.y >= 0 ? rhs[io.y] : 0.0;
        const int kind = io.x >> 29, di = io.x & ((1 << 29) - 1);
        if (MODE == 1) out[io.x] += acc;
        else if (kind == 0) sv.rhs_s[di] = acc;
        else tbuf[di] = acc;
      }
    }
  }
}

// Up to three sweeps of one pipelined launch, one cluster each (cluster i runs st[i]).
struct SweepMulti {
  SweepArgs st[3];
  int first[4];  // grid-family launch: stage i owns CTAs [first[i], first[i+1])
  int nst;       // stages; cluster index nst (if launched) is the L2 prefetch cluster
  int pf_dist;   // prefetch slabs [k + 1, k + pf_dist] while a stage works on slab k
};

// L2 prefetch cluster (cluster launch only): the sweeps stream every slab's factor
// and dense-top rows once, through per-warp TMA rings whose depth shared memory
// caps, so each level waits on an HBM round trip.  Idle SMs pull the next slabs'
// data into L2 (126 MB) while the stages work, so the rings hit L2 instead
// (~250 vs ~600+ cycles).  Pure hint: no effect on results.
__device__ __forceinline__ void l2_prefetch_range(const void *base, int64_t bytes, int part, int nparts, int lane) {
  uintptr_t b0 = reinterpret_cast<uintptr_t>(base), b1 = b0 + (uintptr_t)bytes;
  b0 = (b0 + 15) & ~(uintptr_t)15;
  b1 &= ~(uintptr_t)15;
  if (b1 <= b0) return;
  const uintptr_t len = b1 - b0, per = ((len + nparts - 1) / nparts + 15) & ~(uintptr_t)15;
  const uintptr_t p0 = b0 + (uintptr_t)part * per, p1 = min(b1, p0 + per);
  constexpr uintptr_t kChunk = 32768;
  for (uintptr_t c = p0 + (uintptr_t)lane * kChunk; c < p1; c += 32 * kChunk) {
    const unsigned sz = (unsigned)min(kChunk, p1 - c);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(c), "r"(sz) : "memory");
  }
}

__device__ void l2_prefetch_cluster(const SweepMulti &m, int crank) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int next[3] = {0, 0, 0};
  unsigned long long last_change;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(last_change));
  long long seen[3] = {-2, -2, -2};
  for (;;) {
    bool all = true, moved = false;
    for (int s = 0; s < m.nst; ++s) {
      const SweepArgs &a = m.st[s];
      if (next[s] >= a.nslab) continue;
      all = false;
      unsigned long long v;
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.progress) : "memory");
      const long long cur = (int)(v >> 32) == a.epoch ? (long long)(v & 0xffffffffu) : -1;
      if (cur != seen[s]) {
        seen[s] = cur;
        moved = true;
      }
      const long long lim = min((long long)a.nslab - 1, max(cur, 0LL) + m.pf_dist);
      for (; next[s] <= lim; ++next[s]) {
        const int j = next[s];
        l2_prefetch_range(a.factors + (int64_t)j * a.fstride, a.fstride * 8, crank, 16, lane);
        if (a.dense && a.kstride) l2_prefetch_range(a.ktop + (int64_t)j * a.kstride, a.kstride * 8, crank, 16, lane);
        if (a.prog_hdr && a.prog_per_slab)
          l2_prefetch_range(a.prog_vals + (int64_t)j * a.prog_nent, a.prog_nent * 8, crank, 16, lane);
        if (a.post_hdr && a.post_per_slab)
          l2_prefetch_range(a.post_vals + (int64_t)j * a.post_nent, a.post_nent * 8, crank, 16, lane);
      }
    }
    if (all) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (moved) last_change = t;
    else if (t - last_change > 4000000000ull) return;  // stages not progressing: stop hinting
    __nanosleep(256);
  }
}

template <bool PROF>
__global__ void __launch_bounds__(512, 1) nd_sweep_kernel(const __grid_constant__ SweepMulti m) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long mbar[16][kRing];
  __shared__ SweepArgs sa;
  __shared__ const double *s_src[8];  // coupling sources of the current slab (by source id)
  // grid-family launch (no clusters, software barriers): stages own CTA ranges;
  // cluster launch: stage = cluster index, rank = rank in the cluster
  const bool grid = m.st[0].gbar != nullptr;
  unsigned cid;
  int crank;
  if (!grid && (int)cluster_index() >= m.nst) {
    l2_prefetch_cluster(m, (int)cluster_rank());
    return;
  }
  if (grid) {
    const int b = (int)blockIdx.x;
    cid = b >= m.first[2] ? 2u : (b >= m.first[1] ? 1u : 0u);
    crank = b - m.first[cid];
  } else {
    cid = cluster_index();
    crank = (int)cluster_rank();
  }
  if (threadIdx.x == 0) {
    if (cid == 0) sa = m.st[0];
    else if (cid == 1) sa = m.st[1];
    else sa = m.st[2];
  }
  __syncthreads();
  const SweepArgs &a = sa;
  unsigned gphase = 0;  // grid barrier: top bit of the barrier word after the last completion
  if (a.gbar && threadIdx.x == 0) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gphase) : "l"(a.gbar) : "memory");
    gphase &= 0x80000000u;
  }
  WarpCtx w;
  w.lane = threadIdx.x & 31;
  w.wl = threadIdx.x >> 5;
  const int lane = w.lane, wl = w.wl;
  // (top-phase task lists are interleaved across CTAs: global warp wl * ncta + crank)
  w.v = sm + wl * a.vstride;
  w.slot0 = w.v + (a.vstride - kRing * a.slot);
  w.slotsz = a.slot;
  w.jc = w.icount = w.rt = w.rc = w.rslab = 0;
  for (int i = 0; i < 10; ++i) w.acc[i] = 0;
  w.tl_out = nullptr;
  w.tl_n = 0;
  long long tb = 0;
  SubView sv;
  sv.ys = sm + (int64_t)a.warps * a.vstride;
  sv.xs = sv.ys + a.sub_len;
  sv.cbs = sv.xs + a.sub_len;
  sv.rhs_s = sv.cbs + a.sub_cb;
  sv.zs = sv.rhs_s + a.sub_len;
  sv.ftab = nullptr;
  sv.btab = nullptr;
  if (a.tab_ints) {  // this CTA's subtree front tables, resident for the whole launch
    int *tb = reinterpret_cast<int *>((reinterpret_cast<uintptr_t>(sv.zs + a.zlen) + 15) & ~(uintptr_t)15);
    const int o = a.tab_ptr[crank], nt = a.tab_ptr[crank + 1] - o;
    for (int i = threadIdx.x; i < nt; i += blockDim.x) tb[i] = a.tab[o + i];
    sv.ftab = tb;
    sv.btab = reinterpret_cast<const unsigned short *>(tb + a.tab_nf[crank]);
    if (threadIdx.x == 0) s_bband = a.tab_band + a.tab_band_ptr[crank];
    __syncthreads();
  }
  sv.first = a.sub_info[4 * crank + 0];
  sv.len = a.sub_info[4 * crank + 1];
  sv.cbfirst = a.sub_info[4 * crank + 2];
  {
    // copy this warp's task list and level bounds into shared memory (static for
    // the whole sweep: no global round trip per level or task afterwards)
    const int gid = crank * a.warps + wl;
    const uintptr_t base =
        (reinterpret_cast<uintptr_t>(sv.zs + a.zlen) + 15 + (size_t)a.tab_ints * 4) & ~(uintptr_t)15;
    char *area = reinterpret_cast<char *>(base) + (size_t)wl * a.tstride;
    int *bnd = reinterpret_cast<int *>(area);
    SweepTask *tl = reinterpret_cast<SweepTask *>(area + ((a.nl + 1 + 3) / 4) * 16);
    const int o = a.wl_off[gid];
    const int nt = a.wl_off[gid + 1] - o;
    for (int i = lane; i <= a.nl; i += 32) bnd[i] = a.wl_bnd[(size_t)gid * (a.nl + 1) + i];
    const int4 *src = reinterpret_cast<const int4 *>(a.wl_tasks + o);
    int4 *dst = reinterpret_cast<int4 *>(tl);
    for (int i = lane; i < 2 * nt; i += 32) dst[i] = src[i];
    __syncwarp();
    w.tl = tl;
    w.bnd = bnd;
    w.nt = nt;
    if (nt > 0) w.rc = first_item(tl[0]);
  }
  if (lane == 0) {
    const unsigned cnt = a.ldgsts ? 32u : 1u;  // warp-wide cp.async: one arrival per lane
    for (int r = 0; r < kRing; ++r)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&mbar[wl][r])), "r"(cnt) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  if (!a.null_work && w.nt > 0)  // fill the ring
    for (int r = 0; r < kRing; ++r) ring_next(a, w, mbar);
  __syncwarp();
  const int64_t n = a.n;
  int step = 0;
  const bool early = a.early_cpl && !a.post_hdr && a.prog_hdr;
  const bool has_sub = sv.len > 0;
  sweep_trace(a, step, crank);
  for (int k = 0; k < a.nslab; ++k) {
    const double *rhs = a.rhsp + (int64_t)k * n;
    double *x = a.xp + (int64_t)k * n;
    if (a.progress && threadIdx.x == 0 && crank == 0) {
      const unsigned long long v = ((unsigned long long)(unsigned)a.epoch << 32) | (unsigned)k;
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(a.progress), "l"(v) : "memory");
    }
    if (a.dense && a.kpref && lane == 0 && !a.null_work) {
      // the dense-top K rows of this warp for slab k, into L2 one slab phase ahead of
      // their use (the ring then streams them from L2)
      for (int ti = w.bnd[a.nsub + a.ntop]; ti < w.bnd[a.nsub + a.ntop + 1]; ++ti) {
        const SweepTask &t = w.tl[ti];
        const double *src = a.ktop + (int64_t)k * a.kstride + t.foff;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"((unsigned)(t.c1 * t.bsz * 8))
                     : "memory");
      }
    }
    if (a.prog_hdr && !a.null_work) {
      // fused coupling (CTA-local): rhs_k + sum_c coef_c C_c src_c for this CTA's items.
      // Sources by id: 0 x_{k-1}, 1 x_{k-1} of the own subtree (shared memory),
      // 2 x_{k-2}, 3/4 external stages' outputs at slab k; sources that do not exist
      // yet read zeros.  (Early coupling: a subtree CTA arrives here straight from its
      // subtree backward of slab k-1, with no grid barrier in between.)
      if (threadIdx.x == 0) {
        s_src[0] = k >= 1 ? a.xp + (int64_t)(k - 1) * n : a.zero;
        s_src[1] = k >= 1 ? (const double *)sv.xs : a.zero;
        s_src[2] = k >= 2 ? a.xp + (int64_t)(k - 2) * n : a.zero;
        s_src[3] = a.ext_xp[0] ? a.ext_xp[0] + (int64_t)k * a.ext_n[0] : a.zero;
        s_src[4] = a.ext_xp[1] ? a.ext_xp[1] + (int64_t)k * a.ext_n[1] : a.zero;
        s_src[5] = s_src[6] = s_src[7] = a.zero;  // 5: own x_k (post-slab program only)
      }
      // wait until every CTA of each producer has published slab k (pipelined launch),
      // and, for a CTA without a subtree in early mode, until every subtree CTA of this
      // stage has published slab k-1
      const int nprod = (a.nwait > 0 ? a.ext_ncta[0] : 0) + (a.nwait > 1 ? a.ext_ncta[1] : 0);
      const int nsubw = (early && !has_sub && k >= 1) ? a.nroots : 0;
      for (int t = threadIdx.x; t < nprod + nsubw; t += blockDim.x) {
        const int *f;
        if (t < nprod) {
          const int e = t < a.ext_ncta[0] ? 0 : 1, c = e ? t - a.ext_ncta[0] : t;
          f = a.flag_in[e] + (int64_t)k * a.ext_ncta[e] + c;
        } else {
          f = a.flag_out + (int64_t)(k - 1) * a.ncta + (t - nprod);
        }
        if (ld_acquire_gpu(f) != a.epoch) {
          // the poll loop is on the critical path of every slab: only the flag load per
          // iteration; the clock and the fault word are checked every 256 polls
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          for (unsigned it = 1; ld_acquire_gpu(f) != a.epoch; ++it) {
            if (it & 255u) continue;
            if (*(volatile int *)a.fault) break;  // an earlier wait already gave up
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (t1 - t0 > 4000000000ull) {
              // 4 s: a producer is not running (not co-resident).  Record the fault
              // instead of trapping (a trap kills the CUDA context); the stages run
              // to completion without further waits and the host raises STMHD_CUDA.
              atomicExch(a.fault, 1);
              *(volatile int *)a.fault_host = 1;
              __threadfence_system();
              break;
            }
          }
        }
      }
      __syncthreads();
      const double *vk = a.prog_vals + (a.prog_per_slab ? (int64_t)k * a.prog_nent : 0);
      long long tp0 = pclock<PROF>();
      run_program<0>(a.prog_hdr[crank], a.prog_items, a.prog_ecol, vk, rhs, nullptr, sv, a.tbuf, s_src, a.cpl16 != 0);
      if (PROF) w.acc[9] += pclock<PROF>() - tp0;
      tb = pclock<PROF>(); __syncthreads(); if (PROF) w.acc[3] += pclock<PROF>() - tb;
      sweep_trace(a, step, crank);
    }
    const double *F = a.factors + (int64_t)k * a.fstride;
    // phase levels of this warp's list: subtree forward (CTA-local), top forward,
    // top backward (cluster-wide), subtree backward (CTA-local)
    int L = 0;
    unsigned long long tph0 = 0;
    if (PROF && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tph0));
    for (int h = 0; h < a.nsub; ++h, ++L) {
      const int t1 = a.null_work ? w.bnd[L] : w.bnd[L + 1];
      if (PROF) {
        w.tl_out = (a.tline && k == 1 && crank == 0) ? a.tline + (size_t)wl * 128 : nullptr;
        tl_mark(w, 1);
      }
      for (int ti = w.bnd[L]; ti < t1; ++ti) forward_task<true, PROF>(a, w.tl[ti], F, rhs, sv, w, mbar);
      if (PROF) tl_mark(w, 4);
      tb = pclock<PROF>(); __syncthreads(); if (PROF) w.acc[3] += pclock<PROF>() - tb;
    }
    if (PROF && threadIdx.x == 0 && a.pcta && k == 1) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.pcta[2 * crank] = t - tph0;
    }
    if (a.nsub || a.prog_hdr) {  // subtree roots' updates and coupled top rows visible
      tb = pclock<PROF>(); sweep_barrier(a, crank, gphase); if (PROF) w.acc[3] += pclock<PROF>() - tb;
      sweep_trace(a, step, crank);
    }
    // band forward levels (cluster/grid-wide tree levels below the K region)
    for (int t = 0; t < a.ntop; ++t, ++L) {
      const int t1 = a.null_work ? w.bnd[L] : w.bnd[L + 1];
      for (int ti = w.bnd[L]; ti < t1; ++ti) forward_task<false, PROF>(a, w.tl[ti], F, rhs, sv, w, mbar);
      tb = pclock<PROF>(); sweep_barrier(a, crank, gphase); if (PROF) w.acc[3] += pclock<PROF>() - tb;
      sweep_trace(a, step, crank);
    }
    if (a.dense) {
      // z_T = coupled rhs of the K unknowns + the updates of the K region's children
      // (all CTAs gather the whole vector), then x_T = K z_T as row tasks
      if (PROF) tl_mark(w, 5);
      const double *rt = a.prog_hdr ? a.tbuf : rhs;
      for (int i0 = threadIdx.x; i0 < a.kpad; i0 += 4 * blockDim.x) {
        int4 t0[4], t1[4];  // four entries per thread: every table load, then every value load in flight
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = i0 + q * blockDim.x;
          t0[q] = i < a.ntT ? a.ztab[2 * i] : make_int4(-1, -1, -1, -1);
          t1[q] = i < a.ntT ? a.ztab[2 * i + 1] : make_int4(-1, -1, -1, -1);
        }
        double z[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double r0 = t0[q].x >= 0 ? rt[t0[q].x] : 0.0;
          const double c0 = t0[q].y >= 0 ? a.cbv[t0[q].y] : 0.0, c1 = t0[q].z >= 0 ? a.cbv[t0[q].z] : 0.0;
          const double c2 = t0[q].w >= 0 ? a.cbv[t0[q].w] : 0.0, c3 = t1[q].x >= 0 ? a.cbv[t1[q].x] : 0.0;
          z[q] = r0 + ((c0 + c1) + (c2 + c3));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i0 + q * (int)blockDim.x < a.kpad) sv.zs[i0 + q * blockDim.x] = z[q];
      }
      tb = pclock<PROF>(); __syncthreads(); if (PROF) w.acc[3] += pclock<PROF>() - tb;
      sweep_trace(a, step, crank);
      const int t1 = a.null_work ? w.bnd[L] : w.bnd[L + 1];
      if (PROF) tl_mark(w, 1);
      double *dred = sv.zs + a.kpad;
      for (int ti = w.bnd[L]; ti < t1; ++ti) dense_task<PROF>(a, w.tl[ti], sv.zs, dred, w, mbar);
      if (PROF) tl_mark(w, 4);
      ++L;
      __syncthreads();
      // x_T rows of this CTA's groups: the pieces' partials summed in a fixed order
      for (int t = threadIdx.x; t < a.dgroups * a.kr; t += blockDim.x) {
        const int j = t / a.kr, r = t - j * a.kr;
        const int row = (crank + a.ncta * j) * a.kr + r;
        if (row < a.ntT) {
          const double *pr = dred + (int64_t)j * a.dpieces * a.kr + r;
          double sum = pr[0];
          for (int q = 1; q < a.dpieces; ++q) sum += pr[q * a.kr];
          x[a.ztab[2 * row].x] = sum;
        }
      }
      tb = pclock<PROF>(); sweep_barrier(a, crank, gphase); if (PROF) w.acc[3] += pclock<PROF>() - tb;  // x_T visible
      if (a.tab_ints) {  // stage x_T in shared memory for the subtree backward tables
        for (int i = threadIdx.x; i < a.ntT; i += blockDim.x) sv.zs[i] = x[a.ztab[2 * i].x];
        __syncthreads();
      }
      sweep_trace(a, step, crank);
    }
    // band backward levels
    for (int t = a.ntop - 1; t >= 0; --t, ++L) {
      const int t1 = a.null_work ? w.bnd[L] : w.bnd[L + 1];
      for (int ti = w.bnd[L]; ti < t1; ++ti) backward_task<false, PROF>(a, w.tl[ti], F, x, sv, w, mbar);
      if (t > 0 || a.nsub || k + 1 < a.nslab) {
        tb = pclock<PROF>();
        sweep_barrier(a, crank, gphase);
        if (PROF) w.acc[3] += pclock<PROF>() - tb;
      }
      sweep_trace(a, step, crank);
    }
    if (PROF && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tph0));
    for (int h = a.nsub - 1; h >= 0; --h, ++L) {
      const int t1 = a.null_work ? w.bnd[L] : w.bnd[L + 1];
      if (PROF) tl_mark(w, 5);
      for (int ti = w.bnd[L]; ti < t1; ++ti) backward_task<true, PROF>(a, w.tl[ti], F, x, sv, w, mbar);
      if (PROF) tl_mark(w, 6);
      tb = pclock<PROF>(); __syncthreads(); if (PROF) w.acc[3] += pclock<PROF>() - tb;
    }
    if (PROF && threadIdx.x == 0 && a.pcta && k == 1) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.pcta[2 * crank + 1] = t - tph0;
    }
    if (a.post_hdr && !a.null_work) {
      // post-slab program: rows of another stage's right-hand side from this stage's
      // x_k (all CTAs' parts: cluster barrier) and external sources at slab k
      sweep_barrier(a, crank, gphase);
      if (threadIdx.x == 0) {
        s_src[3] = a.ext_xp[0] ? a.ext_xp[0] + (int64_t)k * a.ext_n[0] : a.zero;
        s_src[4] = a.ext_xp[1] ? a.ext_xp[1] + (int64_t)k * a.ext_n[1] : a.zero;
        s_src[5] = a.xp + (int64_t)k * n;
      }
      __syncthreads();
      const double *vk = a.post_vals + (a.post_per_slab ? (int64_t)k * a.post_nent : 0);
      run_program<1>(a.post_hdr[crank], a.post_items, a.post_ecol, vk, nullptr, a.post_out + (int64_t)k * a.post_n,
                     sv, nullptr, s_src);
    }
    if (a.flag_out) {  // publish this CTA's part of x_k at gpu scope (consumers, early coupling)
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(a.flag_out + (int64_t)k * a.ncta + crank, a.epoch);
    }
    if (early) {
      // no grid barrier: a subtree CTA's next coupling reads only its own x_k (shared
      // memory) and separator values final since the band levels; the CTAs without a
      // subtree wait for the subtree CTAs' flags before coupling the top rows
      if (k + 1 < a.nslab) sweep_trace(a, step, crank);
    } else if (a.nsub && k + 1 < a.nslab) {  // x_k visible to every CTA's next coupling
      tb = pclock<PROF>(); sweep_barrier(a, crank, gphase); if (PROF) w.acc[3] += pclock<PROF>() - tb;
      sweep_trace(a, step, crank);
    }
  }
  if (PROF && lane == 0 && a.prof)  // (only the traced stage of a pipelined launch has counters)
    for (int i = 0; i < 10; ++i) a.prof[(crank * a.warps + wl) * 10 + i] = (unsigned long long)w.acc[i];
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
// ---------------------------------------------------------------------------
// Fused slab-coupling program (built once per coupling set and plan): the coupled
// right-hand-side rows are split by owner -- subtree rows to their CTA (written to
// its shared memory; x_{k-1} of the same subtree read from shared memory), top rows
// balanced over the CTAs (written to tbuf).  Each entry is (source id << 28 | index)
// with sources 0 x_{k-1}, 1 own-subtree x_{k-1} (shared), 2 x_{k-2}, 3 + e external
// stage e at slab k; its value is gathered per launch by cpl_vals_kernel.
static const CplProgram &get_program(const NDSweepPlan &sp, const NDPlan &p, const SweepCoupling *cpl, int ncpl,
                                     const std::vector<int> *const *ext_pos, cudaStream_t s) {
  std::vector<const void *> key;
  for (int c = 0; c < ncpl; ++c) {
    key.push_back(cpl[c].rowptr);
    key.push_back(cpl[c].rowend);
    key.push_back(cpl[c].col);
    key.push_back(reinterpret_cast<const void *>((intptr_t)(cpl[c].col_off * 16 + cpl[c].lag * 4 + cpl[c].ext + 1)));
  }
  auto it = sp.prog_cache.find(key);
  if (it != sp.prog_cache.end()) return *it->second;
  auto pg = std::make_unique<CplProgram>();
  const int64_t n = p.n;
  const int ncta = sp.ncta;
  std::vector<int> owner(n, -1);
  for (int c = 0; c < ncta; ++c)
    for (int64_t q = sp.sub_info_h[4 * c]; q < sp.sub_info_h[4 * c] + sp.sub_info_h[4 * c + 1]; ++q) owner[q] = c;
  struct Ent {
    int col, cid, e;
  };
  struct Item {
    int dst, rhs;
    std::vector<Ent> ents;
  };
  std::vector<std::vector<Item>> items(ncta);
  // coupling rows on the host: [beg[i], end[i]) and columns
  std::vector<std::vector<int>> rb(ncpl), re(ncpl), cl(ncpl);
  for (int c = 0; c < ncpl; ++c) {
    rb[c].resize(n + 1);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(rb[c].data(), cpl[c].rowptr, (n + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    re[c].resize(n);
    if (cpl[c].rowend)
      STMHD_CUDA_CHECK(cudaMemcpyAsync(re[c].data(), cpl[c].rowend, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    if (!cpl[c].rowend)
      for (int64_t i = 0; i < n; ++i) re[c][i] = rb[c][i + 1];
    int mx = 0;
    for (int64_t i = 0; i < n; ++i) mx = std::max(mx, re[c][i]);
    cl[c].resize(std::max(mx, 1));
    if (mx) STMHD_CUDA_CHECK(cudaMemcpy(cl[c].data(), cpl[c].col, mx * sizeof(int), cudaMemcpyDeviceToHost));
  }
  auto entries_of = [&](int64_t q, Item &itm, int own) {
    const int io = sp.iperm_h[q];
    for (int c = 0; c < ncpl; ++c)
      for (int e = rb[c][io]; e < re[c][io]; ++e) {
        const int jr = cl[c][e] - cpl[c].col_off;
        int enc;
        if (cpl[c].ext >= 0) {
          const std::vector<int> &ep = *ext_pos[cpl[c].ext];
          require(jr >= 0 && jr < (int)ep.size(), "sweep coupling: external column out of range");
          enc = ((3 + cpl[c].ext) << 28) | ep[jr];
        } else {
          require(jr >= 0 && jr < n && (cpl[c].lag == 1 || cpl[c].lag == 2), "sweep coupling: bad column or lag");
          const int j = sp.pos_h[jr];
          if (cpl[c].lag == 2) enc = (2 << 28) | j;
          else if (own >= 0 && owner[j] == own) enc = (1 << 28) | (int)(j - sp.sub_info_h[4 * own]);
          else enc = j;
        }
        itm.ents.push_back({enc, c, e});
      }
  };
  std::vector<int64_t> top_rows;
  for (int64_t q = 0; q < n; ++q)
    if (owner[q] < 0) top_rows.push_back(q);
  for (int64_t q = 0; q < n; ++q) {  // subtree rows -> their CTA (shared memory)
    const int o = owner[q];
    if (o < 0) continue;
    Item itm{(int)(q - sp.sub_info_h[4 * o]), (int)q, {}};
    entries_of(q, itm, o);
    items[o].push_back(std::move(itm));
  }
  // top rows -> balanced over the CTAs (tbuf); only over the CTAs that own no subtree
  // when there are some (the early-coupling schedule relies on it)
  std::vector<int> load(ncta);
  bool idle = false;
  for (int c = 0; c < ncta; ++c) idle |= sp.sub_info_h[4 * c + 1] == 0;
  for (int c = 0; c < ncta; ++c)
    load[c] = (idle && sp.sub_info_h[4 * c + 1] > 0) ? INT_MAX / 2 : (int)items[c].size();
  for (int64_t q : top_rows) {
    const int d = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    ++load[d];
    Item itm{(1 << 29) | (int)q, (int)q, {}};
    entries_of(q, itm, -1);
    items[d].push_back(std::move(itm));
  }
  require(n < (1 << 28), "sweep coupling program: index overflow");
  std::vector<int4> hdr(ncta);
  std::vector<int2> it2;
  std::vector<int> ecol;
  std::vector<int2> esrc;
  for (int c = 0; c < ncta; ++c) {
    int width = 0;
    for (auto &x : items[c]) width = std::max(width, (int)x.ents.size());
    const int ni = (int)items[c].size();
    hdr[c] = make_int4((int)it2.size(), ni, (int)ecol.size(), width);
    for (auto &x : items[c]) it2.push_back(make_int2(x.dst, x.rhs));
    const size_t base = ecol.size();
    ecol.resize(base + (size_t)width * ni, 0);  // pad: source 0 index 0 with value 0
    esrc.resize(base + (size_t)width * ni, make_int2(-1, 0));
    for (int i = 0; i < ni; ++i)
      for (int sl = 0; sl < (int)items[c][i].ents.size(); ++sl) {
        const Ent &en = items[c][i].ents[sl];
        ecol[base + (size_t)sl * ni + i] = en.col;
        esrc[base + (size_t)sl * ni + i] = make_int2(en.cid, en.e);
      }
  }
  if (ecol.empty()) {
    ecol.push_back(0);
    esrc.push_back(make_int2(-1, 0));
  }
  if (it2.empty()) it2.push_back(make_int2(0, -1));
  pg->nent = (int64_t)ecol.size();
  pg->hdr = upload_vec(hdr, s);
  pg->items = upload_vec(it2, s);
  pg->ecol = upload_vec(ecol, s);
  pg->esrc = upload_vec(esrc, s);
  pg->ok = true;
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  if (getenv("STMHD_SWEEP_TRACE")) {
    fprintf(stderr, "[sweep-prog] ncpl %d top rows %zu nent %lld | per CTA items/width:", ncpl, top_rows.size(),
            (long long)pg->nent);
    for (int c = 0; c < ncta; ++c) fprintf(stderr, " %d/%d", hdr[c].y, hdr[c].w);
    fprintf(stderr, "\n");
  }
  const CplProgram &ref = *pg;
  sp.prog_cache[key] = std::move(pg);
  return ref;
}

constexpr int kMaxCpl = 4;

struct CplVals {
  const double *val[kMaxCpl];
  int64_t stride[kMaxCpl], shift[kMaxCpl];
  double coef[kMaxCpl];
};

// vals[b][id] = coef * val_c[(b - shift_c) * stride_c + e] for the program entries
// (b = slab when any coupling has per-slab values, else a single block; blocks before
// the first one of a coupling are zero -- their source reads zeros anyway)
__global__ void cpl_vals_kernel(const int2 *esrc, int64_t nent, CplVals cv, int per_slab, double *vals) {
  const int b = blockIdx.y;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < nent; id += (int64_t)gridDim.x * blockDim.x) {
    const int2 sr = esrc[id];
    double v = 0.0;
    if (sr.x >= 0) {
      const int64_t blk = per_slab && cv.stride[sr.x] ? (int64_t)b - cv.shift[sr.x] : 0;
      if (blk >= 0) v = cv.coef[sr.x] * cv.val[sr.x][blk * cv.stride[sr.x] + sr.y];
    }
    vals[(int64_t)b * nent + id] = v;
  }
}

// ---------------------------------------------------------------------------
// Dense top operator K = (A^{-1})_TT, one per batch entry: push 32 identity columns
// at a time through the top supernodes' forward (FL) and backward (FU) factors --
// exactly the operations of the sweep's top levels, applied to a block of
// right-hand sides.  Warp per row, lane per column; fronts staged in shared memory.
struct TopKArgs {
  const TopSN *tsn;
  const int4 *tchild;
  const int *emap, *tidx, *bpos;
  const double *factors;
  int64_t fstride;
  int ntsn, nT, kpad, kr, nbatch, ncb;
  double *scratch;    // per CTA: Xw (nT x 32) | CBw (tcb_total x 32)
  int64_t scr_stride;
  double *K;          // [nbatch][nT][kpad]
  int64_t kstride;
};

// acc[i][h] = sum_k blk(r0 + i, k) V[k][lane + 32 h], i < 4 (rows >= nrows give 0), h < NC,
// for a factor block stored as row chunks [K][R] (element (r, k) at (r / R) * bsz + k * R +
// r % R).  Every factor load feeds NC x 32 columns.
template <int NC>
__device__ __forceinline__ void topk_rows4(const double *blk, int R, int bsz, int r0, int nrows, int K,
                                           const double *V, int lane, double (&acc)[4][NC]) {
  constexpr int CS = 32 * NC;
  const double *row[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = min(r0 + i, nrows - 1);
    row[i] = blk + (int64_t)(r / R) * bsz + (r % R);
#pragma unroll
    for (int h = 0; h < NC; ++h) acc[i][h] = 0.0;
  }
  int k = 0;
  for (; k + 4 <= K; k += 4) {
    double fv[4][4], vv[4][NC];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < NC; ++h) vv[j][h] = V[(k + j) * CS + lane + 32 * h];
#pragma unroll
      for (int i = 0; i < 4; ++i) fv[i][j] = __ldg(row[i] + (int64_t)(k + j) * R);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int h = 0; h < NC; ++h) acc[i][h] = fma(fv[i][j], vv[j][h], acc[i][h]);
  }
  for (; k < K; ++k) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double f = __ldg(row[i] + (int64_t)k * R);
#pragma unroll
      for (int h = 0; h < NC; ++h) acc[i][h] = fma(f, V[k * CS + lane + 32 * h], acc[i][h]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (r0 + i >= nrows)
#pragma unroll
      for (int h = 0; h < NC; ++h) acc[i][h] = 0.0;
}

// K = (A^{-1})_TT for every slab: item = (slab, block of 32 NC identity columns), lane
// column lane + 32 h; the columns are pushed through the top supernodes' own FL / FU
// blocks (forward in postorder, backward in reverse), so K reproduces exactly what the
// top tree levels of the sweep would compute.
template <int NC>
__global__ void __launch_bounds__(256 * NC) topk_kernel(TopKArgs g) {
  constexpr int CS = 32 * NC;
  extern __shared__ __align__(16) double V[];  // front x CS
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *Xw = g.scratch + (int64_t)blockIdx.x * g.scr_stride;
  double *CBw = Xw + (int64_t)g.nT * CS;
  const int nitems = g.nbatch * g.ncb;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int b = item / g.ncb, col = (item % g.ncb) * CS + lane;
    const double *F = g.factors + (int64_t)b * g.fstride;
    for (int si = 0; si < g.ntsn; ++si) {  // forward, postorder
      const TopSN t = g.tsn[si];
      const int f = t.ns + t.nb;
      for (int r = wl; r < f; r += nw) {
        const int ti = r < t.ns ? g.tidx[t.first + r] : -1;
#pragma unroll
        for (int h = 0; h < NC; ++h) V[r * CS + lane + 32 * h] = (ti == col + 32 * h) ? 1.0 : 0.0;
      }
      __syncthreads();
      for (int c = 0; c < t.nchild; ++c) {  // extend-add the top children's updates
        const int4 ch = g.tchild[t.child0 + c];
        const int cb0 = g.tsn[ch.x].tcb_off;
        for (int a = wl; a < ch.z; a += nw)
#pragma unroll
          for (int h = 0; h < NC; ++h)
            V[g.emap[ch.y + a] * CS + lane + 32 * h] += CBw[(int64_t)(cb0 + a) * CS + lane + 32 * h];
        __syncthreads();
      }
      for (int r0 = wl * 4; r0 < f; r0 += nw * 4) {  // 4 rows per warp, 16 factor loads in flight
        double acc[4][NC];
        topk_rows4<NC>(F + t.fl_off, t.rf, t.bszf, r0, f, t.ns, V, lane, acc);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = r0 + i;
          if (r >= f) break;
#pragma unroll
          for (int h = 0; h < NC; ++h) {
            if (r < t.ns) Xw[(int64_t)g.tidx[t.first + r] * CS + lane + 32 * h] = acc[i][h];  // y
            else CBw[(int64_t)(t.tcb_off + r - t.ns) * CS + lane + 32 * h] = V[r * CS + lane + 32 * h] - acc[i][h];
          }
        }
      }
      __syncthreads();
    }
    for (int si = g.ntsn - 1; si >= 0; --si) {  // backward, reverse postorder
      const TopSN t = g.tsn[si];
      const int f = t.ns + t.nb;
      for (int r = wl; r < f; r += nw) {
        const int pos = r < t.ns ? t.first + r : g.bpos[t.goff + r];
#pragma unroll
        for (int h = 0; h < NC; ++h)  // own y, or the ancestors' x
          V[r * CS + lane + 32 * h] = Xw[(int64_t)g.tidx[pos] * CS + lane + 32 * h];
      }
      __syncthreads();
      for (int k0 = wl * 4; k0 < t.ns; k0 += nw * 4) {
        double acc[4][NC];
        topk_rows4<NC>(F + t.fu_off, t.rb, t.bszb, k0, t.ns, f, V, lane, acc);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (k0 + i < t.ns)
#pragma unroll
            for (int h = 0; h < NC; ++h) Xw[(int64_t)g.tidx[t.first + k0 + i] * CS + lane + 32 * h] = acc[i][h];
      }
      __syncthreads();
    }
#pragma unroll
    for (int h = 0; h < NC; ++h)
      if (col + 32 * h < g.nT)
        for (int i = wl; i < g.nT; i += nw)  // row groups of kr: [group][col][kr]
          g.K[(int64_t)b * g.kstride + (int64_t)(i - i % g.kr) * g.kpad + (int64_t)(col + 32 * h) * g.kr + i % g.kr] =
              Xw[(int64_t)i * CS + lane + 32 * h];
    __syncthreads();
  }
}

// Tensor-core variant (FP64 mma.sync.m8n8k4): the same column pushes, 64 columns per
// item, each warp computing 8-row x 64-column tiles of FL V / FU V (one factor load
// per lane and k-step feeds 8 MMAs; the front block V is [row][kVS] in shared memory,
// row stride 72 doubles so the B-fragment loads of a k-step take two wavefronts).
// Identical operations up to the summation order inside each dot product.
constexpr int kVS = 68;  // row stride 544 B: the four rows of a half-warp B fragment hit distinct banks

// acc[j] += blk rows r0..r0+7 (x K) . V[:, 8j .. 8j+7]; lane holds C(row lane/4,
// cols 8j + 2(lane%4) + {0,1}).  blk is stored as row chunks [K][R].
__device__ __forceinline__ void topk_mma_tile(const double *__restrict__ blk, int R, int bsz, int r0, int nrows, int K,
                                              const double *V, int lane, double (&acc)[8][2]) {
  const int ar = r0 + (lane >> 2), kq = lane & 3;
  const bool rok = ar < nrows;
  const double *arow = blk + (int64_t)((rok ? ar : 0) / R) * bsz + ((rok ? ar : 0) % R);
  const double *vb = V + kq * kVS + (lane >> 2);
  int k = 0;
  const int k16 = K & ~15;
  // A fragments two k-blocks ahead (an: next block, an2: the one after): an L2 round
  // trip is longer than one block's 32 MMAs
  double an[4], an2[4];
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4) {
    an[s4] = (rok && k16 > 0) ? __ldg(arow + (int64_t)(4 * s4 + kq) * R) : 0.0;
    an2[s4] = (rok && 16 < k16) ? __ldg(arow + (int64_t)(16 + 4 * s4 + kq) * R) : 0.0;
  }
  for (; k < k16; k += 16) {
    double a[4];
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
      a[s4] = an[s4];
      an[s4] = an2[s4];
      an2[s4] = (rok && k + 32 < k16) ? __ldg(arow + (int64_t)(k + 32 + 4 * s4 + kq) * R) : 0.0;
    }
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4) {
      const double *vk = vb + (k + 4 * s4) * kVS;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double b = vk[8 * j];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[j][0]), "+d"(acc[j][1])
                     : "d"(a[s4]), "d"(b));
      }
    }
  }
  for (; k < K; k += 4) {
    const bool kok = k + kq < K;
    const double a = (rok && kok) ? __ldg(arow + (int64_t)(k + kq) * R) : 0.0;
    const double *vk = vb + k * kVS;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double b = kok ? vk[8 * j] : 0.0;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[j][0]), "+d"(acc[j][1])
                   : "d"(a), "d"(b));
    }
  }
}

__global__ void __launch_bounds__(512) topk_mma_kernel(TopKArgs g) {
  constexpr int CS = 64;
  extern __shared__ __align__(16) double V[];  // front x kVS
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *Xw = g.scratch + (int64_t)blockIdx.x * g.scr_stride;
  double *CBw = Xw + (int64_t)g.nT * CS;
  const int nitems = g.nbatch * g.ncb;
  const int crow = lane >> 2, ccol = 2 * (lane & 3);
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int b = item / g.ncb, col0 = (item % g.ncb) * CS;
    const double *F = g.factors + (int64_t)b * g.fstride;
    for (int si = 0; si < g.ntsn; ++si) {  // forward, postorder
      const TopSN t = g.tsn[si];
      const int f = t.ns + t.nb;
      // a warp per row, a column pair per lane: one index load per row (broadcast),
      // coalesced 16-byte global accesses, conflict-free 512-byte shared-memory rows
      for (int r = wl; r < f; r += nw) {
        const int ti = r < t.ns ? g.tidx[t.first + r] : -1;
        const int c = 2 * lane;
        *reinterpret_cast<double2 *>(V + r * kVS + c) =
            make_double2(ti == col0 + c ? 1.0 : 0.0, ti == col0 + c + 1 ? 1.0 : 0.0);
      }
      __syncthreads();
      for (int c = 0; c < t.nchild; ++c) {  // extend-add the top children's updates
        const int4 ch = g.tchild[t.child0 + c];
        const int cb0 = g.tsn[ch.x].tcb_off;
        for (int a0 = wl; a0 < ch.z; a0 += 2 * nw) {  // two rows per warp in flight
          const int a1 = a0 + nw;
          const double2 v0 = reinterpret_cast<const double2 *>(CBw + (int64_t)(cb0 + a0) * CS)[lane];
          const double2 v1 = a1 < ch.z ? reinterpret_cast<const double2 *>(CBw + (int64_t)(cb0 + a1) * CS)[lane]
                                       : make_double2(0.0, 0.0);
          double2 *d0 = reinterpret_cast<double2 *>(V + g.emap[ch.y + a0] * kVS) + lane;
          double2 w0 = *d0;
          w0.x += v0.x;
          w0.y += v0.y;
          *d0 = w0;
          if (a1 < ch.z) {
            double2 *d1 = reinterpret_cast<double2 *>(V + g.emap[ch.y + a1] * kVS) + lane;
            double2 w1 = *d1;
            w1.x += v1.x;
            w1.y += v1.y;
            *d1 = w1;
          }
        }
        __syncthreads();
      }
      for (int r0 = wl * 8; r0 < f; r0 += nw * 8) {
        double acc[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
        topk_mma_tile(F + t.fl_off, t.rf, t.bszf, r0, f, t.ns, V, lane, acc);
        const int r = r0 + crow;
        if (r < f) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int c = 8 * j + ccol + i;
              if (r < t.ns) Xw[(int64_t)g.tidx[t.first + r] * CS + c] = acc[j][i];  // y
              else CBw[(int64_t)(t.tcb_off + r - t.ns) * CS + c] = V[r * kVS + c] - acc[j][i];
            }
        }
      }
      __syncthreads();
    }
    for (int si = g.ntsn - 1; si >= 0; --si) {  // backward, reverse postorder
      const TopSN t = g.tsn[si];
      const int f = t.ns + t.nb;
      for (int r = wl; r < f; r += nw) {  // own y, or the ancestors' x
        const int pos = r < t.ns ? t.first + r : g.bpos[t.goff + r];
        reinterpret_cast<double2 *>(V + r * kVS)[lane] =
            reinterpret_cast<const double2 *>(Xw + (int64_t)g.tidx[pos] * CS)[lane];
      }
      __syncthreads();
      for (int k0 = wl * 8; k0 < t.ns; k0 += nw * 8) {
        double acc[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
        topk_mma_tile(F + t.fu_off, t.rb, t.bszb, k0, t.ns, f, V, lane, acc);
        const int r = k0 + crow;
        if (r < t.ns)
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) Xw[(int64_t)g.tidx[t.first + r] * CS + 8 * j + ccol + i] = acc[j][i];
      }
      __syncthreads();
    }
    for (int i = wl; i < g.nT; i += nw) {  // row groups of kr: [group][col][kr]
      const double2 v = reinterpret_cast<const double2 *>(Xw + (int64_t)i * CS)[lane];
      double *kb = g.K + (int64_t)b * g.kstride + (int64_t)(i - i % g.kr) * g.kpad + i % g.kr;
      const int c = col0 + 2 * lane;
      if (c < g.nT) kb[(int64_t)c * g.kr] = v.x;
      if (c + 1 < g.nT) kb[(int64_t)(c + 1) * g.kr] = v.y;
    }
    __syncthreads();
  }
}

static void build_dense_top(const NDFactor &fac, const NDSweepPlan &sp, cudaStream_t s) {
  const NDPlan &p = *fac.dev->plan;
  const int64_t kstride = sp.kstride();
  const size_t kbytes = (size_t)fac.nbatch * kstride * sizeof(double);
  if (fac.ktop.bytes != kbytes) fac.ktop.alloc_async(kbytes, s);
  STMHD_CUDA_CHECK(cudaMemsetAsync(fac.ktop.ptr, 0, kbytes, s));  // padded columns stay zero
  const int fmax = sp.kfmax;  // largest front of the K region (the only fronts staged here)
  TopKArgs g{};
  g.tsn = sp.tsn.as<TopSN>();
  g.tchild = sp.tchild.as<int4>();
  g.emap = fac.dev->emap.as<int>();
  g.tidx = sp.tidx.as<int>();
  g.bpos = sp.bpos.as<int>();
  g.factors = fac.factors.as<double>();
  g.fstride = fac.nbatch == 1 ? 0 : p.factor_size;
  g.ntsn = sp.ntsn;
  g.nT = sp.ntT;
  g.kpad = sp.kpad;
  g.kr = sp.kr;
  g.nbatch = fac.nbatch;
  // NC column halves per lane (STMHD_TOPK_NC, 1 or 2): each factor load feeds 32 NC
  // columns; NC = 2 runs 16 warps per CTA with the wider front block when it fits
  static const int nc_env = env_int2("STMHD_TOPK_NC", 2);
  // FP64 tensor-core construction (STMHD_TOPK_MMA, default on): 64 columns per item
  static const int mma_env = env_int2("STMHD_TOPK_MMA", 1);
  int nc = nc_env == 1 ? 1 : 2;
  if (mma_env) nc = 2;
  if ((size_t)fmax * 64 * sizeof(double) > 200 * 1024) nc = 1;
  const int cs = 32 * nc;
  g.ncb = (sp.ntT + cs - 1) / cs;
  const bool use_mma = mma_env && (size_t)fmax * kVS * sizeof(double) <= 226 * 1024;
  const size_t smem = (size_t)fmax * (use_mma ? kVS : cs) * sizeof(double);
  require(smem <= 226 * 1024, "dense top: front too large");
  // one 16-warp CTA per SM for NC = 2 (two 8-warp CTAs for NC = 1): the same warps per
  // SM and the same scratch footprint (a larger pooled scratch was measured to slow the
  // next factorisation's workspace allocations)
  const int per_sm = nc == 2 ? 1 : std::max(1, std::min(2, (int)((220 * 1024) / std::max<size_t>(smem, 1))));
  const int nitems = g.nbatch * g.ncb;
  const int grid = std::max(1, std::min(nitems, per_sm * num_sms()));
  g.scr_stride = (int64_t)(sp.ntT + sp.tcb_total) * cs;
  DevBuf scr;
  scr.alloc_async((size_t)grid * g.scr_stride * sizeof(double), s);
  g.scratch = scr.as<double>();
  g.K = fac.ktop.as<double>();
  g.kstride = kstride;
  static size_t attr[3] = {0, 0, 0};
  const int ai = use_mma ? 2 : nc - 1;
  const void *fn = use_mma ? (const void *)topk_mma_kernel
                           : (nc == 2 ? (const void *)topk_kernel<2> : (const void *)topk_kernel<1>);
  if (smem > attr[ai]) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[ai] = smem;
  }
  if (getenv("STMHD_SWEEP_PLAN_INFO"))
    fprintf(stderr, "[topk] n=%lld nT=%d nbatch=%d plan ncta=%d warps=%d gen=%llu items=%d grid=%d\n", (long long)p.n,
            sp.ntT, fac.nbatch, sp.ncta, sp.warps, (unsigned long long)fac.gen, nitems, grid);
  if (use_mma) topk_mma_kernel<<<grid, 512, smem, s>>>(g);
  else if (nc == 2) topk_kernel<2><<<grid, 512, smem, s>>>(g);
  else topk_kernel<1><<<grid, 256, smem, s>>>(g);
  STMHD_LAUNCH_CHECK();
  fac.ktop_plan = &sp;
  fac.ktop_gen = fac.gen;
}

// ---------------------------------------------------------------------------
// Stages

struct SweepStage {
  const NDFactor *fac = nullptr;
  const NDSweepPlan *sp = nullptr;
  SweepArgs a{};
  size_t smem = 0;
  double *x = nullptr;
  int64_t ld_x = 0;
  int nrhs = 0;
  DevBuf scratch, zero, pvals, flags, post_vals;
  int64_t flags_slabs = 0;
  // gathered coupling values are reused while (tag, program) are unchanged (tag 0:
  // always regather)
  int64_t vals_tag = 0, post_tag = 0;
  int warps = 0;  // warps per CTA (0: not chosen yet)
  int ncta = 0;   // CTAs of the sweep: kCluster (one cluster) or one per SM (grid mode)
  DevBuf gbar;    // grid-mode barrier word
  DevBuf progress;  // slab in progress (L2 prefetch cluster)
  const std::vector<int> *ext_pos[2] = {nullptr, nullptr};
  const CplProgram *vals_prog = nullptr, *post_prog = nullptr;
};

void SweepStageDeleter::operator()(SweepStage *p) const { delete p; }
int sweep_stage_warps(const SweepStage &st) { return st.warps; }
SweepStagePtr sweep_stage_new() { return SweepStagePtr(new SweepStage()); }

static constexpr int kCluster = 16, kWarps = 16;
static constexpr int kSmemMax = 227 * 1024 - 1536;  // opt-in maximum minus the kernel's static shared memory

// gathered values of a program: vals[b][id] (b = slab if any coupling is per-slab)
static int gather_values(const CplProgram &pg, const SweepCoupling *cpl, int ncpl, int nrhs, DevBuf &buf,
                         cudaStream_t s) {
  int per_slab = 0;
  CplVals cv{};
  for (int c = 0; c < ncpl; ++c) {
    per_slab |= cpl[c].val_stride != 0;
    cv.val[c] = cpl[c].val;
    cv.stride[c] = cpl[c].val_stride;
    cv.shift[c] = cpl[c].val_shift;
    cv.coef[c] = cpl[c].coef;
  }
  const int nblk = per_slab ? nrhs : 1;
  const size_t vneed = (size_t)nblk * pg.nent * sizeof(double);
  if (buf.bytes < vneed) buf.alloc_async(vneed, s);
  cpl_vals_kernel<<<dim3((unsigned)std::min<int64_t>(cdiv(pg.nent, 256), 1024), nblk), 256, 0, s>>>(
      pg.esrc.as<int2>(), pg.nent, cv, per_slab, buf.as<double>());
  STMHD_LAUNCH_CHECK();
  return per_slab;
}

void sweep_stage_prepare(SweepStage &st, const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x,
                         int64_t ld_x, int nrhs, const SweepCoupling *cpl, int ncpl, SweepStage *const *ext,
                         int next, cudaStream_t s, int64_t vals_tag, int ncta, bool grid, int warps_force) {
  const NDDevice &dev = *fac.dev;
  const NDPlan &p = *dev.plan;
  if (ncta <= 0) ncta = kCluster;
  grid = grid || ncta != kCluster;
  if (st.ncta != ncta) st.warps = 0;  // re-choose the warps for a new CTA count
  st.ncta = ncta;
  const int cluster = ncta;
  const int slot = sweep_slot(p);
  // warps per CTA: 16, halved while the plan's shared memory does not fit (large
  // slabs such as configuration 5); the choice sticks to the stage
  auto smem_of = [&](const NDSweepPlan &c, int w) {
    const size_t tstr = ((c.nl + 1 + 3) / 4) * 16 + (size_t)c.max_wtasks * sizeof(SweepTask);
    return ((size_t)w * c.vstride + 3 * c.sub_len + c.sub_cb + c.zlen() + 4) * sizeof(double) + (size_t)c.tab_ints * 4 +
           (size_t)w * tstr;
  };
  // prefer the most warps whose plan keeps the CTA-local subtree phase (fewer
  // cluster/grid barriers per slab), else the most warps whose flat plan fits
  static const int warps_env = env_int2("STMHD_SWEEP_WARPS", 0);  // experiments: warps per CTA
  if (warps_force <= 0 && warps_env > 0) warps_force = warps_env;
  if (warps_force > 0) st.warps = warps_force;
  int warps = st.warps;
  if (!warps) {
    int flat = 0;
    for (int w = kWarps; w >= 4 && !warps; w /= 2) {
      const NDSweepPlan &c = dev.get_sweep_plan(cluster, w, kSmemMax / 8, s);
      if (smem_of(c, w) > (size_t)kSmemMax) continue;
      if (c.nsub > 0 || ncta == kCluster) warps = w;  // cluster mode: first fit (stages of a
      else if (!flat) flat = w;                        // pipelined launch agree on 16)
    }
    if (!warps) warps = flat ? flat : 4;
  }
  st.warps = warps;
  const NDSweepPlan &sp = dev.get_sweep_plan(cluster, warps, kSmemMax / 8, s);
  const int vstride = sp.vstride;
  const int64_t n = p.n;
  st.fac = &fac;
  st.sp = &sp;
  st.x = x;
  st.ld_x = ld_x;
  st.nrhs = nrhs;
  // scratch: rhsp | xp | ybuf | cbv | tbuf; zero: n zeros, never written
  const size_t need = ((size_t)2 * nrhs * n + 2 * n + p.cbv_size + 16) * sizeof(double);
  // stage buffers come from the stream-ordered pool: growing or freeing them never
  // synchronises the device (a new preconditioner per Newton step reuses the blocks)
  if (st.scratch.bytes < need) st.scratch.alloc_async(need, s);
  if (st.zero.bytes < (size_t)n * sizeof(double)) {
    st.zero.alloc_async((size_t)n * sizeof(double), s);
    STMHD_CUDA_CHECK(cudaMemsetAsync(st.zero.ptr, 0, st.zero.bytes, s));
  }
  double *rhsp = st.scratch.as<double>();
  double *xp = rhsp + (int64_t)nrhs * n;
  double *zero = st.zero.as<double>();
  double *ybuf = xp + (int64_t)nrhs * n;
  double *cbv = ybuf + n;
  double *tbuf = cbv + p.cbv_size;
  permute_in_kernel<<<dim3(std::min<int64_t>(cdiv(n, 256), 256), nrhs), 256, 0, s>>>(rhs, ld_rhs, sp.pos.as<int>(), n,
                                                                                    nrhs, rhsp);
  STMHD_LAUNCH_CHECK();
  SweepArgs &a = st.a;
  a = SweepArgs{};
  a.wl_tasks = sp.wl_tasks.as<SweepTask>();
  a.wl_off = sp.wl_off.as<int>();
  a.wl_bnd = sp.wl_bnd.as<int>();
  a.nl = sp.nl;
  a.tstride = ((sp.nl + 1 + 3) / 4) * 16 + sp.max_wtasks * (int)sizeof(SweepTask);
  a.sub_info = sp.sub_info.as<int64_t>();
  a.ntop = sp.ntop;
  a.nsub = sp.nsub;
  a.warps = warps;
  a.sub_len = sp.sub_len;
  a.sub_cb = sp.sub_cb;
  a.g3p = sp.g3p.as<int4>();
  a.g4p = sp.g4p.as<int>();
  a.bpos = sp.bpos.as<int>();
  a.bpos4 = sp.bpos4.as<int>();
  if (sp.tab_ints) {
    a.tab = sp.tab.as<int>();
    a.tab_ptr = sp.tab_ptr.as<int>();
    a.tab_nf = sp.tab_nf.as<int>();
    a.tab_band = sp.tab_band.as<int>();
    a.tab_band_ptr = sp.tab_band_ptr.as<int>();
    a.tab_ints = sp.tab_ints;
  }
  a.nlevels = p.nlevels;
  a.nw = cluster * warps;
  a.n = n;
  a.factors = fac.factors.as<double>();
  a.fstride = fac.nbatch == 1 ? 0 : p.factor_size;
  a.rhsp = rhsp;
  a.xp = xp;
  a.zero = zero;
  a.ybuf = ybuf;
  a.cbv = cbv;
  a.nslab = nrhs;
  a.ncta = cluster;
  require(ncpl <= kMaxCpl && next <= 2, "sweep: at most four coupling terms and two external sources");
  for (int e = 0; e < next; ++e) {
    require(ext[e] && ext[e]->sp && ext[e]->nrhs == nrhs, "sweep: external stage not prepared for these slabs");
    st.ext_pos[e] = &ext[e]->sp->pos_h;
  }
  if (ncpl > 0) {
    const std::vector<int> *ext_pos[2] = {nullptr, nullptr};
    for (int e = 0; e < next; ++e) ext_pos[e] = st.ext_pos[e];
    for (int c = 0; c < ncpl; ++c) require(cpl[c].ext < next, "sweep: coupling refers to a missing external stage");
    const CplProgram &pg = get_program(sp, p, cpl, ncpl, ext_pos, s);
    int per_slab = 0;
    for (int c = 0; c < ncpl; ++c) per_slab |= cpl[c].val_stride != 0;
    if (!(vals_tag && st.vals_tag == vals_tag && st.vals_prog == &pg)) {
      per_slab = gather_values(pg, cpl, ncpl, nrhs, st.pvals, s);
      st.vals_tag = vals_tag;
      st.vals_prog = &pg;
    }
    a.prog_hdr = pg.hdr.as<int4>();
    a.prog_items = pg.items.as<int2>();
    a.prog_ecol = pg.ecol.as<int>();
    a.prog_vals = st.pvals.as<double>();
    a.prog_nent = pg.nent;
    a.prog_per_slab = per_slab;
    a.tbuf = tbuf;
  }
  a.dense = sp.dense;
  a.ntT = sp.ntT;
  a.kpad = sp.kpad;
  a.zlen = sp.zlen();
  a.dpieces = sp.dpieces;
  a.dgroups = sp.dgroups;
  a.kr = sp.kr;
  if (sp.dense) {
    if (fac.ktop_plan != &sp || fac.ktop_gen != fac.gen) build_dense_top(fac, sp, s);
    a.ztab = sp.ztab.as<int4>();
    a.ktop = fac.ktop.as<double>();
    a.kstride = fac.nbatch == 1 ? 0 : sp.kstride();
  }
  a.slot = slot;
  a.vstride = vstride;
  a.null_work = env_int2("STMHD_SWEEP_NULL", 0);
  a.ldgsts = env_int2("STMHD_SWEEP_LDGSTS", 0);
  a.cpl16 = env_int2("STMHD_SWEEP_CPL16", 1);
  a.kpref = env_int2("STMHD_SWEEP_KPREF", 0);  // measured: no gain (dense step not HBM-latency bound)
  a.post_hdr = nullptr;  // set by sweep_stage_set_post for this launch
  a.gbar = nullptr;
  {
    static const int early_env = env_int2("STMHD_SWEEP_EARLY_CPL", 1);
    int nroots = 0;
    for (int c = 0; c < ncta; ++c) nroots += sp.sub_info_h[4 * c + 1] > 0;
    a.nroots = nroots;
    a.early_cpl = early_env && grid && ncpl > 0 && sp.nsub > 0 && nroots > 0 && nroots < ncta;
  }
  if (grid) {  // grid-family launch: software barrier
    if (!st.gbar.ptr) {
      st.gbar.alloc(sizeof(unsigned));
      STMHD_CUDA_CHECK(cudaMemsetAsync(st.gbar.ptr, 0, sizeof(unsigned), s));
    }
    a.gbar = st.gbar.as<unsigned>();
  }
  st.smem = ((size_t)warps * a.vstride + 3 * a.sub_len + a.sub_cb + a.zlen + 4) * sizeof(double) +
            (size_t)a.tab_ints * 4 + (size_t)warps * a.tstride;
  require(st.smem <= (size_t)kSmemMax, "nd sweep: subtree vectors or fronts too large for shared memory");
  // consumers wait on their producers' flags (set at launch)
  a.nwait = next;
  for (int e = 0; e < next; ++e) {
    a.flag_in[e] = nullptr;
    a.ext_xp[e] = ext[e]->a.xp;
    a.ext_n[e] = ext[e]->a.n;
    a.ext_ncta[e] = ext[e]->ncta;
  }
  st.a.flag_out = nullptr;
}

// Post-slab program: rows of `target`'s (permuted) right-hand side, target_rhs[k] +=
// sum_c coef_c C_c src_c, with sources this stage's x_k (couplings with ext < 0) or the
// external stages of this stage at slab k.  Built once per coupling set.
static const CplProgram &get_post_program(const NDSweepPlan &sp, const NDSweepPlan &tp, int64_t n_t,
                                          const SweepCoupling *cpl, int ncpl,
                                          const std::vector<int> *const *ext_pos, cudaStream_t s) {
  std::vector<const void *> key{&tp, nullptr};  // (target plan, marker) distinguishes it from rhs programs
  for (int c = 0; c < ncpl; ++c) {
    key.push_back(cpl[c].rowptr);
    key.push_back(cpl[c].rowend);
    key.push_back(cpl[c].col);
    key.push_back(reinterpret_cast<const void *>((intptr_t)(cpl[c].col_off * 16 + cpl[c].ext + 1)));
  }
  auto it = sp.prog_cache.find(key);
  if (it != sp.prog_cache.end()) return *it->second;
  const int ncta = sp.ncta;
  std::vector<std::vector<int>> rb(ncpl), re(ncpl), cl(ncpl);
  for (int c = 0; c < ncpl; ++c) {
    rb[c].resize(n_t + 1);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(rb[c].data(), cpl[c].rowptr, (n_t + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
    re[c].resize(n_t);
    if (cpl[c].rowend)
      STMHD_CUDA_CHECK(cudaMemcpyAsync(re[c].data(), cpl[c].rowend, n_t * sizeof(int), cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    if (!cpl[c].rowend)
      for (int64_t i = 0; i < n_t; ++i) re[c][i] = rb[c][i + 1];
    int mx = 0;
    for (int64_t i = 0; i < n_t; ++i) mx = std::max(mx, re[c][i]);
    cl[c].resize(std::max(mx, 1));
    if (mx) STMHD_CUDA_CHECK(cudaMemcpy(cl[c].data(), cpl[c].col, mx * sizeof(int), cudaMemcpyDeviceToHost));
  }
  // contiguous blocks of target rows per CTA
  std::vector<int4> hdr(ncta);
  std::vector<int2> it2;
  std::vector<int> ecol;
  std::vector<int2> esrc;
  for (int c = 0; c < ncta; ++c) {
    const int64_t q0 = n_t * c / ncta, q1 = n_t * (c + 1) / ncta;
    std::vector<std::vector<int2>> ents(q1 - q0);  // {enc, cid}, e in a parallel list
    std::vector<std::vector<int>> eids(q1 - q0);
    int width = 0;
    for (int64_t q = q0; q < q1; ++q) {
      const int io = tp.iperm_h[q];
      for (int cc = 0; cc < ncpl; ++cc)
        for (int e = rb[cc][io]; e < re[cc][io]; ++e) {
          const int jr = cl[cc][e] - cpl[cc].col_off;
          int enc;
          if (cpl[cc].ext >= 0) {
            const std::vector<int> &ep = *ext_pos[cpl[cc].ext];
            require(jr >= 0 && jr < (int)ep.size(), "sweep post program: external column out of range");
            enc = ((3 + cpl[cc].ext) << 28) | ep[jr];
          } else {
            require(jr >= 0 && jr < (int)sp.pos_h.size(), "sweep post program: column out of range");
            enc = (5 << 28) | sp.pos_h[jr];
          }
          ents[q - q0].push_back(make_int2(enc, cc));
          eids[q - q0].push_back(e);
        }
      width = std::max(width, (int)ents[q - q0].size());
    }
    const int ni = (int)(q1 - q0);
    hdr[c] = make_int4((int)it2.size(), ni, (int)ecol.size(), width);
    for (int64_t q = q0; q < q1; ++q) it2.push_back(make_int2((int)q, -1));
    const size_t base = ecol.size();
    ecol.resize(base + (size_t)width * ni, 0);
    esrc.resize(base + (size_t)width * ni, make_int2(-1, 0));
    for (int i = 0; i < ni; ++i)
      for (int sl = 0; sl < (int)ents[i].size(); ++sl) {
        ecol[base + (size_t)sl * ni + i] = ents[i][sl].x;
        esrc[base + (size_t)sl * ni + i] = make_int2(ents[i][sl].y, eids[i][sl]);
      }
  }
  if (ecol.empty()) {
    ecol.push_back(0);
    esrc.push_back(make_int2(-1, 0));
  }
  if (it2.empty()) it2.push_back(make_int2(0, -1));
  auto pg = std::make_unique<CplProgram>();
  pg->nent = (int64_t)ecol.size();
  pg->hdr = upload_vec(hdr, s);
  pg->items = upload_vec(it2, s);
  pg->ecol = upload_vec(ecol, s);
  pg->esrc = upload_vec(esrc, s);
  pg->ok = true;
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  const CplProgram &ref = *pg;
  sp.prog_cache[key] = std::move(pg);
  return ref;
}

void sweep_stage_set_post(SweepStage &st, SweepStage &target, const SweepCoupling *cpl, int ncpl, cudaStream_t s,
                          int64_t vals_tag) {
  require(st.sp && target.sp && st.nrhs == target.nrhs, "sweep post program: stages not prepared");
  require(ncpl <= kMaxCpl, "sweep post program: at most four terms");
  const std::vector<int> *ext_pos[2] = {nullptr, nullptr};
  // external sources of the post program are this stage's external stages
  for (int c = 0; c < ncpl; ++c) require(cpl[c].ext < st.a.nwait, "sweep post program: missing external stage");
  for (int e = 0; e < st.a.nwait; ++e) ext_pos[e] = st.ext_pos[e];
  const CplProgram &pg = get_post_program(*st.sp, *target.sp, target.a.n, cpl, ncpl, ext_pos, s);
  int per_slab = 0;
  for (int c = 0; c < ncpl; ++c) per_slab |= cpl[c].val_stride != 0;
  if (!(vals_tag && st.post_tag == vals_tag && st.post_prog == &pg)) {
    per_slab = gather_values(pg, cpl, ncpl, st.nrhs, st.post_vals, s);
    st.post_tag = vals_tag;
    st.post_prog = &pg;
  }
  SweepArgs &a = st.a;
  a.post_hdr = pg.hdr.as<int4>();
  a.post_items = pg.items.as<int2>();
  a.post_ecol = pg.ecol.as<int>();
  a.post_vals = st.post_vals.as<double>();
  a.post_nent = pg.nent;
  a.post_per_slab = per_slab;
  a.post_out = const_cast<double *>(target.a.rhsp);  // target rhsp is its scratch (written here, read after the flag)
  a.post_n = target.a.n;
}

// Fault words of the pipelined launch: a device word the consumers poll (cheap) and a
// host-mapped copy the host reads at the next launch / sweep_check_fault().
static int *g_fault_dev = nullptr;
static volatile int *g_fault_host = nullptr;
static int *g_fault_host_dev = nullptr;

static void fault_words_init() {
  if (g_fault_dev) return;
  STMHD_CUDA_CHECK(cudaMalloc(&g_fault_dev, sizeof(int)));
  STMHD_CUDA_CHECK(cudaMemset(g_fault_dev, 0, sizeof(int)));
  int *h = nullptr;
  STMHD_CUDA_CHECK(cudaHostAlloc(&h, sizeof(int), cudaHostAllocMapped));
  *h = 0;
  STMHD_CUDA_CHECK(cudaHostGetDevicePointer(&g_fault_host_dev, h, 0));
  g_fault_host = h;
}

// Raise (once) if a previous pipelined launch recorded a producer timeout.  Only
// launches that completed are visible, so a caller that needs certainty synchronises
// first (stmhd_device_fault does).
void sweep_check_fault(cudaStream_t s) {
  if (!g_fault_host || !*g_fault_host) return;
  *g_fault_host = 0;
  STMHD_CUDA_CHECK(cudaMemsetAsync(g_fault_dev, 0, sizeof(int), s));
  throw Error(STMHD_CUDA, "pipelined sweep: a consumer stage timed out waiting for its producer "
                          "(stages not co-resident); results of that launch are invalid");
}

void sweep_stages_launch(SweepStage *const *stg, int nst, cudaStream_t s) {
  require(nst >= 1 && nst <= 3, "sweep: 1 to 3 stages per launch");
  fault_words_init();
  sweep_check_fault(s);
  static int epoch = 0;
  ++epoch;
  SweepMulti m{};
  size_t smem = 0;
  for (int i = 0; i < nst; ++i) {
    SweepStage &st = *stg[i];
    st.a.epoch = epoch;
    if (nst > 1 || (st.a.early_cpl && !st.a.post_hdr)) {  // per-slab flags (consumers / early coupling)
      const int64_t need = (int64_t)st.nrhs * st.ncta;
      if (st.flags_slabs < need) {
        st.flags.alloc_async(need * sizeof(int), s);
        STMHD_CUDA_CHECK(cudaMemsetAsync(st.flags.ptr, 0, need * sizeof(int), s));
        st.flags_slabs = need;
      }
      st.a.flag_out = st.flags.as<int>();
    } else {
      st.a.flag_out = nullptr;
    }
    if (!st.progress.ptr) {
      st.progress.alloc_async(sizeof(unsigned long long), s);
      STMHD_CUDA_CHECK(cudaMemsetAsync(st.progress.ptr, 0, sizeof(unsigned long long), s));
    }
    st.a.progress = st.progress.as<unsigned long long>();
    st.a.fault = g_fault_dev;
    st.a.fault_host = g_fault_host_dev;
    smem = std::max(smem, st.smem);
    require(st.warps == stg[0]->warps, "sweep: stages of one launch need the same warps per CTA");
  }
  const int warps = stg[0]->warps;
  const bool grid = stg[0]->a.gbar != nullptr;
  int first[4] = {0, 0, 0, 0};
  for (int i = 0; i < nst; ++i) {
    require((stg[i]->a.gbar != nullptr) == grid, "sweep: all stages of a launch in grid or cluster mode");
    require(grid || stg[i]->ncta == kCluster, "sweep: cluster launches take 16-CTA stages");
    first[i + 1] = first[i] + stg[i]->ncta;
  }
  for (int i = 0; i < nst; ++i) {
    SweepStage &st = *stg[i];
    for (int e = 0; e < st.a.nwait; ++e) {
      int prod = -1;
      for (int j = 0; j < i; ++j)
        if (stg[j]->a.xp == st.a.ext_xp[e]) prod = j;
      require(prod >= 0, "sweep: an external source must be an earlier stage of the same launch");
      st.a.flag_in[e] = stg[prod]->a.flag_out;
    }
    m.st[i] = st.a;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncAttributes fa{};
    for (const void *fn : {(const void *)nd_sweep_kernel<false>, (const void *)nd_sweep_kernel<true>}) {
      STMHD_CUDA_CHECK(cudaFuncGetAttributes(&fa, fn));
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      STMHD_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(227 * 1024 - fa.sharedSizeBytes)));
    }
    attr = true;
  }
  static const int trace_stage = env_int2("STMHD_SWEEP_TRACE_STAGE", 0);
  const int ts = std::min(std::max(trace_stage, 0), nst - 1);
  SweepStage &s0 = *stg[ts];
  const int64_t n0 = s0.a.n;
  const int nrhs0 = s0.nrhs;
  static const int trace_on = env_int2("STMHD_SWEEP_TRACE", 0);
  DevBuf tr;
  int nsteps = 0;
  if (trace_on) {  // stage 0 only
    nsteps = 4 + nrhs0 * (2 * s0.fac->dev->plan->nlevels + 4);
    tr.alloc(nsteps * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(tr.ptr, 0, tr.bytes, s));
    m.st[ts].trace = tr.as<unsigned long long>();
  }
  static const int prof_on = env_int2("STMHD_SWEEP_PROF", 0);
  DevBuf pr;
  DevBuf tlb, pcb;
  if (prof_on) {
    pr.alloc((size_t)stg[ts]->ncta * warps * 10 * sizeof(unsigned long long));
    m.st[ts].prof = pr.as<unsigned long long>();
    tlb.alloc((size_t)warps * 128 * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(tlb.ptr, 0, tlb.bytes, s));
    m.st[ts].tline = tlb.as<unsigned long long>();
    pcb.alloc((size_t)2 * stg[ts]->ncta * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaMemsetAsync(pcb.ptr, 0, pcb.bytes, s));
    m.st[ts].pcta = pcb.as<unsigned long long>();
  }
  // L2 prefetch cluster (cluster mode): one extra 16-CTA cluster when the device
  // can hold it next to the stages (STMHD_SWEEP_L2PF = prefetch distance in slabs, 0 off)
  static const int pf_env = env_int2("STMHD_SWEEP_L2PF", 0);  // off: ~1 % on the wave sweep only, +40 % DRAM reads
  int pf = 0;
  if (!grid && pf_env > 0) {
    static int max_clusters = -1;
    if (max_clusters < 0) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(kCluster * 4);
      q.blockDim = dim3(warps * 32);
      q.dynamicSmemBytes = smem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = kCluster;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int mc = 0;
      if (cudaOccupancyMaxActiveClusters(&mc, (const void *)nd_sweep_kernel<false>, &q) != cudaSuccess) {
        cudaGetLastError();
        mc = 0;
      }
      max_clusters = mc;
      if (env_int2("STMHD_SWEEP_L2PF_DEBUG", 0)) fprintf(stderr, "[sweep] max active 16-CTA clusters %d\n", mc);
    }
    pf = max_clusters >= nst + 1 ? 1 : 0;
  }
  m.nst = nst;
  m.pf_dist = pf_env;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid ? first[nst] : kCluster * (nst + pf));
  for (int i = 0; i < 4; ++i) m.first[i] = i <= nst ? first[i] : first[nst];
  cfg.blockDim = dim3(warps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  int nat = 1;
  if (grid) {  // no cluster; all CTAs co-resident (cooperative) for the grid barrier
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  }
  // the stages wait on each other: all clusters must be co-resident.  When the
  // occupancy query says the device holds at least nst such clusters at once they are
  // (the launch is the only work on the device for its duration), and the launch goes
  // without the cooperative attribute so profilers can replay it; otherwise it is a
  // cooperative launch.  STMHD_PIPE_COOP=1 forces the attribute, 0 never sets it.  A
  // consumer that still waits more than 4 s records a fault (sweep_check_fault).
  static const int coop_env = env_int2("STMHD_PIPE_COOP", -1);
  if (nst > 1 && !grid && coop_env != 0) {
    static int max_cl = -1;
    if (max_cl < 0) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(kCluster * nst);
      q.blockDim = dim3(warps * 32);
      q.dynamicSmemBytes = smem;
      q.attrs = at;
      q.numAttrs = 1;
      int mc = 0;
      if (cudaOccupancyMaxActiveClusters(&mc, (const void *)nd_sweep_kernel<false>, &q) != cudaSuccess) {
        cudaGetLastError();
        mc = 0;
      }
      max_cl = mc;
    }
    if (coop_env == 1 || max_cl < nst) {
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      nat = 2;
    }
  }
  cfg.attrs = at;
  cfg.numAttrs = nat;
  void *args[] = {&m};
  STMHD_CUDA_CHECK(cudaLaunchKernelExC(
      &cfg, prof_on ? (const void *)nd_sweep_kernel<true> : (const void *)nd_sweep_kernel<false>, args));
  count_launch();
  for (int i = 0; i < nst; ++i) {
    SweepStage &st = *stg[i];
    const int64_t n = st.a.n;
    permute_out_kernel<<<dim3(std::min<int64_t>(cdiv(n, 256), 256), st.nrhs), 256, 0, s>>>(
        st.a.xp, st.sp->pos.as<int>(), n, st.nrhs, st.x, st.ld_x);
    STMHD_LAUNCH_CHECK();
  }
  if (trace_on) {
    const SweepArgs &a = s0.a;
    const NDPlan &p = *s0.fac->dev->plan;
    std::vector<unsigned long long> h(nsteps);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(h.data(), tr.ptr, nsteps * 8, cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    const bool fz = a.prog_hdr != nullptr;
    auto entries = [&](int k) {
      return (int)fz + ((a.nsub || fz) ? 1 : 0) + (a.dense ? 2 : 0) + 2 * a.ntop + (a.nsub && k + 1 < a.nslab);
    };
    const int per = entries(1), base = 1 + entries(0);
    fprintf(stderr, "[sweep] n=%lld levels=%d top=%d sub=%d fused=%d stages=%d total=%.1f us | slab1 (us):",
            (long long)n0, p.nlevels, a.ntop, a.nsub, (int)fz, nst,
            (*std::max_element(h.begin(), h.end()) - h[0]) / 1e3);
    for (int i = 0; i < per && base + i < nsteps; ++i) fprintf(stderr, " %.2f", (h[base + i] - h[base + i - 1]) / 1e3);
    fprintf(stderr, "\n[sweep] factor/slab %.2f MB nslab %d (batch %d) smem %zu B vstride %d slot %d sub_len %lld sub_cb %lld\n",
            p.factor_size * 8e-6, nrhs0, s0.fac->nbatch, smem, a.vstride, a.slot, (long long)a.sub_len,
            (long long)a.sub_cb);
  }
  if (prof_on) {
    const int nwp = stg[ts]->ncta * warps;
    std::vector<unsigned long long> h((size_t)nwp * 10);
    STMHD_CUDA_CHECK(cudaMemcpyAsync(h.data(), pr.ptr, h.size() * 8, cudaMemcpyDeviceToHost, s));
    STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
    double mean[10] = {0}, mx[10] = {0};
    for (int w = 0; w < nwp; ++w)
      for (int i = 0; i < 10; ++i) {
        mean[i] += (double)h[w * 10 + i] / nwp;
        mx[i] = std::max(mx[i], (double)h[w * 10 + i]);
      }
    const double us = 1.0 / 1963.0 / nrhs0;  // cycles -> us per slab at the loaded SM clock
    fprintf(stderr,
            "[sweep-prof] per slab per warp (us) mean/max: gather %.2f/%.2f wait %.2f/%.2f gemv %.2f/%.2f "
            "barrier %.2f/%.2f | tasks %.1f/%.0f chunks %.1f/%.0f | gemv-only fwd %.2f bwd %.2f | issue %.2f | coupling %.2f/%.2f\n",
            mean[0] * us, mx[0] * us, mean[1] * us, mx[1] * us, mean[2] * us, mx[2] * us, mean[3] * us, mx[3] * us,
            mean[4] / nrhs0, mx[4] / nrhs0, mean[5] / nrhs0, mx[5] / nrhs0, mean[6] * us, mean[7] * us, mean[8] * us,
            mean[9] * us, mx[9] * us);
    // timeline of slab 1, CTA 0: per warp, events (1 level start fwd, 2 gathered, 3 chunk, 4 level done fwd,
    // 5 level start bwd, 6 level done bwd) in us from the first event
    std::vector<unsigned long long> tv((size_t)warps * 128);
    STMHD_CUDA_CHECK(cudaMemcpy(tv.data(), tlb.ptr, tv.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (auto v : tv)
      if (v) t0 = std::min(t0, v & ((1ull << 56) - 1));
    {
      std::vector<unsigned long long> pc((size_t)2 * stg[ts]->ncta);
      STMHD_CUDA_CHECK(cudaMemcpy(pc.data(), pcb.ptr, pc.size() * 8, cudaMemcpyDeviceToHost));
      fprintf(stderr, "[pcta] slab 1 subtree fwd/bwd (us) per CTA:");
      for (int c = 0; c < stg[ts]->ncta; ++c) fprintf(stderr, " %d:%.1f/%.1f", c, pc[2 * c] / 1e3, pc[2 * c + 1] / 1e3);
      fprintf(stderr, "\n");
    }
    for (int wv = 0; wv < warps; ++wv) {
      fprintf(stderr, "[tl] w%02d:", wv);
      for (int i = 0; i < 128; ++i) {
        const unsigned long long v = tv[(size_t)wv * 128 + i];
        if (!v) break;
        const char *c = "?SGCEsE";
        fprintf(stderr, " %c%.2f", c[(v >> 56) & 7], ((v & ((1ull << 56) - 1)) - t0) / 1e3);
      }
      fprintf(stderr, "\n");
    }
  }
}

void nd_sweep(const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
              const SweepCoupling *cpl, int ncpl, cudaStream_t s) {
  // one stage per factor structure, owned by it (reused across calls and
  // factorisations; launches are stream ordered)
  SweepStagePtr &sp = fac.dev->single_stage;
  if (!sp) sp = sweep_stage_new();
  // grid mode (one CTA per SM, software grid barrier) when a slab's factor is large
  // enough that 16 SMs cannot stream it (configuration 5: 75 MB per slab); the
  // cluster mode keeps the cheaper hardware barrier for the MHD blocks
  static const int grid_env = env_int2("STMHD_SWEEP_GRID", -1);
  const double fbytes = 8.0 * (double)fac.dev->plan->factor_size;
  // (amalgamated plans need more subtrees than a 16-CTA cluster has CTAs)
  const bool grid = grid_env == 1 || (grid_env < 0 && (fbytes > 32e6 || fac.dev->plan->nwide > 0));
  sweep_stage_prepare(*sp, fac, rhs, ld_rhs, x, ld_x, nrhs, cpl, ncpl, nullptr, 0, s, 0,
                      grid ? num_sms() : kCluster, grid);
  SweepStage *one = sp.get();
  sweep_stages_launch(&one, 1, s);
}

}  // namespace stmhd
