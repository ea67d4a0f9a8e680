// Nested-dissection supernodal LU: host symbolic plan + device numeric/solve.
//
// Replaces the per-slab SuperLU factorisations and solves of the reference
// (LUFactor, pkg/src/stmhd/linalg.py:71-96; used by precond.py:75,85,96 and
// problems.py:225-228).  One symbolic structure is shared by a batch of
// matrices with the same pattern (all time slabs), so the numeric work is a
// batch of dense front operations.  Each supernode s eliminates its columns
// `cols` (a separator or a leaf region) and owns a dense front over
// cols ++ bnd, where bnd are the ancestor unknowns coupled to its subtree.
//
// Stored per supernode and matrix (inverse-based, so every solve step is a
// dense GEMV with no sequential dependency inside the block):
//   FL = [ L11^{-1} P ; L21 L11^{-1} P ]      (f x ns)   forward step
//   FU = [ U11^{-1} | -U11^{-1} U12 ]         (ns x f)   backward step
// with P the partial-pivoting row permutation inside the diagonal block.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <vector>

#include "common.cuh"

namespace stmhd {

struct NDPlan {
  int64_t n = 0;
  int nsn = 0;      // supernodes (postorder: children before parents)
  int nlevels = 0;  // height+1; level 0 = leaves
  std::vector<int> level, ns, nb, parent;
  std::vector<int64_t> first;    // elimination position of the first column of s
  std::vector<int64_t> idx_off;  // offset of the front index list (f entries) in idx
  std::vector<int> idx;          // cols ++ bnd, original unknown ids
  std::vector<int> child_ptr, child_list;
  std::vector<int64_t> emap_off;  // nb entries per s: position of bnd[a] in parent's front
  std::vector<int> emap;
  std::vector<int64_t> scat_ptr;  // per supernode range in scat_src/scat_dst
  std::vector<int64_t> scat_src;  // index into the caller's value array
  std::vector<int64_t> scat_dst;  // position fi*f+fj inside the front
  // Factor storage (per matrix): for each supernode the forward operator
  // FL (f x ns) and the backward operator FU (ns x f) are cut into row chunks
  // of R rows; chunk c is one contiguous block [K][R] (K = ns for FL, f for FU,
  // rows past the end zero padded, block padded to an even number of doubles),
  // so a chunk is a single 1D bulk copy.  chunk_f/chunk_b = R per direction.
  std::vector<int> rf, rb;             // rows per chunk (forward / backward)
  std::vector<int64_t> bsz_f, bsz_b;   // doubles per chunk block
  std::vector<int64_t> fl_off, fu_off, front_off, cbv_off;
  int64_t factor_size = 0, front_size = 0, cbv_size = 0;
  // column-major staging layout written by the factorisation kernel
  std::vector<int64_t> sfl_off, sfu_off;
  int64_t stage_size = 0;
  int64_t sym_nnz = 0;  // nnz of L+U implied by the supernodal structure
  int max_front = 0;
  std::vector<std::vector<int>> level_sn;
  // amalgamated supernodes (nd_analyze merge_depth) have up to four children; a front row
  // then takes up to four child updates (the gather tables carry two more slots)
  int nwide = 0;
  bool wide(int s) const { return child_ptr[s + 1] - child_ptr[s] > 2; }
};

// Build the plan.  gx/gy may be null (graph bisection).  value_map (may be null)
// maps pattern entries to caller value indices.
NDPlan nd_analyze(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *gx,
                  const int32_t *gy, int leaf_max, const int32_t *value_map, unsigned merge_mask = 0);

// Work item of the cluster-resident time sweep (nd_sweep.cu), built lazily for a
// launch shape: a contiguous chunk range of one supernode.  32 bytes, so a warp's
// whole task list sits in shared memory.
struct alignas(16) SweepTask {
  int foff;             // offset of chunk 0 in a slab's factors (forward FL or backward FU blocks)
  int goff;             // offset of the supernode's front tables
  int first;            // elimination position of the first column
  int cboff;            // update-vector offset
  short c0, c1;         // chunk range
  short ns, f, rows;    // columns, front size, rows of the step (f forward, ns backward)
  unsigned char R;      // rows per chunk (power of two <= 32)
  unsigned char flags;  // 1: update vector to global memory; 4: front table rides in the ring first
                        // (8: backward table = aligned bpos at cboff, else forward g3 at goff); 2: dense top row
  int bsz;              // doubles per chunk block
};
static_assert(sizeof(SweepTask) == 32, "SweepTask must stay 32 bytes");

// Slab-coupling "program" of a sweep with subtrees: per CTA, the output items it
// computes at the start of every slab (its subtree rows into shared memory and a
// share of the top rows into global memory).
struct CplProgram {
  bool ok = false;
  int64_t nent = 0;      // entries (all CTAs)
  DevBuf hdr;            // int4 per CTA {item_off, nitems, ent_off, width}
  DevBuf items;          // int2 per item {dst (kind << 29 | index), rhs row or -1}
  DevBuf ecol;           // int per entry, [slot][item] per CTA: source id << 28 | index (pad: 0 with value 0)
  DevBuf esrc;           // int2 per entry {coupling, value index} ({-1, 0} pad)
};

struct NDSweepPlan {
  int ncta = 0, warps = 0;
  // top of the tree: cluster-wide level steps (ntop); bottom: one subtree per CTA,
  // CTA-local level steps (nsub, 0 = none) with its vectors in shared memory
  int ntop = 0, nsub = 0;
  int64_t sub_len = 0, sub_cb = 0;  // max subtree columns / internal update-vector doubles per CTA
  DevBuf sub_info;                  // per CTA int64 {first col, ncols, first cb, ncb}
  // per physical warp (cta * warps + w): its task list for one slab in kernel order
  // (subtree forward levels, top forward, top backward, subtree backward) and the
  // start of every phase level in it (nl = 2 nsub + 2 ntop levels, nl + 1 bounds)
  int nl = 0, max_wtasks = 0;
  int vstride = 0;          // doubles of shared memory per warp (gather buffer + two TMA slots)
  DevBuf wl_tasks, wl_off, wl_bnd;
  // dense top (dense = 1): after the subtree forward phase the top unknowns are
  //   x_T = K z_T,  z_T = top rows of the coupled rhs + the subtree roots' updates,
  // K = (A^{-1})_TT (inverse of the top Schur complement, NDFactor::ktop) -- one GEMV
  // step instead of 2 * ntop tree levels.  Top unknowns in elimination order.
  // K is stored in row groups of kr rows: block (group g, column chunk c) holds kr x kc
  // entries column-major ([kc][kr]), so one ring item feeds kr rows (kr = 1: plain rows).
  int dense = 0, ntT = 0, kc = 0, nch = 0, kpad = 0, kr = 1;
  // the row groups of K are spread over the CTAs (group g on CTA g % ncta, local index
  // g / ncta) and each group's nch column chunks over that CTA's warps in dpieces
  // pieces; the partial dot products meet in shared memory (dred, dgroups x dpieces x kr
  // doubles per CTA) and are summed in a fixed order, so the result is deterministic
  int dpieces = 1, dgroups = 0;
  int zlen() const { return kpad + dgroups * dpieces * kr; }  // shared doubles: z_T + partials
  int64_t kstride() const { return (int64_t)((ntT + kr - 1) / kr * kr) * kpad; }
  DevBuf ztab;              // int4 x 2 per top unknown {pos, cb0, cb1, cb2}, {cb3, -1, -1, -1}
  DevBuf tidx;              // n: top index of a permuted position, or -1
  DevBuf tsn, tchild;       // top supernodes (postorder) and their top children (K construction)
  int ntsn = 0;
  int kfmax = 1;            // largest front among the top (K region) supernodes
  int64_t tcb_total = 0;    // sum of nb over top supernodes
  // per-CTA subtree front tables kept in shared memory (dense mode): ints per CTA
  // block [tab_ptr[c], tab_ptr[c+1]): forward int32 entries, then backward uint16 pairs
  int tab_ints = 0;
  DevBuf tab, tab_ptr, tab_nf;
  DevBuf tab_band, tab_band_ptr;  // per-CTA band positions referenced by the backward tables
  DevBuf g3p;   // int4 per front position: {permuted rhs index or -1, cb1, cb2, cb3} (cb3: wide supernodes)
  DevBuf g4p;   // int per front position: cb4 of wide supernodes (else -1)
  DevBuf bpos;  // int per front position: permuted position of the front entry
  DevBuf bpos4; // bpos per supernode, each block 16-byte aligned (TMA ring table items)
  DevBuf pos;   // n: elimination position of each original index
  DevBuf iperm; // n: original index at each elimination position
    std::vector<int64_t> sub_info_h;  // host copy of sub_info
  std::vector<int> pos_h, iperm_h;  // host copies of pos / iperm
  // fused slab-coupling programs (nd_sweep.cu), keyed by the coupling index arrays
  mutable std::map<std::vector<const void *>, std::unique_ptr<struct CplProgram>> prog_cache;
};

// Device-resident copy of a plan plus the solve schedules.
struct SweepStage;
struct SweepStageDeleter {
  void operator()(SweepStage *p) const;
};

struct NDDevice {
  const NDPlan *plan = nullptr;
  DevBuf ns, nb, first, idx_off, idx, child_ptr, child_list, emap_off, emap, scat_ptr,
      scat_src, scat_dst, fl_off, fu_off, sfl_off, sfu_off, rf, rb, bsz_f, bsz_b, front_off, cbv_off, lvl_sn,
      lvl_ptr;
  // solve work items: int4 {sn, row_begin, row_end, 0} (32-row chunks); per level ranges
  DevBuf gather4;  // int per front position: fourth child update of wide supernodes
  DevBuf fwd_items, bwd_items, gather3;  // SolveItem lists + flat forward gather table (int4 per front position)
  std::vector<int> fwd_ptr, bwd_ptr;  // host copies of level ranges (nlevels+1)
  DevBuf fwd_ptr_d, bwd_ptr_d;
  int max_front = 0;
  void build(const NDPlan &p, cudaStream_t s);
  // sweep plans by (CTAs, warps per CTA): a stage's launch shape (the pipelined
  // grid-family launch, a single-stage sweep, the warp-count trials) each keep their
  // own plan; never evicted, so a plan's address identifies it for the device's
  // lifetime (NDFactor::ktop_plan compares addresses)
  mutable std::vector<std::unique_ptr<NDSweepPlan>> sweep_plans;
  const NDSweepPlan &get_sweep_plan(int ncta, int warps, int64_t smem_budget, cudaStream_t s, int mode = 0) const;
  // the single-stage sweep of nd_sweep() for this structure (handle-owned: lives and
  // dies with the device structure, reused across calls and factorisations)
  mutable std::unique_ptr<SweepStage, SweepStageDeleter> single_stage;
};

// A coupling term of a sequential block sweep:
//   rhs_k += coef * C_(k) x_(k-lag)          (lag 1 or 2: the sweep's own output)
//   rhs_k += coef * C_(k) e_(k)              (ext >= 0: another stage's output)
// C is CSR-like: row i holds entries [rowptr[i], rowend ? rowend[i] : rowptr[i+1])
// with columns col[e] - col_off and values val[(k - val_shift) * val_stride + e].
struct SweepCoupling {
  const int32_t *rowptr = nullptr;
  const int32_t *rowend = nullptr;
  const int32_t *col = nullptr;
  int col_off = 0;
  const double *val = nullptr;
  int64_t val_stride = 0;  // 0: shared matrix
  int64_t val_shift = 0;   // value block used for slab k is (k - val_shift)
  int lag = 0;             // 1 or 2 (own output); 0 with ext >= 0
  int ext = -1;            // external source stage (sweep_stages_launch), lag 0
  double coef = 0.0;
};

// Flat descriptor of one solve work item: everything a warp needs in one load.
struct alignas(16) SolveItem {
  int s, r0, r1, kl;  // supernode, row range, lanes per row
  int ns, f, wide, pad1;  // wide: the supernode has more than two children (gather3.w / gather4 in use)
  int64_t foff;   // factor offset (FL^T forward, FU^T backward)
  int64_t goff;   // offset of the supernode's front lists (idx / gather3)
  int64_t first;  // elimination position of the first column
  int64_t cboff;  // update-vector offset
};

struct NDFactor {
  const NDDevice *dev = nullptr;
  int nbatch = 0;
  DevBuf factors;  // nbatch * factor_size doubles
  DevBuf status;   // int[2]: 0 ok / 1+ singular (first failing supernode+1); smallest pivot ratio (float bits)
  mutable float min_pivot_ratio = 1.0f;  // of the last factorisation (check_status)
  uint64_t gen = 0;  // bumped by every factorisation
  // dense inverse of the top Schur complement per batch entry (nd_sweep.cu), built
  // lazily for the sweep plan that uses it: [nbatch][kstride()] doubles (row groups of kr)
  mutable DevBuf ktop;
  mutable DevBuf scratch, bar;  // batched-solve scratch and grid-barrier words (per factor)
  // small shared factors (nbatch == 1, n <= 2048): dense A^{-1} (column-major), built
  // once per factorisation by solving A X = I; batched solves are then one FP64
  // tensor-core GEMM (dense_solve_gemm, nd_numeric.cu)
  mutable DevBuf dinv, gemm_ws;
  mutable uint64_t dinv_gen = ~0ull;
  bool dense_ok = false;  // set for the discretisation's constant factors only
  mutable const void *ktop_plan = nullptr;
  mutable uint64_t ktop_gen = ~0ull;
  void factor(const double *values, int64_t value_stride, cudaStream_t s);
  // x_b = A_b^{-1} rhs_b (b < nrhs; factor b, or 0 if nbatch == 1).
  void solve(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
             cudaStream_t s) const;
  void solve_nd(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
                cudaStream_t s) const;  // the supernodal substitution path
  // Sequential sweep over slabs k = 0..nrhs-1:
  //   x_k = A_k^{-1}( rhs_k + sum_t coef_t C_t x_(k-lag_t) )
  void sweep(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
             const SweepCoupling *cpl, int ncpl, cudaStream_t s) const;
  int check_status(cudaStream_t s) const;  // synchronises
};

#if defined(__CUDACC__)
// One warp computes the R rows of a chunk block [K][R] against v[0..K):
// lane = (kq, rl) with rl = lane % R, kq = lane / R; a warp load touches 32
// consecutive doubles.  16 loads per lane are issued before the FMAs.  The
// result is valid in every lane for row rl.
template <bool GLOBAL>
__device__ __forceinline__ double chunk_gemv(const double *__restrict__ blk, int R, int K, const double *v, int lane) {
  const int kl = 32 / R, rl = lane & (R - 1), kq = lane / R;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (K > 0) {
    for (int t = kq; t < K; t += 16 * kl) {
      double m[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const double *ptr = blk + (int64_t)min(t + q * kl, K - 1) * R + rl;
        m[q] = GLOBAL ? __ldg(ptr) : *ptr;
      }
      asm volatile("" ::: "memory");
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int tq = t + q * kl;
        acc[q & 3] = fma(m[q], tq < K ? v[tq] : 0.0, acc[q & 3]);
      }
    }
  }
  double out = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  for (int o = R; o < 32; o <<= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
  return out;
}
#endif

// A prepared sweep (one cluster of a pipelined launch), nd_sweep.cu (declared above).
using SweepStagePtr = std::unique_ptr<SweepStage, SweepStageDeleter>;
SweepStagePtr sweep_stage_new();
// Permute the stage's right-hand sides in and bind its couplings; ext[e] are stages
// prepared before whose (permuted) output feeds the couplings with ext = e.
// vals_tag != 0: the coupling values are unchanged since the last prepare with the
// same tag (a preconditioner's lifetime), so their gathered copy is reused.
void sweep_stage_prepare(SweepStage &st, const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x,
                         int64_t ld_x, int nrhs, const SweepCoupling *cpl, int ncpl, SweepStage *const *ext,
                         int next, cudaStream_t s, int64_t vals_tag = 0, int ncta = 0, bool grid = false,
                         int warps_force = 0);
int sweep_stage_warps(const SweepStage &st);
// After every slab k, add sum_c coef_c C_c src_c(k) to target's right-hand side of
// slab k (before publishing slab k).  Sources: this stage's x_k (ext < 0) or its
// external stages.  Call after both stages are prepared, before the launch.
void sweep_stage_set_post(SweepStage &st, SweepStage &target, const SweepCoupling *cpl, int ncpl, cudaStream_t s,
                          int64_t vals_tag = 0);
// Run prepared stages in ONE launch, one 16-CTA cluster each, pipelined slab by slab
// (a consumer waits on per-slab release flags of its producers); then permute out.
// Stages prepared with grid = true (or ncta != 16) form a grid-family launch: no
// clusters, cooperative launch, stage i on its own ncta CTAs with a software barrier.
void sweep_stages_launch(SweepStage *const *st, int nst, cudaStream_t s);
// throws STMHD_CUDA if a completed pipelined launch recorded a producer timeout
void sweep_check_fault(cudaStream_t s);

// Cluster-resident sweep in nested-dissection order (nd_sweep.cu).
void nd_sweep(const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
              const SweepCoupling *cpl, int ncpl, cudaStream_t s);

}  // namespace stmhd
