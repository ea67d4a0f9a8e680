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
  std::vector<int64_t> fl_off, fu_off, front_off, cbv_off;
  int64_t factor_size = 0, front_size = 0, cbv_size = 0;
  int64_t sym_nnz = 0;  // nnz of L+U implied by the supernodal structure
  int max_front = 0;
  std::vector<std::vector<int>> level_sn;
};

// Build the plan.  gx/gy may be null (graph bisection).  value_map (may be null)
// maps pattern entries to caller value indices.
NDPlan nd_analyze(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *gx,
                  const int32_t *gy, int leaf_max, const int32_t *value_map);

// Work list of the cluster-resident time sweep (nd_sweep.cu), built lazily for
// a launch shape: per level and warp, contiguous chunk ranges of one supernode.
struct alignas(16) SweepTask {
  int s, c0, c1, kl;  // supernode, chunk range (chunks of 32/kl rows), lanes per row
  int ns, f, rows, pad;
  int64_t foff;   // factor offset (FL^T forward, FU^T backward)
  int64_t goff;   // offset of the supernode's front tables
  int64_t first;  // elimination position of the first column
  int64_t cboff;  // update-vector offset
};

struct NDSweepPlan {
  int ncta = 0, warps = 0;
  DevBuf fwd_tasks, bwd_tasks, fwd_wptr, bwd_wptr;
  DevBuf g3p;   // int4 per front position: {permuted rhs index or -1, cb1, cb2, 0}
  DevBuf bpos;  // int per front position: permuted position of the front entry
  DevBuf pos;   // n: elimination position of each original index
  DevBuf iperm; // n: original index at each elimination position
  DevBuf seprows;  // permuted rows owned by non-leaf supernodes
  int64_t nsep = 0;
  // permuted column indices of coupling matrices, keyed by their column array
  // (owned by the same discretisation as this plan, so lifetimes match)
  // {rowptr, colp, eidx} of a coupling matrix in elimination order
  mutable std::map<const int *, std::unique_ptr<std::vector<DevBuf>>> colp_cache;
};

// Device-resident copy of a plan plus the solve schedules.
struct NDDevice {
  const NDPlan *plan = nullptr;
  DevBuf ns, nb, first, idx_off, idx, child_ptr, child_list, emap_off, emap, scat_ptr,
      scat_src, scat_dst, fl_off, fu_off, front_off, cbv_off, lvl_sn, lvl_ptr;
  // solve work items: int4 {sn, row_begin, row_end, 0} (32-row chunks); per level ranges
  DevBuf fwd_items, bwd_items, gather3;  // SolveItem lists + flat forward gather table (int4 per front position)
  std::vector<int> fwd_ptr, bwd_ptr;  // host copies of level ranges (nlevels+1)
  DevBuf fwd_ptr_d, bwd_ptr_d;
  int max_front = 0;
  void build(const NDPlan &p, cudaStream_t s);
  mutable std::unique_ptr<NDSweepPlan> sweep_plan;
  const NDSweepPlan &get_sweep_plan(int ncta, int warps, cudaStream_t s) const;
};

// A coupling term of a sequential block sweep:
//   rhs_k += coef * C_(k) x_(k-lag)   (C in CSR with per-slab value stride)
struct SweepCoupling {
  const int32_t *rowptr = nullptr;
  const int32_t *col = nullptr;
  const double *val = nullptr;
  int64_t val_stride = 0;  // 0: shared matrix
  int64_t val_shift = 0;   // value block used for slab k is (k - val_shift)
  int lag = 0;             // 0 = unused
  double coef = 0.0;
};

// Flat descriptor of one solve work item: everything a warp needs in one load.
struct alignas(16) SolveItem {
  int s, r0, r1, kl;  // supernode, row range, lanes per row
  int ns, f, pad0, pad1;
  int64_t foff;   // factor offset (FL^T forward, FU^T backward)
  int64_t goff;   // offset of the supernode's front lists (idx / gather3)
  int64_t first;  // elimination position of the first column
  int64_t cboff;  // update-vector offset
};

struct NDFactor {
  const NDDevice *dev = nullptr;
  int nbatch = 0;
  DevBuf factors;  // nbatch * factor_size doubles
  DevBuf status;   // int: 0 ok, 1+ singular (first failing supernode+1)
  void factor(const double *values, int64_t value_stride, cudaStream_t s);
  // x_b = A_b^{-1} rhs_b (b < nrhs; factor b, or 0 if nbatch == 1).
  void solve(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
             cudaStream_t s) const;
  // Sequential sweep over slabs k = 0..nrhs-1:
  //   x_k = A_k^{-1}( rhs_k + sum_t coef_t C_t x_(k-lag_t) )
  void sweep(const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
             const SweepCoupling *cpl, int ncpl, cudaStream_t s) const;
  int check_status(cudaStream_t s) const;  // synchronises
};

// Cluster-resident sweep in nested-dissection order (nd_sweep.cu).
void nd_sweep(const NDFactor &fac, const double *rhs, int64_t ld_rhs, double *x, int64_t ld_x, int nrhs,
              const SweepCoupling *cpl, int ncpl, cudaStream_t s);

}  // namespace stmhd
