// Discretisation handle: named device tables + constant factorisations.
#pragma once

#include <memory>
#include <string>
#include <unordered_map>

#include "nd.hpp"
#include "stspmv.hpp"

struct stmhd_disc_s;

namespace stmhd {

struct HostArray {
  std::vector<char> data;
  int elem = 0;
  int64_t count = 0;
  template <class T> const T *as() const { return reinterpret_cast<const T *>(data.data()); }
};

// Compressed sparse rows on the device (field-local coordinates).
struct DCsr {
  const int *rowptr = nullptr, *col = nullptr;
  const double *val = nullptr;
  int nrows = 0;
};

// One term of the batched multi-term SpMV (spmv.cu).
struct SpTerm {
  const int *beg = nullptr;  // row r entries: [beg[r], end ? end[r] : beg[r+1])
  const int *end = nullptr;
  const int *col = nullptr;
  const double *val = nullptr;
  int64_t val_stride = 0;  // per-slab stride of the values (0: shared)
  int val_shift = 0;       // slab k uses value block k - val_shift
  const double *x = nullptr;
  int64_t x_stride = 0;  // slab stride of x
  int col_off = 0;       // x index = (k-lag)*x_stride + col - col_off
  int lag = 0;           // term skipped for k < lag
  int rel = 0;           // 1: columns relative to slab start, may reach into k-1 (skip <0)
  double alpha = 1.0;
};

struct SpmvArgs {
  int nrows = 0, nslab = 0, kbeg = 0;
  double *y = nullptr;
  int64_t y_stride = 0;
  const double *z = nullptr;  // y = beta*z + sum terms
  int64_t z_stride = 0;
  double beta = 0.0;
  SpTerm t[4];
  int nterms = 0;
};

void spmv(const SpmvArgs &a, cudaStream_t s, int group = 8);
// y[k*ys + off] += alpha * dot(w, x[k*xs .. +n])   for k < nslab  (dense row)
void dense_row(const double *w, int n, const double *x, int64_t xs, double *y, int64_t ys,
               int nslab, double alpha, cudaStream_t s);

}  // namespace stmhd

struct stmhd_disc_s {
  std::unordered_map<std::string, int64_t> ints;
  std::unordered_map<std::string, double> reals;
  std::unordered_map<std::string, stmhd::HostArray> host;
  std::unordered_map<std::string, stmhd::DevBuf> dev;
  bool finalized = false;
  // grid-family pipelined P_T^-1: common warps per CTA of its stages, chosen by the
  // velocity stage at the first launch and kept for every later preconditioner (a
  // per-preconditioner choice re-prepared the wave / M_j stages, rebuilding their K)
  int pipe_warps = 0;
  // nested-dissection plans (symbolic) and constant factors
  std::unique_ptr<stmhd::NDPlan> plan_fu, plan_ca, plan_fa, plan_fp, plan_mj, plan_ma, plan_mp, plan_kp;
  std::unique_ptr<stmhd::NDDevice> dev_fu, dev_ca, dev_fa, dev_fp, dev_mj, dev_ma, dev_mp, dev_kp;
  std::unique_ptr<stmhd::NDFactor> lu_mj, lu_ma, lu_mp, lu_kp;
  stmhd::DevBuf clamped;  // nt*slab clamped state workspace
  std::unique_ptr<stmhd::StSpmvPlan> jv_plan;  // J.v row blocks (built at the first apply)
  // side stream + fork/join events of the P_T^-1 pre-steps (pressure chain), owned by
  // the discretisation: buffers pooled on it are released before it is destroyed
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~stmhd_disc_s();

  int64_t I(const char *k) const;
  double R(const char *k) const;
  template <class T> const T *D(const char *k) const {
    auto it = dev.find(k);
    if (it == dev.end()) throw stmhd::Error(STMHD_MISSING, std::string("missing device array '") + k + "'");
    return it->second.as<T>();
  }
  const stmhd::HostArray &H(const char *k) const;
  stmhd::DCsr csr(const char *prefix) const;
  int64_t slab() const { return I("n_u") + I("n_p") + I("n_j") + I("n_a"); }
};
