// Preconditioner handle (reference SpaceTimePreconditioner, precond.py:60-387).
#pragma once

#include "disc.hpp"

namespace stmhd {

struct PC {
  stmhd_disc_s *d;
  const double *js, *fp;  // caller-owned per-slab values (Jacobian, F_p)
  int variant;
  int nt, n_u, n_p, n_j, n_a;
  int64_t slab, o_p, o_j, o_a, nnz_js, nnz_fp, nnz_ca, nnz_s1;
  DevBuf alf, ca_vals, s1_vals;
  DevBuf tu1, tu2, ta1, ta2, ta3, tp1, tp2, tp3, tj;
  std::unique_ptr<NDFactor> fu, ca, fa, fpf;
  SweepStagePtr st_wave, st_mj, st_vel;  // pipelined apply_inverse (TRIANGULAR)
  int64_t vals_tag = 0;                  // this preconditioner's coupling-value generation

  PC(stmhd_disc_s *d, cudaStream_t s, const double *js, const double *fp, const double *alf, int variant);
  void ensure_forward_factors(cudaStream_t s);

  void apply_potential(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void solve_potential(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void apply_wave(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void solve_wave(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void magnetic_schur_inverse(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void magnetic_schur_apply(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void apply_pressure_cd(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void solve_pressure_cd(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void pressure_schur_inverse(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void pressure_schur_apply(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void solve_velocity(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void apply_velocity(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s);
  void coupling_u(const double *z, int64_t lz, double beta, const double *xs, int64_t lxs, double alpha,
                  const double *xp, int64_t lxp, double alpha_p, double *out, int64_t lo, cudaStream_t s);
  void wave_couplings(SweepCoupling *c) const;
  void apply_inverse(const double *r, double *x, cudaStream_t s);
  void apply_inverse_pipelined(const double *r, double *x, cudaStream_t s);
  void apply_forward(const double *x, double *out, cudaStream_t s);
  void op(int which, const double *in, double *out, cudaStream_t s);
};

void assemble(stmhd_disc_s *d, cudaStream_t s, const double *state, const double *ic_u, const double *ic_a,
              double *res, double *js, double *fp, double *alf);
int64_t gs_work_size(int64_t n, int nvec);
void gs_dots(cudaStream_t s, const double *V, int64_t ldv, int nvec, const double *w, int64_t n, double *h,
             double *work);
void gs_update(cudaStream_t s, const double *V, int64_t ldv, int nvec, const double *h, double *w, int64_t n,
               double *h2, double *nrm2, double *work);
void gs_normalize(cudaStream_t s, const double *x, double *y, int64_t n, const double *nrm2);
void gs_combine(cudaStream_t s, const double *Z, int64_t ldz, int nvec, const double *c, double *x, int64_t n);
void axpby(cudaStream_t s, double a, const double *x, double b, const double *y, double *out, int64_t n,
           double *nrm2, double *work);

}  // namespace stmhd

struct stmhd_pc_s {
  std::unique_ptr<stmhd::PC> pc;
};
