// K3-K6: the space-time block preconditioner P_T and its sub-operators.
//
// Reference: SpaceTimePreconditioner (pkg/src/stmhd/precond.py:60-387).
// Setup builds C_A,k = f_a,k D^-1 f_a,k + s_k K_A^bc0 and the wave
// sub-diagonals with fixed gather plans (precond.py:91-105), then factors
// F_u,k and C_A,k for all slabs at once (nested-dissection supernodal LU,
// nd_numeric.cu).  Applications chain batched exact solves, block-bidiagonal
// SpMVs and the two sequential sweeps exactly in the reference order
// (precond.py:270-301).
#include "pc.hpp"

namespace stmhd {

__global__ void ca_values_kernel(int nnz, int nt, const int *pptr, const int *pa, const int *pb, const double *pw,
                                 const double *kval, const double *js, int64_t nnz_js, const double *alf,
                                 double *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  for (int k = blockIdx.y; k < nt; k += gridDim.y) {
    const double *f = js + (int64_t)k * nnz_js;
    double acc = 0.0;
    for (int p = pptr[t]; p < pptr[t + 1]; ++p) acc += f[pa[p]] * pw[p] * f[pb[p]];
    out[(int64_t)k * nnz + t] = acc + alf[k] * kval[t];
  }
}

__global__ void s1_values_kernel(int nnz, int nt1, const int *pptr, const double *coef, const int *idx,
                                 const int *which, const double *js, int64_t nnz_js, double *out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nnz) return;
  for (int k = blockIdx.y; k < nt1; k += gridDim.y) {
    double acc = 0.0;
    for (int p = pptr[t]; p < pptr[t + 1]; ++p) acc += coef[p] * js[(int64_t)(k + which[p]) * nnz_js + idx[p]];
    out[(int64_t)k * nnz + t] = acc;
  }
}

__global__ void zero_pin_copy(const double *in, int64_t ld_in, double *out, int64_t ld_out, int n, int pin) {
  const int k = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[(int64_t)k * ld_out + i] = (i == pin) ? 0.0 : in[(int64_t)k * ld_in + i];
}

// x_k = -y_k + alpha_k, alpha_k = (r_pin - (-y_k).w) / p_mean_mass (precond.py:224-226)
__global__ void pressure_alpha_kernel(const double *y, int64_t ld_y, const double *r, int64_t ld_r, int pin,
                                      const double *w, int n, double pmm, double *out, int64_t ld_out) {
  __shared__ double sh[32];
  const int k = blockIdx.x;
  const double *yk = y + (int64_t)k * ld_y;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += (-yk[i]) * w[i];
  acc = block_sum(acc, sh);
  const double alpha = (r[(int64_t)k * ld_r + pin] - acc) / pmm;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[(int64_t)k * ld_out + i] = -yk[i] + alpha;
}

__global__ void copy2d(const double *in, int64_t ld_in, double *out, int64_t ld_out, int n) {
  const int k = blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[(int64_t)k * ld_out + i] = in[(int64_t)k * ld_in + i];
}

// ---------------------------------------------------------------------------

PC::PC(stmhd_disc_s *dd, cudaStream_t s, const double *js_, const double *fp_, const double *alf_, int var)
    : d(dd), js(js_), fp(fp_), variant(var) {
  nt = (int)d->I("nt");
  n_u = (int)d->I("n_u");
  n_p = (int)d->I("n_p");
  n_j = (int)d->I("n_j");
  n_a = (int)d->I("n_a");
  slab = d->slab();
  o_p = n_u;
  o_j = n_u + n_p;
  o_a = o_j + n_j;
  nnz_js = d->I("nnz_js");
  nnz_fp = d->I("nnz_fp");
  nnz_ca = d->H("ca_col").count;
  nnz_s1 = d->H("s1_col").count;
  alf.alloc_async(nt * sizeof(double), s);
  STMHD_CUDA_CHECK(cudaMemcpyAsync(alf.ptr, alf_, nt * sizeof(double), cudaMemcpyDeviceToDevice, s));
  // C_A and sub1 values (precond.py:91-105)
  ca_vals.alloc_async((size_t)nt * nnz_ca * sizeof(double), s);
  ca_values_kernel<<<dim3(cdiv(nnz_ca, 256), std::min(nt, 16)), 256, 0, s>>>(
      (int)nnz_ca, nt, d->D<int>("ca_pptr"), d->D<int>("ca_a"), d->D<int>("ca_b"), d->D<double>("ca_w"),
      d->D<double>("ca_k"), js, nnz_js, alf.as<double>(), ca_vals.as<double>());
  STMHD_LAUNCH_CHECK();
  if (nt > 1) {
    s1_vals.alloc_async((size_t)(nt - 1) * nnz_s1 * sizeof(double), s);
    s1_values_kernel<<<dim3(cdiv(nnz_s1, 256), std::min(nt - 1, 16)), 256, 0, s>>>(
        (int)nnz_s1, nt - 1, d->D<int>("s1_pptr"), d->D<double>("s1_coef"), d->D<int>("s1_idx"),
        d->D<int>("s1_which"), js, nnz_js, s1_vals.as<double>());
    STMHD_LAUNCH_CHECK();
  } else {
    s1_vals.alloc_async(sizeof(double), s);
  }
  // workspaces
  tu1.alloc_async((size_t)nt * n_u * sizeof(double), s);
  tu2.alloc_async((size_t)nt * n_u * sizeof(double), s);
  ta1.alloc_async((size_t)nt * n_a * sizeof(double), s);
  ta2.alloc_async((size_t)nt * n_a * sizeof(double), s);
  ta3.alloc_async((size_t)nt * n_a * sizeof(double), s);
  tp1.alloc_async((size_t)nt * n_p * sizeof(double), s);
  tp2.alloc_async((size_t)nt * n_p * sizeof(double), s);
  tp3.alloc_async((size_t)nt * n_p * sizeof(double), s);
  tj.alloc_async((size_t)nt * n_j * sizeof(double), s);
  // factorisations (precond.py:75, 96)
  fu = std::make_unique<NDFactor>();
  fu->dev = d->dev_fu.get();
  fu->nbatch = nt;
  fu->factor(js, nnz_js, s);
  if (int st = fu->check_status(s)) throw Error(STMHD_SINGULAR, "F_u factorisation: zero pivot", "F_u");
  ca = std::make_unique<NDFactor>();
  ca->dev = d->dev_ca.get();
  ca->nbatch = nt;
  ca->factor(ca_vals.as<double>(), nnz_ca, s);
  if (int st = ca->check_status(s)) throw Error(STMHD_SINGULAR, "C_A factorisation: zero pivot", "C_A");
}

void PC::ensure_forward_factors(cudaStream_t s) {
  if (!fa) {
    fa = std::make_unique<NDFactor>();
    fa->dev = d->dev_fa.get();
    fa->nbatch = nt;
    fa->factor(js, nnz_js, s);
    if (fa->check_status(s)) throw Error(STMHD_SINGULAR, "F_A factorisation: zero pivot", "F_A");
  }
  if (!fpf) {
    fpf = std::make_unique<NDFactor>();
    fpf->dev = d->dev_fp.get();
    fpf->nbatch = nt;
    fpf->factor(fp, nnz_fp, s);
    if (fpf->check_status(s)) throw Error(STMHD_SINGULAR, "F_p factorisation: zero pivot", "F_p");
  }
}

static SpTerm csr_term(const DCsr &c, const double *x, int64_t xs, double alpha, int lag = 0) {
  SpTerm t;
  t.beg = c.rowptr;
  t.col = c.col;
  t.val = c.val;
  t.x = x;
  t.x_stride = xs;
  t.alpha = alpha;
  t.lag = lag;
  return t;
}

// ---- field operators (in/out are nt x n blocks with leading dimensions) ----

void PC::apply_potential(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_a;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  SpTerm f;
  f.beg = d->D<int>("js_seg0") + o_a;
  f.end = d->D<int>("js_rowptr") + o_a + 1;
  f.col = d->D<int>("js_col");
  f.val = js;
  f.val_stride = nnz_js;
  f.x = in;
  f.x_stride = li;
  f.col_off = (int)o_a;
  a.t[0] = f;
  a.t[1] = csr_term(d->csr("ma_dt"), in, li, -1.0, 1);
  a.nterms = 2;
  spmv(a, s, 8);
}

// C~_A sweep couplings (precond.py:194-205): sub-diagonal S1_k (per slab) and the
// shared second sub-diagonal S2
void PC::wave_couplings(SweepCoupling *c) const {
  c[0].rowptr = d->D<int>("s1_rowptr");
  c[0].col = d->D<int>("s1_col");
  c[0].val = s1_vals.as<double>();
  c[0].val_stride = nnz_s1;
  c[0].val_shift = 1;
  c[0].lag = 1;
  c[0].coef = -1.0;
  DCsr s2 = d->csr("sub2");
  c[1].rowptr = s2.rowptr;
  c[1].col = s2.col;
  c[1].val = s2.val;
  c[1].lag = 2;
  c[1].coef = -1.0;
}

void PC::solve_wave(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SweepCoupling c[2];
  wave_couplings(c);
  ca->sweep(in, li, out, lo, nt, c, 2, s);
}

void PC::apply_wave(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_a;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  SpTerm c;
  c.beg = d->D<int>("ca_rowptr");
  c.col = d->D<int>("ca_col");
  c.val = ca_vals.as<double>();
  c.val_stride = nnz_ca;
  c.x = in;
  c.x_stride = li;
  a.t[0] = c;
  SpTerm s1;
  s1.beg = d->D<int>("s1_rowptr");
  s1.col = d->D<int>("s1_col");
  s1.val = s1_vals.as<double>();
  s1.val_stride = nnz_s1;
  s1.val_shift = 1;
  s1.x = in;
  s1.x_stride = li;
  s1.lag = 1;
  a.t[1] = s1;
  a.t[2] = csr_term(d->csr("sub2"), in, li, 1.0, 2);
  a.nterms = 3;
  spmv(a, s, 8);
}

void PC::solve_potential(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  ensure_forward_factors(s);
  DCsr m = d->csr("ma_dt");
  SweepCoupling c;
  c.rowptr = m.rowptr;
  c.col = m.col;
  c.val = m.val;
  c.lag = 1;
  c.coef = 1.0;
  fa->sweep(in, li, out, lo, nt, &c, 1, s);
}

void PC::magnetic_schur_inverse(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  d->lu_ma->solve(in, li, ta1.as<double>(), n_a, nt, s);
  apply_potential(ta1.as<double>(), n_a, ta2.as<double>(), n_a, s);
  solve_wave(ta2.as<double>(), n_a, out, lo, s);
}

void PC::magnetic_schur_apply(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  apply_wave(in, li, ta1.as<double>(), n_a, s);
  solve_potential(ta1.as<double>(), n_a, ta2.as<double>(), n_a, s);
  SpmvArgs a;
  a.nrows = n_a;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  a.t[0] = csr_term(d->csr("mabc"), ta2.as<double>(), n_a, 1.0);
  a.nterms = 1;
  spmv(a, s, 8);
}

void PC::apply_pressure_cd(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_p;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  SpTerm f;
  f.beg = d->D<int>("fp_rowptr");
  f.col = d->D<int>("fp_col");
  f.val = fp;
  f.val_stride = nnz_fp;
  f.x = in;
  f.x_stride = li;
  a.t[0] = f;
  a.t[1] = csr_term(d->csr("mp_dt"), in, li, -1.0, 1);
  a.nterms = 2;
  spmv(a, s, 8);
}

void PC::solve_pressure_cd(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  ensure_forward_factors(s);
  DCsr m = d->csr("mp_dt");
  SweepCoupling c;
  c.rowptr = m.rowptr;
  c.col = m.col;
  c.val = m.val;
  c.lag = 1;
  c.coef = 1.0;
  fpf->sweep(in, li, out, lo, nt, &c, 1, s);
}

void PC::pressure_schur_inverse(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  const int pin = (int)d->I("p_pin");
  zero_pin_copy<<<dim3(cdiv(n_p, 256), nt), 256, 0, s>>>(in, li, tp1.as<double>(), n_p, n_p, pin);
  STMHD_LAUNCH_CHECK();
  d->lu_kp->solve(tp1.as<double>(), n_p, tp2.as<double>(), n_p, nt, s);
  apply_pressure_cd(tp2.as<double>(), n_p, tp1.as<double>(), n_p, s);
  d->lu_mp->solve(tp1.as<double>(), n_p, tp2.as<double>(), n_p, nt, s);
  pressure_alpha_kernel<<<nt, 256, 0, s>>>(tp2.as<double>(), n_p, in, li, pin, d->D<double>("p_mean_row"), n_p,
                                           d->R("p_mean_mass"), out, lo);
  STMHD_LAUNCH_CHECK();
}

void PC::pressure_schur_apply(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_p;
  a.nslab = nt;
  a.y = tp1.as<double>();
  a.y_stride = n_p;
  a.t[0] = csr_term(d->csr("mp"), in, li, 1.0);
  a.nterms = 1;
  spmv(a, s, 8);
  solve_pressure_cd(tp1.as<double>(), n_p, tp2.as<double>(), n_p, s);
  SpmvArgs b;
  b.nrows = n_p;
  b.nslab = nt;
  b.y = out;
  b.y_stride = lo;
  b.t[0] = csr_term(d->csr("kpz"), tp2.as<double>(), n_p, -1.0);
  b.nterms = 1;
  spmv(b, s, 8);
  const int pin = (int)d->I("p_pin");
  dense_row(d->D<double>("p_mean_row"), n_p, in, li, out + pin, lo, nt, 1.0, s);
}

void PC::solve_velocity(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  DCsr m = d->csr("mu_dt");
  SweepCoupling c;
  c.rowptr = m.rowptr;
  c.col = m.col;
  c.val = m.val;
  c.lag = 1;
  c.coef = 1.0;
  fu->sweep(in, li, out, lo, nt, &c, 1, s);
}

void PC::apply_velocity(const double *in, int64_t li, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_u;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  SpTerm f;
  f.beg = d->D<int>("js_rowptr");
  f.end = d->D<int>("js_seg0");
  f.col = d->D<int>("js_col");
  f.val = js;
  f.val_stride = nnz_js;
  f.x = in;
  f.x_stride = li;
  a.t[0] = f;
  a.t[1] = csr_term(d->csr("mu_dt"), in, li, -1.0, 1);
  a.nterms = 2;
  spmv(a, s, 8);
}

// y = z*beta + Z_j xj + Z_a xa (rows u), with the per-slab blocks of the merged pattern
void PC::coupling_u(const double *z, int64_t lz, double beta, const double *xs, int64_t lxs, double alpha,
                    const double *xp, int64_t lxp, double alpha_p, double *out, int64_t lo, cudaStream_t s) {
  SpmvArgs a;
  a.nrows = n_u;
  a.nslab = nt;
  a.y = out;
  a.y_stride = lo;
  a.z = z;
  a.z_stride = lz;
  a.beta = beta;
  SpTerm zj;
  zj.beg = d->D<int>("js_seg0");
  zj.end = d->D<int>("js_rowptr") + 1;  // z_j | z_a segments are contiguous
  zj.col = d->D<int>("js_col");
  zj.val = js;
  zj.val_stride = nnz_js;
  zj.x = xs;
  zj.x_stride = lxs;
  zj.alpha = alpha;
  a.t[0] = zj;
  a.nterms = 1;
  if (xp) {
    a.t[1] = csr_term(d->csr("divt"), xp, lxp, alpha_p);
    a.nterms = 2;
  }
  spmv(a, s, 8);
}

// TRIANGULAR P_T^{-1} (precond.py:270-300) with the three sequential sweeps of one
// application -- the C~_A wave sweep (x_A), the M_j solves (x_j = M_j^{-1}(r_j - K x_A))
// and the F_u sweep (rhs r_u - B^T x_p - Z_j x_j - Z_a x_A) -- in ONE launch, one
// cluster each, pipelined slab by slab: slab k of a consumer starts as soon as its
// producers have published slab k.  Same arithmetic as apply_inverse's sequential
// path up to the summation order of the coupled right-hand sides.
void PC::apply_inverse_pipelined(const double *r, double *x, cudaStream_t s) {
  const double *r_u = r, *r_p = r + o_p, *r_j = r + o_j, *r_a = r + o_a;
  // batched (slab-parallel) pre-steps; the pressure chain runs on a second stream,
  // overlapped with the wave right-hand side, and joins before the velocity stage
  // side stream and events owned by the discretisation (it outlives its
  // preconditioners; buffers pooled on the stream are released before it is destroyed)
  if (!d->side) {
    STMHD_CUDA_CHECK(cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking));
    STMHD_CUDA_CHECK(cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming));
    STMHD_CUDA_CHECK(cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming));
  }
  cudaStream_t side = d->side;
  cudaEvent_t ev_fork = d->ev_fork, ev_join = d->ev_join;
  STMHD_CUDA_CHECK(cudaEventRecord(ev_fork, s));
  STMHD_CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork, 0));
  pressure_schur_inverse(r_p, slab, x + o_p, slab, side);
  {  // tu1 = r_u - B^T x_p
    cudaStream_t s = side;
    SpmvArgs a;
    a.nrows = n_u;
    a.nslab = nt;
    a.y = tu1.as<double>();
    a.y_stride = n_u;
    a.z = r_u;
    a.z_stride = slab;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("divt"), x + o_p, slab, -1.0);
    a.nterms = 1;
    spmv(a, s, 8);
  }
  STMHD_CUDA_CHECK(cudaEventRecord(ev_join, side));
  d->lu_ma->solve(r_a, slab, ta1.as<double>(), n_a, nt, s);
  apply_potential(ta1.as<double>(), n_a, ta2.as<double>(), n_a, s);
  if (!st_wave) {
    st_wave = sweep_stage_new();
    st_mj = sweep_stage_new();
    st_vel = sweep_stage_new();
  }
  SweepCoupling cw[2];
  wave_couplings(cw);
  // gathered coupling values depend only on this preconditioner's values: reuse them
  static int64_t next_tag = 0;
  if (!vals_tag) vals_tag = ++next_tag;
  const int64_t tag = vals_tag;
  // large velocity factors (64^2 meshes: 45 MB per slab) stream faster from most of
  // the GPU: grid-family launch with the wave and M_j sweeps on 16 CTAs each and the
  // velocity sweep on the remaining SMs (software barriers); smaller ones keep the
  // three-cluster launch (hardware cluster barrier, dense top)
  static const int grid_env = [] {
    const char *e = getenv("STMHD_PC_GRID");
    return e ? atoi(e) : -1;
  }();
  // (round 2: with the 2^(levels-5)-subtree plans and early coupling the grid family
  // also wins at 32^2 -- C2 2.74 -> 2.47 ms -- but not at 16^2, C1 0.26 vs 0.37 ms:
  // velocity factors above 4 MB per slab take it)
  const bool grid = grid_env == 1 || (grid_env < 0 && 8.0 * (double)fu->dev->plan->factor_size > 4e6 &&
                                      num_sms() >= 64);
  static const int fu_ctas_env = [] {
    const char *e = getenv("STMHD_PC_FU_CTAS");
    return e ? atoi(e) : 0;
  }();
  // CTAs of the wave and M_j stages in the grid-family launch (STMHD_PC_SIDE_CTAS,
  // default 16); the velocity stage takes the remaining SMs
  static const int side_env = [] {
    const char *e = getenv("STMHD_PC_SIDE_CTAS");
    return e ? atoi(e) : 16;
  }();
  const int nc_side = grid ? std::max(1, std::min(side_env, 32)) : 16;
  const int nc_fu = grid ? (fu_ctas_env > 0 ? std::min(fu_ctas_env, num_sms() - 2 * nc_side)
                                            : num_sms() - 2 * nc_side)
                         : 16;
  // grid-family launches need one warp count for all stages: the velocity stage's
  // choice (the others have slack) is remembered on the discretisation after the first
  // preparation
  int &pipe_warps = d->pipe_warps;
  const int wf = grid ? pipe_warps : 0;
  sweep_stage_prepare(*st_wave, *ca, ta2.as<double>(), n_a, x + o_a, slab, nt, cw, 2, nullptr, 0, s, tag, nc_side, grid, wf);
  SweepCoupling cj;  // -K_jA x_A
  DCsr mix = d->csr("mixja");
  cj.rowptr = mix.rowptr;
  cj.col = mix.col;
  cj.val = mix.val;
  cj.ext = 0;
  cj.coef = -1.0;
  SweepStage *wj[1] = {st_wave.get()};
  sweep_stage_prepare(*st_mj, *d->lu_mj, r_j, slab, x + o_j, slab, nt, &cj, 1, wj, 1, s, tag, nc_side, grid, wf);
  SweepCoupling cu;  // + M_u/dt x_u(k-1); waits on the M_j stage (which adds the Z terms)
  DCsr m = d->csr("mu_dt");
  cu.rowptr = m.rowptr;
  cu.col = m.col;
  cu.val = m.val;
  cu.lag = 1;
  cu.coef = 1.0;
  SweepStage *ju[1] = {st_mj.get()};
  STMHD_CUDA_CHECK(cudaStreamWaitEvent(s, ev_join, 0));  // tu1 (pressure chain) ready
  sweep_stage_prepare(*st_vel, *fu, tu1.as<double>(), n_u, x, slab, nt, &cu, 1, ju, 1, s, tag, nc_fu, grid, wf);
  if (grid && !pipe_warps) {
    pipe_warps = sweep_stage_warps(*st_vel);
    if (sweep_stage_warps(*st_wave) != pipe_warps || sweep_stage_warps(*st_mj) != pipe_warps) {
      sweep_stage_prepare(*st_wave, *ca, ta2.as<double>(), n_a, x + o_a, slab, nt, cw, 2, nullptr, 0, s, tag, nc_side,
                          grid, pipe_warps);
      sweep_stage_prepare(*st_mj, *d->lu_mj, r_j, slab, x + o_j, slab, nt, &cj, 1, wj, 1, s, tag, nc_side, grid,
                          pipe_warps);
      sweep_stage_prepare(*st_vel, *fu, tu1.as<double>(), n_u, x, slab, nt, &cu, 1, ju, 1, s, tag, nc_fu, grid,
                          pipe_warps);
    }
  }
  // after slab k of the M_j stage: rhs_u(k) += -Z_j x_j(k) - Z_a x_A(k)
  SweepCoupling cz[2];
  cz[0].rowptr = d->D<int>("js_seg0");  // z_j segment of the u rows, slab columns o_j + j
  cz[0].rowend = d->D<int>("js_seg1");
  cz[0].col = d->D<int>("js_col");
  cz[0].col_off = (int)o_j;
  cz[0].val = js;
  cz[0].val_stride = nnz_js;
  cz[0].coef = -1.0;                    // source: the M_j stage's own x_j(k)
  cz[1].rowptr = d->D<int>("js_seg1");  // z_a segment, slab columns o_a + a
  cz[1].rowend = d->D<int>("js_rowptr") + 1;
  cz[1].col = d->D<int>("js_col");
  cz[1].col_off = (int)o_a;
  cz[1].val = js;
  cz[1].val_stride = nnz_js;
  cz[1].ext = 0;                        // source: the wave stage's x_A(k)
  cz[1].coef = -1.0;
  sweep_stage_set_post(*st_mj, *st_vel, cz, 2, s, tag);
  SweepStage *all[3] = {st_wave.get(), st_mj.get(), st_vel.get()};
  sweep_stages_launch(all, 3, s);
}

void PC::apply_inverse(const double *r, double *x, cudaStream_t s) {
  static const int pipelined = [] {
    const char *e = getenv("STMHD_PC_PIPELINE");
    return e ? atoi(e) : 1;
  }();
  if (variant == 0 && pipelined) {
    apply_inverse_pipelined(r, x, s);
    return;
  }
  const double *r_u = r, *r_p = r + o_p, *r_j = r + o_j, *r_a = r + o_a;
  int64_t lr_u = slab, lr_p = slab, lr_a = slab;
  if (variant == 2) {
    // FULL: r_A += Y F_u^{-1} (Z_j M_j^{-1} r_j - r_u)   (precond.py:276-283)
    d->lu_mj->solve(r_j, slab, tj.as<double>(), n_j, nt, s);
    // tu1 = Z_j tj - r_u  (z_j columns are slab coordinates o_j + n)
    SpmvArgs a;
    a.nrows = n_u;
    a.nslab = nt;
    a.y = tu1.as<double>();
    a.y_stride = n_u;
    a.z = r_u;
    a.z_stride = slab;
    a.beta = -1.0;
    SpTerm zj;
    zj.beg = d->D<int>("js_seg0");
    zj.end = d->D<int>("js_seg1");
    zj.col = d->D<int>("js_col");
    zj.val = js;
    zj.val_stride = nnz_js;
    zj.x = tj.as<double>();
    zj.x_stride = n_j;
    zj.col_off = (int)o_j;
    a.t[0] = zj;
    a.nterms = 1;
    spmv(a, s, 8);
    solve_velocity(tu1.as<double>(), n_u, tu2.as<double>(), n_u, s);
    SpmvArgs b;
    b.nrows = n_a;
    b.nslab = nt;
    b.y = ta3.as<double>();
    b.y_stride = n_a;
    b.z = r_a;
    b.z_stride = slab;
    b.beta = 1.0;
    SpTerm y;
    y.beg = d->D<int>("js_rowptr") + o_a;
    y.end = d->D<int>("js_seg0") + o_a;
    y.col = d->D<int>("js_col");
    y.val = js;
    y.val_stride = nnz_js;
    y.x = tu2.as<double>();
    y.x_stride = n_u;
    b.t[0] = y;
    b.nterms = 1;
    spmv(b, s, 8);
    r_a = ta3.as<double>();
    lr_a = n_a;
  }
  // x_A = S_A^{-1} r_A (precond.py:285)
  magnetic_schur_inverse(r_a, lr_a, x + o_a, slab, s);
  // x_j = M_j^{-1}(r_j - K_jA x_A) (precond.py:286-288)
  {
    SpmvArgs a;
    a.nrows = n_j;
    a.nslab = nt;
    a.y = tj.as<double>();
    a.y_stride = n_j;
    a.z = r_j;
    a.z_stride = slab;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("mixja"), x + o_a, slab, -1.0);
    a.nterms = 1;
    spmv(a, s, 8);
    d->lu_mj->solve(tj.as<double>(), n_j, x + o_j, slab, nt, s);
  }
  // t_u = r_u - Z_j x_j - Z_a x_A (precond.py:289-291) -> tu1
  coupling_u(r_u, lr_u, 1.0, x, slab, -1.0, nullptr, 0, 0.0, tu1.as<double>(), n_u, s);
  if (variant == 1 || variant == 2) {
    // r_p -= B F_u^{-1} t_u (precond.py:293-296)
    solve_velocity(tu1.as<double>(), n_u, tu2.as<double>(), n_u, s);
    SpmvArgs a;
    a.nrows = n_p;
    a.nslab = nt;
    a.y = tp3.as<double>();
    a.y_stride = n_p;
    a.z = r_p;
    a.z_stride = slab;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("div"), tu2.as<double>(), n_u, -1.0);
    a.nterms = 1;
    spmv(a, s, 8);
    r_p = tp3.as<double>();
    lr_p = n_p;
  }
  // x_p = S_p^{-1} r_p (precond.py:298)
  pressure_schur_inverse(r_p, lr_p, x + o_p, slab, s);
  // rhs_u = t_u - B^T x_p ; x_u = F_u^{-1} rhs_u (precond.py:299-300)
  {
    SpmvArgs a;
    a.nrows = n_u;
    a.nslab = nt;
    a.y = tu2.as<double>();
    a.y_stride = n_u;
    a.z = tu1.as<double>();
    a.z_stride = n_u;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("divt"), x + o_p, slab, -1.0);
    a.nterms = 1;
    spmv(a, s, 8);
  }
  solve_velocity(tu2.as<double>(), n_u, x, slab, s);
}

void PC::apply_forward(const double *xin, double *out, cudaStream_t s) {
  // precond.py:303-340
  const double *x_u = xin, *x_p = xin + o_p, *x_j = xin + o_j, *x_a = xin + o_a;
  // o_j = M_j x_j + K_jA x_a
  {
    SpmvArgs a;
    a.nrows = n_j;
    a.nslab = nt;
    a.y = out + o_j;
    a.y_stride = slab;
    a.t[0] = csr_term(d->csr("mj"), x_j, slab, 1.0);
    a.t[1] = csr_term(d->csr("mixja"), x_a, slab, 1.0);
    a.nterms = 2;
    spmv(a, s, 8);
  }
  magnetic_schur_apply(x_a, slab, out + o_a, slab, s);
  if (variant == 0) {
    // o_u = F_u x_u (bidiagonal) + Z_j x_j + Z_a x_a + B^T x_p
    apply_velocity(x_u, slab, tu1.as<double>(), n_u, s);
    coupling_u(tu1.as<double>(), n_u, 1.0, xin, slab, 1.0, x_p, slab, 1.0, out, slab, s);
    pressure_schur_apply(x_p, slab, out + o_p, slab, s);
    return;
  }
  // SIMPLIFIED / FULL: velocity-pressure upper factor t_u = F_u x_u + B^T x_p
  apply_velocity(x_u, slab, tu1.as<double>(), n_u, s);
  {
    SpmvArgs a;
    a.nrows = n_u;
    a.nslab = nt;
    a.y = tu1.as<double>();
    a.y_stride = n_u;
    a.z = tu1.as<double>();
    a.z_stride = n_u;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("divt"), x_p, slab, 1.0);
    a.nterms = 1;
    spmv(a, s, 8);
  }
  pressure_schur_apply(x_p, slab, out + o_p, slab, s);
  // velocity-pressure lower factor: o_p += B F_u^{-1} t_u
  solve_velocity(tu1.as<double>(), n_u, tu2.as<double>(), n_u, s);
  {
    SpmvArgs a;
    a.nrows = n_p;
    a.nslab = nt;
    a.y = out + o_p;
    a.y_stride = slab;
    a.z = out + o_p;
    a.z_stride = slab;
    a.beta = 1.0;
    a.t[0] = csr_term(d->csr("div"), tu2.as<double>(), n_u, 1.0);
    a.nterms = 1;
    spmv(a, s, 8);
  }
  // o_u = t_u + Z_j x_j + Z_a x_a (the velocity-magnetic upper factor absorbed F_u^{-1})
  coupling_u(tu1.as<double>(), n_u, 1.0, xin, slab, 1.0, nullptr, 0, 0.0, out, slab, s);
  if (variant == 2) {
    // velocity-magnetic lower factor: o_A += Y F_u^{-1}(o_u - Z_j M_j^{-1} o_j)
    d->lu_mj->solve(out + o_j, slab, tj.as<double>(), n_j, nt, s);
    SpmvArgs a;
    a.nrows = n_u;
    a.nslab = nt;
    a.y = tu1.as<double>();
    a.y_stride = n_u;
    a.z = out;
    a.z_stride = slab;
    a.beta = 1.0;
    SpTerm zj;
    zj.beg = d->D<int>("js_seg0");
    zj.end = d->D<int>("js_seg1");
    zj.col = d->D<int>("js_col");
    zj.val = js;
    zj.val_stride = nnz_js;
    zj.x = tj.as<double>();
    zj.x_stride = n_j;
    zj.col_off = (int)o_j;
    zj.alpha = -1.0;
    a.t[0] = zj;
    a.nterms = 1;
    spmv(a, s, 8);
    solve_velocity(tu1.as<double>(), n_u, tu2.as<double>(), n_u, s);
    SpmvArgs b;
    b.nrows = n_a;
    b.nslab = nt;
    b.y = out + o_a;
    b.y_stride = slab;
    b.z = out + o_a;
    b.z_stride = slab;
    b.beta = 1.0;
    SpTerm y;
    y.beg = d->D<int>("js_rowptr") + o_a;
    y.end = d->D<int>("js_seg0") + o_a;
    y.col = d->D<int>("js_col");
    y.val = js;
    y.val_stride = nnz_js;
    y.x = tu2.as<double>();
    y.x_stride = n_u;
    b.t[0] = y;
    b.nterms = 1;
    spmv(b, s, 8);
  }
}

void PC::op(int which, const double *in, double *out, cudaStream_t s) {
  switch (which) {
    case 0: solve_velocity(in, n_u, out, n_u, s); break;
    case 1: apply_velocity(in, n_u, out, n_u, s); break;
    case 2: solve_wave(in, n_a, out, n_a, s); break;
    case 3: apply_wave(in, n_a, out, n_a, s); break;
    case 4: apply_potential(in, n_a, out, n_a, s); break;
    case 5: solve_potential(in, n_a, out, n_a, s); break;
    case 6: pressure_schur_inverse(in, n_p, out, n_p, s); break;
    case 7: pressure_schur_apply(in, n_p, out, n_p, s); break;
    case 8: magnetic_schur_inverse(in, n_a, out, n_a, s); break;
    case 9: magnetic_schur_apply(in, n_a, out, n_a, s); break;
    case 10: apply_pressure_cd(in, n_p, out, n_p, s); break;
    case 11: solve_pressure_cd(in, n_p, out, n_p, s); break;
    default: throw Error(STMHD_CONFIG, "stmhd_pc_op: unknown operator");
  }
}

}  // namespace stmhd
