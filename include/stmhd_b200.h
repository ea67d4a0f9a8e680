/*
 * stmhd_b200 -- C-ABI of the B200-native space-time Newton--FGMRES hot path.
 *
 * The reference (arXiv 2309.00768, package `stmhd`) is pure Python; its
 * "plugin interface" for this path is the duck-typed operator API that
 * `_newton` binds (reference pkg/src/stmhd/solver.py:91-101):
 *
 *   residual(state, disc)                 spacetime.py:65      -> stmhd_assemble(residual)
 *   assemble_jacobian(state, disc)        spacetime.py:167     -> stmhd_assemble(slab_values)
 *   SpaceTimeJacobian.apply(v)            spacetime.py:131     -> stmhd_jac_apply
 *   SpaceTimePreconditioner(jac,disc,st)  precond.py:67        -> stmhd_pc_create
 *   SpaceTimePreconditioner.apply_inverse precond.py:270       -> stmhd_pc_apply(direction=0)
 *   SpaceTimePreconditioner.apply_forward precond.py:303       -> stmhd_pc_apply(direction=1)
 *   solve_velocity/solve_wave/...         precond.py:122-250   -> stmhd_pc_op
 *   compute_alfven_scaling                precond.py:46        -> stmhd_assemble(alfven)
 *   gmres MGS/Givens inner products       linalg.py:163-199    -> stmhd_gs_* (fused CGS2)
 *   LUFactor(matrix).solve(b)             linalg.py:71-86      -> stmhd_lu_*
 *
 * Conventions
 *  - Every vector / value pointer is DEVICE memory owned by the caller
 *    (FP64).  Index and table arrays handed to *_upload / *_create are HOST
 *    memory; the library copies them and owns the device copies.
 *  - Space-time vectors are slab-major: slab k occupies [k*slab,(k+1)*slab),
 *    fields u|p|j|A inside a slab (reference linalg.py:14-68), u component-major.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All calls are
 *    asynchronous on that stream unless stated otherwise.  A handle is not
 *    thread safe.
 *  - Return value: STMHD_OK or an error status; stmhd_last_error() returns a
 *    thread-local message.  Status -> Python exception (errors.py):
 *    SINGULAR -> SingularMatrixError / PreconditionerError(block),
 *    NONFINITE -> BreakdownError, CONFIG/MISSING -> ConfigurationError.
 */
#ifndef STMHD_B200_H
#define STMHD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STMHD_OK 0
#define STMHD_CONFIG 1
#define STMHD_SINGULAR 2
#define STMHD_NONFINITE 3
#define STMHD_CUDA 4
#define STMHD_MISSING 5

typedef struct stmhd_disc_s *stmhd_disc;
typedef struct stmhd_pc_s *stmhd_pc;
typedef struct stmhd_lu_s *stmhd_lu;

/* 2 since stmhd_pc_apply directions 2/3 (round 2); the Python loader refuses others */
int stmhd_abi_version(void);
/* number of kernels this library has launched so far (all handles) */
int64_t stmhd_launch_count(void);
const char *stmhd_last_error(void);
/* synchronise `stream` and return STMHD_CUDA if a completed pipelined preconditioner
   launch recorded a producer timeout (stages not co-resident); 0 otherwise.  Later
   pipelined launches also report it.  Replaces a device trap, which would kill the
   context. */
int stmhd_device_fault(void *stream);
/* block name of the last SINGULAR status inside the preconditioner ("F_u", "C_A", ...) */
const char *stmhd_last_block(void);

/* ---- discretisation (reference problems.py:141-256; data built on host) -- */
int stmhd_disc_create(stmhd_disc *out);
int stmhd_disc_destroy(stmhd_disc d);
/* scalar parameters: "nt","n_u","n_p","n_j","n_a","nv","np","ne","nn_v","nn_p","nn_1",
   "p_pin", reals "dt","mu","eta","mu0","p_mean_target","p_mean_mass","area","elem_area" */
int stmhd_disc_set_int(stmhd_disc d, const char *key, int64_t value);
int stmhd_disc_set_real(stmhd_disc d, const char *key, double value);
/* named host array (int32 when elem_size==4, float64 when 8); see DESIGN.md
   "device tables" for the list of keys */
int stmhd_disc_upload(stmhd_disc d, const char *key, const void *host, int64_t count,
                      int elem_size);
/* validate, build the nested-dissection symbolic factorisations and factor the
   constant blocks M_j, M_A^bc, M_p, K_p^pin (problems.py:225-228) */
int stmhd_disc_finalize(stmhd_disc d, void *stream);
/* bytes held on the device by this handle */
int64_t stmhd_disc_device_bytes(stmhd_disc d);

/* ---- K1: residual + Jacobian assembly (spacetime.py:65-112, fem.py:341-472) ----
   state/ic_u/ic_a -> residual[N] (NULL to skip), slab_values[nt*nnz_slab] (f_u|z_j|z_a rows
   of u, y|f_a rows of A, BCs applied), fp_values[nt*nnz_fp] (F_p = M_p/dt + W_p + mu K_p,
   precond.py:80-84), alfven[nt] (precond.py:46-57).  Any output may be NULL. */
int stmhd_assemble(stmhd_disc d, void *stream, const double *state, const double *ic_u,
                   const double *ic_a, double *residual, double *slab_values,
                   double *fp_values, double *alfven);
/* ---- K2: space-time Jacobian matvec y = J x (spacetime.py:131-153) ---- */
int stmhd_jac_apply(stmhd_disc d, void *stream, const double *slab_values, const double *x,
                    double *y);
/* the same J.v from the sliced-ELL copy of the slab values (stspmv.cu): size per slab
   (-1 on error), relayout once per assembly, apply */
int64_t stmhd_jac_sell_size(stmhd_disc d, void *stream);
int stmhd_jac_relayout(stmhd_disc d, void *stream, const double *slab_values, double *sell);
int stmhd_jac_apply_sell(stmhd_disc d, void *stream, const double *sell, const double *x, double *y);

/* ---- K3-K6: preconditioner (precond.py:67-301) ----
   variant: 0 TRIANGULAR, 1 SIMPLIFIED, 2 FULL (precond.py:40-43).
   The handle keeps `slab_values`/`fp_values` pointers (caller keeps them alive). */
int stmhd_pc_create(stmhd_disc d, void *stream, const double *slab_values,
                    const double *fp_values, const double *alfven, int variant, stmhd_pc *out);
int stmhd_pc_destroy(stmhd_pc p);
/* direction 0: x = P^{-1} r (apply_inverse); 1: x = P r (apply_forward);
   2 / 3: the same with the TRIANGULAR operator whatever the handle's variant (the
   single-step preconditioner, precond.py:344-387, is always triangular) */
int stmhd_pc_apply(stmhd_pc p, void *stream, int direction, const double *r, double *x);
/* sub-operators on (nt x n_field) slab-major blocks:
   0 solve_velocity  1 apply_velocity  2 solve_wave   3 apply_wave   4 apply_potential
   5 solve_potential 6 pressure_schur_inverse 7 pressure_schur_apply
   8 magnetic_schur_inverse 9 magnetic_schur_apply 10 apply_pressure_cd 11 solve_pressure_cd */
int stmhd_pc_op(stmhd_pc p, void *stream, int op, const double *in, double *out);
/* export per-slab matrix values for inspection: what 0 = C_A values (nt x nnz_ca),
   1 = sub1 values ((nt-1) x nnz_s1), 2 = sub2 values (nnz_s2), 3 = the smallest
   restricted-pivoting ratios {F_u, C_A} (2 doubles; |pivot| / max |column entry below the
   diagonal incl. contribution-block rows|, 1 = as good as unrestricted partial pivoting) */
int stmhd_pc_export(stmhd_pc p, void *stream, int what, double *out);

/* ---- K8: fused Gram-Schmidt / FGMRES vector kernels (linalg.py:163-199) ----
   V is row-major (nvec rows of length n, leading dimension ldv). `work` must hold
   stmhd_gs_work_size(n, nvec) doubles. Results land in device memory. */
int64_t stmhd_gs_work_size(int64_t n, int nvec);
/* h[i] = V_i . w, i < nvec */
int stmhd_gs_dots(void *stream, const double *V, int64_t ldv, int nvec, const double *w,
                  int64_t n, double *h, double *work);
/* w -= sum_i h[i] V_i ; then h2[i] = V_i . w (h2 may be NULL) ; nrm2[0] = ||w||^2 (may be NULL) */
int stmhd_gs_update(void *stream, const double *V, int64_t ldv, int nvec, const double *h,
                    double *w, int64_t n, double *h2, double *nrm2, double *work);
/* y = alpha * x  where alpha = scale / sqrt(*nrm2_dev) (scale by a device norm) */
int stmhd_gs_normalize(void *stream, const double *x, double *y, int64_t n,
                       const double *nrm2_dev);
/* x += sum_i c[i] Z_i (c on device) */
int stmhd_gs_combine(void *stream, const double *Z, int64_t ldz, int nvec, const double *c,
                     double *x, int64_t n);
/* out = a*x + b*y ; nrm2 (optional) = ||out||^2 */
int stmhd_axpby(void *stream, double a, const double *x, double b, const double *y, double *out,
                int64_t n, double *nrm2, double *work);

/* ---- generic batched sparse LU (LUFactor, linalg.py:71-96) ----
   Nested-dissection supernodal LU, static symbolic structure shared by a batch of
   matrices with the same pattern; partial pivoting inside supernode diagonal
   blocks.  gx/gy: integer grid coordinates per unknown (NULL -> graph bisection).
   value_map (nnz, may be NULL): index of each pattern entry in the caller's value
   array (per-matrix stride value_stride). */
int stmhd_lu_create(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *gx,
                    const int32_t *gy, int nbatch, int leaf_max, stmhd_lu *out);
int stmhd_lu_destroy(stmhd_lu lu);
int stmhd_lu_factor(stmhd_lu lu, void *stream, const double *values, int64_t value_stride,
                    const int32_t *value_map_host);
/* solve A_b x_b = rhs_b for nrhs right-hand sides; rhs b uses factor
   (nbatch==1 ? 0 : b).  Vectors: rhs[b*ld + i]. */
int stmhd_lu_solve(stmhd_lu lu, void *stream, const double *rhs, int64_t ld_rhs, double *x,
                   int64_t ld_x, int nrhs);
/* sequential sweep over nrhs slabs (factor b for slab b, or 0 if nbatch == 1):
     x_b = A_b^{-1} (rhs_b + c_coef * C x_{b-1})       (C may be NULL: independent solves)
   C in CSR (device arrays).  Reference: solve_potential / solve_velocity,
   precond.py:122-131,173-180; oracle/c5.py C5.solve. */
int stmhd_lu_sweep(stmhd_lu lu, void *stream, const double *rhs, int64_t ld_rhs, double *x,
                   int64_t ld_x, int nrhs, const int32_t *c_rowptr, const int32_t *c_col,
                   const double *c_val, double c_coef);
/* storage diagnostics: [0] factor doubles per matrix, [1] supernodes, [2] levels,
   [3] max front, [4] symbolic nnz(L+U) per matrix */
int stmhd_lu_info(stmhd_lu lu, int64_t *info5);
/* host-only symbolic analysis statistics (no device needed): [0] factor doubles,
   [1] supernodes, [2] levels, [3] max front, [4] symbolic nnz(L+U), [5] front
   workspace doubles, [6] CB-vector doubles, [7] forward work items */
int stmhd_nd_plan_info(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *gx,
                       const int32_t *gy, int leaf_max, int64_t *info8);

/* ---- state-independent operators on the device (constops.cu) ----
   CSR of sum_e P_r(e)^T local[e & 1] P_c(e) on the uniform right-triangulated mesh:
   the reference's assemble_mass / assemble_stiffness / assemble_divergence
   (fem.py:211-271) as used by Discretization (problems.py:185-204).  Row space with nr
   and column space with nc nodes per element; (ne_ptr, ne_code) lists the elements of
   each row node (code = element * 16 + local row, ascending), elem_c the column nodes
   per element, local the two orientation matrices [2][nr][nc].  All pointers are HOST
   arrays (one-time setup): rowptr (n_rows + 1), col / val (capacity entries) and *nnz
   are written; columns sorted, structural zeros kept, contributions summed in
   ascending element order.  Synchronises. */
int stmhd_const_assemble(void *stream, int64_t n_rows, int nr, int nc, int64_t ne,
                         const int32_t *ne_ptr, const int32_t *ne_code, const int32_t *elem_c,
                         const double *local, int32_t *rowptr, int32_t *col, double *val,
                         int64_t capacity, int64_t *nnz);

/* ---- configuration-5 scalar advection-diffusion block (oracle/c5.py) ----
   values[k*nnz + e] = base[e] + sum over the entry's element contributions cinfo
   ({element, local row i, local col j, orientation o}, ranges cptr) of
   sum_c grad12[o][j][c] * sum_m mloc9[i][m] * u[k][node_m][c]
   (the P1 advection term int psi_i (u_k . grad psi_j), reference fem.py:430-462 with a
   P1 vector velocity).  Device arrays except mloc9 / grad12 (host, 9 / 12 doubles). */
int stmhd_c5_values(void *stream, int64_t nnz, int nt, const double *base, const int32_t *cptr,
                    const int32_t *cinfo, const int32_t *elem, const double *u, int64_t n_nodes,
                    const double *mloc9, const double *grad12, double *values);
/* configuration-5 advection fields on the device: u[k][node][2] for k < nt from the
   per-slab modes (host, nt x 8 x {kx, ky, amplitude}, drawn as c5.c5_velocity_fields
   draws them) at the node coordinates xy (device, n_nodes x 2), rescaled to
   max |u_k| = 1; the host generator's sums in the same order.  Synchronises. */
int stmhd_c5_velocity(void *stream, int64_t n_nodes, int nt, const double *xy, const double *modes_host,
                      double *u);
/* block-bidiagonal batched SpMV: y_k = F_k x_k + c_coef * C x_{k-1} (F per slab with
   value stride val_stride, C shared, may be NULL).  oracle/c5.py C5.apply;
   the space-time Jacobian's structure (spacetime.py:131-153). */
int stmhd_bidiag_spmv(void *stream, int64_t n, int nt, const int32_t *rowptr, const int32_t *col,
                      const double *vals, int64_t val_stride, const int32_t *c_rowptr,
                      const int32_t *c_col, const double *c_val, double c_coef, const double *x,
                      double *y);

/* ---- sliced-ELL space-time SpMV plan (stspmv.cu) ----
   y_k = alpha * A_k x_k + c_coef * C x_{k + rel}  for k in [0, nt), x and y with slab
   stride n.  A: per-slab values (stride val_stride) on the CSR pattern (rowptr, col);
   C: shared values on (c_rowptr, c_col) (may be NULL), its columns shifted by
   c_col_shift into slab-relative form (-n: C couples slab k-1; negative relative
   columns are skipped at k = 0).  The space-time Jacobian (spacetime.py:131-153) and
   configuration 5's F_k / -C bidiagonal (oracle/c5.py C5.apply).  Index arrays and
   c_val are HOST memory (copied); values and vectors device memory. */
typedef struct stmhd_spmv_s *stmhd_spmv;
int stmhd_spmv_create(int64_t n, const int32_t *rowptr, const int32_t *col, const int32_t *c_rowptr,
                      const int32_t *c_col, const double *c_val, int32_t c_col_shift, void *stream,
                      stmhd_spmv *out);
int stmhd_spmv_destroy(stmhd_spmv plan);
/* per-slab length of the sliced-ELL value array (rows sorted by length in windows of
   128 and cut into slices of 32, entries column-major per slice, padded) */
int64_t stmhd_spmv_sell_size(stmhd_spmv plan);
/* sell[k*sell_size + e] <- vals[k*val_stride + csr index of e] for k < nt (once per assembly) */
int stmhd_spmv_relayout(stmhd_spmv plan, void *stream, int nt, const double *vals, int64_t val_stride,
                        double *sell);
int stmhd_spmv_apply(stmhd_spmv plan, void *stream, int nt, const double *sell, double alpha, double c_coef,
                     const double *x, double *y);

#ifdef __cplusplus
}
#endif
#endif
