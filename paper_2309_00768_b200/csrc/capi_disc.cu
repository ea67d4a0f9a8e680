// extern "C" entry points: discretisation handle, assembly, Jacobian matvec,
// preconditioner and Krylov kernels (see include/stmhd_b200.h).
#include <cstring>

#include "capi_common.hpp"

#include "pc.hpp"

using namespace stmhd;


int64_t stmhd_disc_s::I(const char *k) const {
  auto it = ints.find(k);
  if (it == ints.end()) throw Error(STMHD_MISSING, std::string("missing int parameter '") + k + "'");
  return it->second;
}
double stmhd_disc_s::R(const char *k) const {
  auto it = reals.find(k);
  if (it == reals.end()) throw Error(STMHD_MISSING, std::string("missing real parameter '") + k + "'");
  return it->second;
}
const HostArray &stmhd_disc_s::H(const char *k) const {
  auto it = host.find(k);
  if (it == host.end()) throw Error(STMHD_MISSING, std::string("missing host array '") + k + "'");
  return it->second;
}
DCsr stmhd_disc_s::csr(const char *prefix) const {
  std::string p(prefix);
  DCsr c;
  c.rowptr = D<int>((p + "_rowptr").c_str());
  c.col = D<int>((p + "_col").c_str());
  c.val = D<double>((p + "_val").c_str());
  c.nrows = (int)(H((p + "_rowptr").c_str()).count - 1);
  return c;
}

static std::unique_ptr<NDPlan> make_plan(stmhd_disc_s *d, const std::string &pat, const char *gx, const char *gy,
                                         const char *map, int leaf, unsigned merge_mask = 0) {
  const HostArray &rp = d->H((pat + "_rowptr").c_str());
  const HostArray &ci = d->H((pat + "_col").c_str());
  const int32_t *vmap = map ? d->H(map).as<int32_t>() : nullptr;
  auto p = std::make_unique<NDPlan>(nd_analyze(rp.count - 1, rp.as<int32_t>(), ci.as<int32_t>(),
                                               d->H(gx).as<int32_t>(), d->H(gy).as<int32_t>(), leaf, vmap, merge_mask));
  return p;
}

extern "C" {

int stmhd_disc_create(stmhd_disc *out) {
  CAPI_BEGIN
  require(out, "stmhd_disc_create: null output");
  *out = new stmhd_disc_s();
  CAPI_END
}

stmhd_disc_s::~stmhd_disc_s() {
  // release every member first (pooled frees may be queued on the side stream), then
  // the stream and events; errors are ignored in a destructor
  if (side) cudaStreamSynchronize(side);
  jv_plan.reset();
  lu_mj.reset();
  lu_ma.reset();
  lu_mp.reset();
  lu_kp.reset();
  dev_fu.reset();
  dev_ca.reset();
  dev_fa.reset();
  dev_fp.reset();
  dev_mj.reset();
  dev_ma.reset();
  dev_mp.reset();
  dev_kp.reset();
  clamped = stmhd::DevBuf();
  dev.clear();
  if (side) {
    cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
  }
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
}

int stmhd_disc_destroy(stmhd_disc d) {
  CAPI_BEGIN
  delete d;
  CAPI_END
}

int stmhd_disc_set_int(stmhd_disc d, const char *key, int64_t v) {
  CAPI_BEGIN
  require(d && key, "stmhd_disc_set_int: bad arguments");
  d->ints[key] = v;
  CAPI_END
}

int stmhd_disc_set_real(stmhd_disc d, const char *key, double v) {
  CAPI_BEGIN
  require(d && key, "stmhd_disc_set_real: bad arguments");
  d->reals[key] = v;
  CAPI_END
}

int stmhd_disc_upload(stmhd_disc d, const char *key, const void *host, int64_t count, int elem) {
  CAPI_BEGIN
  require(d && key && (host || count == 0) && (elem == 4 || elem == 8), "stmhd_disc_upload: bad arguments");
  HostArray &h = d->host[key];
  h.elem = elem;
  h.count = count;
  h.data.assign((const char *)host, (const char *)host + count * elem);
  DevBuf &b = d->dev[key];
  b.alloc(std::max<int64_t>(count * elem, 8));
  if (count) STMHD_CUDA_CHECK(cudaMemcpy(b.ptr, host, count * elem, cudaMemcpyHostToDevice));
  CAPI_END
}

int stmhd_disc_finalize(stmhd_disc d, void *stream) {
  CAPI_BEGIN
  require(d, "stmhd_disc_finalize: null handle");
  cudaStream_t s = (cudaStream_t)stream;
  for (const char *k : {"nt", "n_u", "n_p", "n_j", "n_a", "nv", "npl", "ne", "nnv", "nnp", "nn1", "nnz_js", "nnz_fp"})
    (void)d->I(k);
  int lf = (int)d->I("leaf_fu"), lc = (int)d->I("leaf_ca"), lk = (int)d->I("leaf_c");
  // velocity block of the grid-family sweeps (n_u >= 8000: 32^2 P2 meshes and larger): the
  // separators at tree depths 4, 6 and 8 absorb their children (nd_analyze) -- one
  // grid-wide band level fewer per sweep direction between the 64 CTA-local subtrees and
  // the dense top, and three instead of five CTA-local levels inside a subtree (C4_512
  // P_T^-1 33.8 -> 30.5 ms for +14 % factor bytes; STMHD_ND_MERGE_MASK: bit d = depth d, 0 off)
  unsigned merge_mask = d->I("n_u") >= 8000 ? (1u << 4 | 1u << 6 | 1u << 8) : 0u;
  if (const char *e = getenv("STMHD_ND_MERGE_MASK")) merge_mask = (unsigned)atoi(e);
  d->plan_fu = make_plan(d, "fu", "fu_gx", "fu_gy", "fu_map", lf, merge_mask);
  d->plan_fa = make_plan(d, "fa", "p1_gx", "p1_gy", "fa_map", lc);
  d->plan_ca = make_plan(d, "ca", "p1_gx", "p1_gy", nullptr, lc);
  d->plan_fp = make_plan(d, "fp", "prs_gx", "prs_gy", nullptr, lc);
  d->plan_mj = make_plan(d, "lu_mj", "p1_gx", "p1_gy", nullptr, lk);
  d->plan_ma = make_plan(d, "lu_ma", "p1_gx", "p1_gy", nullptr, lk);
  d->plan_mp = make_plan(d, "lu_mp", "prs_gx", "prs_gy", nullptr, lk);
  d->plan_kp = make_plan(d, "lu_kp", "prs_gx", "prs_gy", nullptr, lk);
  auto mk = [&](std::unique_ptr<NDPlan> &p) {
    auto dv = std::make_unique<NDDevice>();
    dv->build(*p, s);
    return dv;
  };
  d->dev_fu = mk(d->plan_fu);
  d->dev_fa = mk(d->plan_fa);
  d->dev_ca = mk(d->plan_ca);
  d->dev_fp = mk(d->plan_fp);
  d->dev_mj = mk(d->plan_mj);
  d->dev_ma = mk(d->plan_ma);
  d->dev_mp = mk(d->plan_mp);
  d->dev_kp = mk(d->plan_kp);
  struct C {
    std::unique_ptr<NDFactor> *f;
    NDDevice *dv;
    const char *key;
    const char *block;
  } cs[] = {{&d->lu_mj, d->dev_mj.get(), "lu_mj_val", "M_j"},
            {&d->lu_ma, d->dev_ma.get(), "lu_ma_val", "M_A"},
            {&d->lu_mp, d->dev_mp.get(), "lu_mp_val", "M_p"},
            {&d->lu_kp, d->dev_kp.get(), "lu_kp_val", "K_p"}};
  for (auto &c : cs) {
    *c.f = std::make_unique<NDFactor>();
    (*c.f)->dev = c.dv;
    (*c.f)->nbatch = 1;
    (*c.f)->dense_ok = true;  // constant, well-conditioned (mass / pinned Laplacian): dense inverse allowed
    (*c.f)->factor(d->D<double>(c.key), 0, s);
    if ((*c.f)->check_status(s)) throw Error(STMHD_SINGULAR, std::string("constant factor ") + c.block + " is singular");
  }
  d->finalized = true;
  CAPI_END
}

int64_t stmhd_disc_device_bytes(stmhd_disc d) {
  if (!d) return 0;
  int64_t b = 0;
  for (auto &kv : d->dev) b += kv.second.bytes;
  for (auto *f : {d->lu_mj.get(), d->lu_ma.get(), d->lu_mp.get(), d->lu_kp.get()})
    if (f) b += f->factors.bytes;
  return b + d->clamped.bytes;
}

int stmhd_assemble(stmhd_disc d, void *stream, const double *state, const double *ic_u, const double *ic_a,
                   double *residual, double *js, double *fp, double *alf) {
  CAPI_BEGIN
  require(d && d->finalized, "stmhd_assemble: handle not finalized");
  assemble(d, (cudaStream_t)stream, state, ic_u, ic_a, residual, js, fp, alf);
  CAPI_END
}

int stmhd_jac_apply(stmhd_disc d, void *stream, const double *js, const double *x, double *y) {
  CAPI_BEGIN
  require(d && d->finalized && js && x && y, "stmhd_jac_apply: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slab = d->slab();
  const int nt = (int)d->I("nt");
  SpmvArgs a;
  a.nrows = (int)slab;
  a.nslab = nt;
  a.y = y;
  a.y_stride = slab;
  SpTerm t0;
  t0.beg = d->D<int>("js_rowptr");
  t0.col = d->D<int>("js_col");
  t0.val = js;
  t0.val_stride = d->I("nnz_js");
  t0.x = x;
  t0.x_stride = slab;
  SpTerm t1;
  t1.beg = d->D<int>("jc_rowptr");
  t1.col = d->D<int>("jc_col");
  t1.val = d->D<double>("jc_val");
  t1.x = x;
  t1.x_stride = slab;
  t1.rel = 1;
  a.t[0] = t0;
  a.t[1] = t1;
  a.nterms = 2;
  spmv(a, s, 8);
  // pressure mean-constraint row (spacetime.py:140-141)
  const int o_p = (int)d->I("n_u"), pin = (int)d->I("p_pin");
  dense_row(d->D<double>("p_mean_row"), (int)d->I("n_p"), x + o_p, slab, y + o_p + pin, slab, nt, 1.0, s);
  CAPI_END
}

// J.v in the sliced-ELL layout (stspmv.cu): per-slab merged rows [f_u|z_j|z_a ; y|f_a]
// + the shared couplings (B^T, B, M_j, K_jA, -M/dt with slab-relative columns reaching
// into slab k-1); plan built once from the host patterns.
static const StSpmvPlan &jv_plan(stmhd_disc d, cudaStream_t s) {
  if (!d->jv_plan) {
    auto p = std::make_unique<StSpmvPlan>();
    p->build((int)d->slab(), d->H("js_rowptr").as<int>(), d->H("js_col").as<int>(), d->H("jc_rowptr").as<int>(),
             d->H("jc_col").as<int>(), d->H("jc_val").as<double>(), 0, s);
    d->jv_plan = std::move(p);
  }
  return *d->jv_plan;
}

int64_t stmhd_jac_sell_size(stmhd_disc d, void *stream) {
  try {
    if (!d || !d->finalized) return -1;
    return jv_plan(d, (cudaStream_t)stream).sell_a;
  } catch (const Error &e) {
    set_last_error(e.what(), e.block);
    return -1;
  }
}

int stmhd_jac_relayout(stmhd_disc d, void *stream, const double *js, double *sell) {
  CAPI_BEGIN
  require(d && d->finalized && js && sell, "stmhd_jac_relayout: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  jv_plan(d, s).relayout((int)d->I("nt"), js, d->I("nnz_js"), sell, s);
  CAPI_END
}

int stmhd_jac_apply_sell(stmhd_disc d, void *stream, const double *sell, const double *x, double *y) {
  CAPI_BEGIN
  require(d && d->finalized && sell && x && y, "stmhd_jac_apply_sell: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slab = d->slab();
  jv_plan(d, s).apply((int)d->I("nt"), sell, 1.0, 1.0, x, slab, y, slab, s);
  const int o_p = (int)d->I("n_u"), pin = (int)d->I("p_pin");
  dense_row(d->D<double>("p_mean_row"), (int)d->I("n_p"), x + o_p, slab, y + o_p + pin, slab, (int)d->I("nt"), 1.0, s);
  CAPI_END
}

int stmhd_pc_create(stmhd_disc d, void *stream, const double *js, const double *fp, const double *alf, int variant,
                    stmhd_pc *out) {
  CAPI_BEGIN
  require(d && d->finalized && js && fp && alf && out, "stmhd_pc_create: bad arguments");
  require(variant >= 0 && variant <= 2, "stmhd_pc_create: variant must be 0, 1 or 2");
  auto h = std::make_unique<stmhd_pc_s>();
  h->pc = std::make_unique<PC>(d, (cudaStream_t)stream, js, fp, alf, variant);
  *out = h.release();
  CAPI_END
}

int stmhd_pc_destroy(stmhd_pc p) {
  CAPI_BEGIN
  delete p;
  CAPI_END
}

int stmhd_pc_apply(stmhd_pc p, void *stream, int direction, const double *r, double *x) {
  CAPI_BEGIN
  require(p && r && x, "stmhd_pc_apply: bad arguments");
  require(direction >= 0 && direction <= 3, "stmhd_pc_apply: direction must be 0..3");
  // directions 2/3: the TRIANGULAR operator whatever the handle's variant -- the
  // single-step preconditioner is always the triangular one (precond.py:344-387)
  PC &pc = *p->pc;
  const int saved = pc.variant;
  if (direction >= 2) pc.variant = 0;
  struct Restore {
    PC &pc;
    int v;
    ~Restore() { pc.variant = v; }
  } restore{pc, saved};
  if ((direction & 1) == 0)
    pc.apply_inverse(r, x, (cudaStream_t)stream);
  else
    pc.apply_forward(r, x, (cudaStream_t)stream);
  CAPI_END
}

int stmhd_pc_op(stmhd_pc p, void *stream, int op, const double *in, double *out) {
  CAPI_BEGIN
  require(p && in && out, "stmhd_pc_op: bad arguments");
  p->pc->op(op, in, out, (cudaStream_t)stream);
  CAPI_END
}

int stmhd_pc_export(stmhd_pc p, void *stream, int what, double *out) {
  CAPI_BEGIN
  require(p && out, "stmhd_pc_export: bad arguments");
  PC &c = *p->pc;
  const DevBuf *b = what == 0 ? &c.ca_vals : what == 1 ? &c.s1_vals : nullptr;
  if (what == 3) {  // smallest restricted-pivoting ratios of the F_u and C~_A factorisations
    const double h[2] = {c.fu->min_pivot_ratio, c.ca->min_pivot_ratio};
    STMHD_CUDA_CHECK(cudaMemcpyAsync(out, h, sizeof(h), cudaMemcpyHostToDevice, (cudaStream_t)stream));
    STMHD_CUDA_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  } else if (what == 2) {
    DCsr s2 = c.d->csr("sub2");
    int64_t n = c.d->H("sub2_val").count;
    STMHD_CUDA_CHECK(cudaMemcpyAsync(out, s2.val, n * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  } else {
    require(b != nullptr, "stmhd_pc_export: unknown item");
    int64_t n = what == 0 ? (int64_t)c.nt * c.nnz_ca : (int64_t)(c.nt - 1) * c.nnz_s1;
    if (n > 0) STMHD_CUDA_CHECK(cudaMemcpyAsync(out, b->ptr, n * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  CAPI_END
}

int64_t stmhd_gs_work_size(int64_t n, int nvec) { return gs_work_size(n, nvec); }

int stmhd_gs_dots(void *stream, const double *V, int64_t ldv, int nvec, const double *w, int64_t n, double *h,
                  double *work) {
  CAPI_BEGIN
  gs_dots((cudaStream_t)stream, V, ldv, nvec, w, n, h, work);
  CAPI_END
}

int stmhd_gs_update(void *stream, const double *V, int64_t ldv, int nvec, const double *h, double *w, int64_t n,
                    double *h2, double *nrm2, double *work) {
  CAPI_BEGIN
  gs_update((cudaStream_t)stream, V, ldv, nvec, h, w, n, h2, nrm2, work);
  CAPI_END
}

int stmhd_gs_normalize(void *stream, const double *x, double *y, int64_t n, const double *nrm2) {
  CAPI_BEGIN
  gs_normalize((cudaStream_t)stream, x, y, n, nrm2);
  CAPI_END
}

int stmhd_gs_combine(void *stream, const double *Z, int64_t ldz, int nvec, const double *c, double *x, int64_t n) {
  CAPI_BEGIN
  gs_combine((cudaStream_t)stream, Z, ldz, nvec, c, x, n);
  CAPI_END
}

int stmhd_axpby(void *stream, double a, const double *x, double b, const double *y, double *out, int64_t n,
                double *nrm2, double *work) {
  CAPI_BEGIN
  axpby((cudaStream_t)stream, a, x, b, y, out, n, nrm2, work);
  CAPI_END
}

}  // extern "C"
