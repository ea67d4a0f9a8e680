// K1: space-time residual and Jacobian-value assembly on the device.
//
// Reference: residual (spacetime.py:65-85, _slab_galerkin :42-62),
// linearize_slab (spacetime.py:99-112), the state-dependent blocks of
// fem.py:341-472, F_p (precond.py:80-84) and the Alfven scaling
// (precond.py:46-57).  Every value is a contraction of the element state with
// exact per-orientation tensors (see fem.py in this package); rows and CSR
// entries gather their element contributions in a fixed order, so the
// assembly is deterministic (no atomics).
#include <cstdlib>
#include <cstring>

#include "disc.hpp"

namespace stmhd {

struct TOff {
  int MV, KV, TV, MX, G1, M1, K1, MP, KP, TP, BD, total;
};

__host__ __device__ constexpr TOff toff(int NV, int NP) {
  TOff o{};
  o.MV = 0;
  o.KV = o.MV + NV * NV;
  o.TV = o.KV + 2 * NV * NV;
  o.MX = o.TV + 2 * NV * NV * NV * 2;
  o.G1 = o.MX + NV * 3;
  o.M1 = o.G1 + 12;
  o.K1 = o.M1 + 9;
  o.MP = o.K1 + 18;
  o.KP = o.MP + NP * NP;
  o.TP = o.KP + 2 * NP * NP;
  o.BD = o.TP + 2 * NP * NV * NP * 2;
  o.total = o.BD + 2 * NP * NV * 2;
  return o;
}

struct AsmArgs {
  int nt, n_u, n_p, n_j, n_a, nnv, nn1, ne, p_pin;
  int64_t slab;
  double dt, mu, eta, mu0;
  const double *tensors;
  const int *elem_v, *elem_p, *elem_1;
  const int *ne_v_ptr, *ne_v, *ne_p_ptr, *ne_p, *ne_1_ptr, *ne_1;
  const int *u_bc_mask, *a_bc_mask;
  const double *u_bc_val, *a_bc_val, *flux, *e_load;
  const double *state, *ic_u, *ic_a;
  const double *sc;  // clamped state
  double *res;
};

__global__ void clamp_kernel(AsmArgs a, double *out) {
  const int64_t N = (int64_t)a.nt * a.slab;
  const int o_a = a.n_u + a.n_p + a.n_j;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t % a.slab);
    double v = a.state[t];
    if (i < a.n_u) {
      if (a.u_bc_mask[i]) v = a.u_bc_val[i];
    } else if (i >= o_a) {
      if (a.a_bc_mask[i - o_a]) v = a.a_bc_val[i - o_a];
    }
    out[t] = v;
  }
}

template <int NV, int NP>
__device__ __forceinline__ void load_u(const AsmArgs &a, const double *s, int e, double (&u)[2][NV]) {
#pragma unroll
  for (int m = 0; m < NV; ++m) {
    int g = a.elem_v[e * NV + m];
    u[0][m] = s[g];
    u[1][m] = s[a.nnv + g];
  }
}

template <int NV, int NP>
__global__ void __launch_bounds__(256) residual_kernel(AsmArgs a) {
  extern __shared__ double T[];
  constexpr TOff O = toff(NV, NP);
  for (int t = threadIdx.x; t < O.total; t += blockDim.x) T[t] = a.tensors[t];
  __syncthreads();
  const int k = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.slab) return;
  const int o_p = a.n_u, o_j = a.n_u + a.n_p, o_a = o_j + a.n_j;
  const double *s = a.sc + (int64_t)k * a.slab;
  const double *raw = a.state + (int64_t)k * a.slab;
  // previous slab: clamped k-1, or the raw initial condition for k = 0
  const double *pu = k ? a.sc + (int64_t)(k - 1) * a.slab : a.ic_u;
  const double *pa = k ? a.sc + (int64_t)(k - 1) * a.slab + o_a : a.ic_a;
  const double idt = 1.0 / a.dt;
  double out = 0.0;
  if (r < a.n_u) {
    if (a.u_bc_mask[r]) {
      out = raw[r] - a.u_bc_val[r];
    } else {
      const int d = r / a.nnv, node = r % a.nnv;
      double mass = 0.0, visc = 0.0, pres = 0.0, adv = 0.0, lor = 0.0;
      for (int q = a.ne_v_ptr[node]; q < a.ne_v_ptr[node + 1]; ++q) {
        const int code = a.ne_v[q], e = code >> 4, il = code & 15, o = e & 1;
        double u[2][NV], up[2][NV];
        load_u<NV, NP>(a, s, e, u);
        load_u<NV, NP>(a, pu, e, up);
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          mass += T[O.MV + il * NV + j] * (u[d][j] - up[d][j]);
          visc += T[O.KV + (o * NV + il) * NV + j] * u[d][j];
        }
#pragma unroll
        for (int n = 0; n < NP; ++n)
          pres += T[O.BD + ((o * NP + n) * NV + il) * 2 + d] * s[o_p + a.elem_p[e * NP + n]];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            double acc = 0.0;
#pragma unroll
            for (int n = 0; n < NV; ++n) acc += T[O.TV + (((o * NV + il) * NV + m) * NV + n) * 2 + c] * u[d][n];
            adv += u[c][m] * acc;
          }
        double ga = 0.0, jm = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          int g = a.elem_1[e * 3 + n];
          ga += s[o_a + g] * T[O.G1 + (o * 3 + n) * 2 + d];
          jm += s[o_j + g] * T[O.MX + il * 3 + n];
        }
        lor += ga * jm;
      }
      out = mass * idt + a.mu * visc + pres + adv + lor;
    }
  } else if (r < o_j) {
    const int m = r - o_p;
    if (m == a.p_pin) return;  // mean-constraint row: pin_row_kernel
    double acc = 0.0;
    for (int q = a.ne_p_ptr[m]; q < a.ne_p_ptr[m + 1]; ++q) {
      const int code = a.ne_p[q], e = code >> 4, ml = code & 15, o = e & 1;
      double u[2][NV];
      load_u<NV, NP>(a, s, e, u);
#pragma unroll
      for (int n = 0; n < NV; ++n)
#pragma unroll
        for (int c = 0; c < 2; ++c) acc += T[O.BD + ((o * NP + ml) * NV + n) * 2 + c] * u[c][n];
    }
    out = acc;
  } else if (r < o_a) {
    const int m = r - o_j;
    double mj = 0.0, kj = 0.0;
    for (int q = a.ne_1_ptr[m]; q < a.ne_1_ptr[m + 1]; ++q) {
      const int code = a.ne_1[q], e = code >> 4, ml = code & 15, o = e & 1;
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        int g = a.elem_1[e * 3 + n];
        mj += T[O.M1 + ml * 3 + n] * s[o_j + g];
        kj += T[O.K1 + (o * 3 + ml) * 3 + n] * s[o_a + g];
      }
    }
    out = mj + kj / a.mu0 - a.flux[m];
  } else {
    const int m = r - o_a;
    if (a.a_bc_mask[m]) {
      out = raw[r] - a.a_bc_val[m];
    } else {
      double mass = 0.0, diff = 0.0, adv = 0.0;
      for (int q = a.ne_1_ptr[m]; q < a.ne_1_ptr[m + 1]; ++q) {
        const int code = a.ne_1[q], e = code >> 4, ml = code & 15, o = e & 1;
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          int g = a.elem_1[e * 3 + n];
          double av = s[o_a + g];
          mass += T[O.M1 + ml * 3 + n] * (av - pa[g]);
          diff += T[O.K1 + (o * 3 + ml) * 3 + n] * av;
          gx += av * T[O.G1 + (o * 3 + n) * 2 + 0];
          gy += av * T[O.G1 + (o * 3 + n) * 2 + 1];
        }
        double u[2][NV];
        load_u<NV, NP>(a, s, e, u);
        double mx = 0.0, my = 0.0;
#pragma unroll
        for (int n = 0; n < NV; ++n) {
          mx += T[O.MX + n * 3 + ml] * u[0][n];
          my += T[O.MX + n * 3 + ml] * u[1][n];
        }
        adv += gx * mx + gy * my;
      }
      out = mass * idt + (a.eta / a.mu0) * diff + adv + a.e_load[m];
    }
  }
  a.res[(int64_t)k * a.slab + r] = out;
}

// r_p[pin] = w . p_raw - target  (spacetime.py:78), one block per slab
__global__ void pin_row_kernel(const double *state, const double *w, int n_p, int64_t slab, int o_p,
                               int pin, double target, double *res) {
  __shared__ double sh[32];
  const int k = blockIdx.x;
  const double *p = state + (int64_t)k * slab + o_p;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n_p; i += blockDim.x) acc += w[i] * p[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) res[(int64_t)k * slab + o_p + pin] = acc - target;
}

// s_k = |mean grad A_k|^2 / mu0 on the clamped potential (precond.py:46-57)
__global__ void alfven_kernel(AsmArgs a, const double *g1, double elem_area, double area, double *out) {
  extern __shared__ double T[];
  __shared__ double sh[32];
  constexpr int G1off = 0;
  for (int t = threadIdx.x; t < 12; t += blockDim.x) T[t] = g1[t];
  __syncthreads();
  const int k = blockIdx.x;
  const int o_a = a.n_u + a.n_p + a.n_j;
  const double *s = a.sc + (int64_t)k * a.slab + o_a;
  double gx = 0.0, gy = 0.0;
  for (int e = threadIdx.x; e < a.ne; e += blockDim.x) {
    int o = e & 1;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      double av = s[a.elem_1[e * 3 + n]];
      gx += av * T[G1off + (o * 3 + n) * 2 + 0];
      gy += av * T[G1off + (o * 3 + n) * 2 + 1];
    }
  }
  gx = block_sum(gx, sh) * elem_area / area;
  gy = block_sum(gy, sh) * elem_area / area;
  if (threadIdx.x == 0) out[k] = (gx * gx + gy * gy) / a.mu0;
}

struct ValArgs {
  int nnz, nt;
  const int *kind, *cptr, *contrib;
  int64_t out_stride;
  double *out;
  int is_fp;
};

// Per-slab Jacobian values in the fixed merged pattern (linearize_slab) or F_p.
template <int NV, int NP>
__global__ void __launch_bounds__(256) values_kernel(AsmArgs a, ValArgs v) {
  extern __shared__ double T[];
  constexpr TOff O = toff(NV, NP);
  for (int t = threadIdx.x; t < O.total; t += blockDim.x) T[t] = a.tensors[t];
  __syncthreads();
  const int ent = blockIdx.x * blockDim.x + threadIdx.x;
  if (ent >= v.nnz) return;
  const int kind = v.is_fp ? 6 : v.kind[ent];
  const int kd = kind & 15, d = (kind >> 4) & 1, c = (kind >> 5) & 1;
  const int q0 = v.cptr[ent], q1 = v.cptr[ent + 1];
  const int o_j = a.n_u + a.n_p, o_a = o_j + a.n_j, o_p = a.n_u;
  const double idt = 1.0 / a.dt;
  const double ceta = a.eta / a.mu0;
  (void)o_p;
  for (int k = blockIdx.y; k < a.nt; k += gridDim.y) {
    const double *s = a.sc + (int64_t)k * a.slab;
    double val = 0.0;
    if (kd == 0) {
      val = 1.0;
    } else {
      for (int q = q0; q < q1; ++q) {
        const int code = v.contrib[q], e = code >> 8, il = (code >> 4) & 15, jl = code & 15, o = e & 1;
        if (kd == 1) {  // f_u (d,c): M/dt + mu K + transport + reaction
          double u[2][NV];
          load_u<NV, NP>(a, s, e, u);
          double t = 0.0;
          if (d == c) {
            double tr = 0.0;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
              for (int m = 0; m < NV; ++m) tr += u[cc][m] * T[O.TV + (((o * NV + il) * NV + m) * NV + jl) * 2 + cc];
            t = T[O.MV + il * NV + jl] * idt + a.mu * T[O.KV + (o * NV + il) * NV + jl] + tr;
          }
          double re = 0.0;
#pragma unroll
          for (int m = 0; m < NV; ++m) re += u[d][m] * T[O.TV + (((o * NV + il) * NV + jl) * NV + m) * 2 + c];
          val += t + re;
        } else if (kd == 2) {  // z_j: (d_d A) int phi_i psi_n
          double ga = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) ga += s[o_a + a.elem_1[e * 3 + n]] * T[O.G1 + (o * 3 + n) * 2 + d];
          val += ga * T[O.MX + il * 3 + jl];
        } else if (kd == 3) {  // z_a: (int j phi_i) d_d psi_n
          double jm = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) jm += s[o_j + a.elem_1[e * 3 + n]] * T[O.MX + il * 3 + n];
          val += jm * T[O.G1 + (o * 3 + jl) * 2 + d];
        } else if (kd == 4) {  // y: (d_c A) int psi_m phi_n
          double ga = 0.0;
#pragma unroll
          for (int n = 0; n < 3; ++n) ga += s[o_a + a.elem_1[e * 3 + n]] * T[O.G1 + (o * 3 + n) * 2 + c];
          val += ga * T[O.MX + jl * 3 + il];
        } else if (kd == 5) {  // f_a: M/dt + (eta/mu0) K + int psi_m u.grad psi_n
          double u[2][NV];
          load_u<NV, NP>(a, s, e, u);
          double mx = 0.0, my = 0.0;
#pragma unroll
          for (int l = 0; l < NV; ++l) {
            mx += u[0][l] * T[O.MX + l * 3 + il];
            my += u[1][l] * T[O.MX + l * 3 + il];
          }
          val += T[O.M1 + il * 3 + jl] * idt + ceta * T[O.K1 + (o * 3 + il) * 3 + jl] +
                 (T[O.G1 + (o * 3 + jl) * 2 + 0] * mx + T[O.G1 + (o * 3 + jl) * 2 + 1] * my);
        } else {  // F_p: M_p/dt + W_p(u) + mu K_p
          double u[2][NV];
          load_u<NV, NP>(a, s, e, u);
          double w = 0.0;
#pragma unroll
          for (int l = 0; l < NV; ++l)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) w += u[cc][l] * T[O.TP + (((o * NP + il) * NV + l) * NP + jl) * 2 + cc];
          val += T[O.MP + il * NP + jl] * idt + w + a.mu * T[O.KP + (o * NP + il) * NP + jl];
        }
      }
    }
    v.out[(int64_t)k * v.out_stride + ent] = val;
  }
}

// ---------------------------------------------------------------------------
// Element-matrix assembly per patch (P2/P1; tables: asm_patches.py).
//
// Per (patch, slab): phase A evaluates the element matrices of every element the
// patch's entries touch into shared memory.  Every entry is affine in the element
// state (u, A, j), so E = W s with per-orientation linear maps built on the host
// (discretisation constants folded in).  A0: one lane per element stages its state
// row (u, 1, grad A, j moments) in shared memory; A1: one thread per output row of
// the maps holds its W row in registers and walks the elements of its orientation
// (state rows are broadcast loads, stores are contiguous): no global loads in the
// FMA loop.  Z_j, Z_A, Y are single products of grad A / the j moments, formed in the
// reference's order (exact cancellations, e.g. d_x A = 0 on a Harris sheet, stay
// exact).  Phase B writes each owned CSR entry of the merged Jacobian pattern and of
// F_p as the sum of its element contributions (16-bit shared-memory offsets).  A CTA
// walks a run of slabs so the W rows are loaded once per run.  Same algebra as
// values_kernel, element-wise instead of entry-wise.
struct PatchArgs {
  int nt, npatch, nnv, kchunk;
  int o_j, o_a;
  int64_t slab;
  const double *sc;  // clamped state
  const int *elem_v, *elem_1;
  const int4 *desc;  // {round offset, rounds, slot offset, n0 | n1 << 16}
  const int *slots, *out;
  const uint4 *codes;  // 8 x uint16 per table entry
  const double *w;     // W1 [o][162][14] (asm_patches.element_linear_maps)
  const double *g1, *mx;  // reference-element G1[o][n][d], MX[il][n]
  int phases;             // bit 0: element matrices, bit 1: entries (diagnostics: STMHD_PATCH_PHASES)
  int pipe;               // double-buffered software pipeline over the slab run
  double *js, *fp;
  int64_t js_stride, fp_stride;
};

constexpr int kPatchESZ = 270, kPatchRound = 256, kPatchMaxC = 6, kPatchThreads = 640;
constexpr int kPatchSSZ = 24;  // state row: u (12), 1, pad, grad A (2), j moments (6), pad (2)
constexpr int kPatchItems = 2 * 162 + 2 * 108;

__global__ void __launch_bounds__(kPatchThreads, 1) values_patch_kernel(const __grid_constant__ PatchArgs P) {
  extern __shared__ __align__(16) double smem_e[];
  const int pt = blockIdx.x;
  const int4 dsc = P.desc[pt];
  const int n0 = dsc.w & 0xffff, n1 = dsc.w >> 16, nsl = n0 + n1;
  // two buffers of element matrices, then two of state rows
  // pipelined: two buffers of element matrices, then two of state rows; sequential:
  // one of each (the buffer pointers alias)
  const int nb = P.pipe ? 2 : 1;
  double *const E0 = smem_e, *const E1 = smem_e + (size_t)(nb - 1) * nsl * kPatchESZ;
  double *const S0 = smem_e + (size_t)nb * nsl * kPatchESZ, *const S1 = S0 + (size_t)(nb - 1) * nsl * kPatchSSZ;
  const int ntab = dsc.y * kPatchRound;
  const int *outp = P.out + (int64_t)dsc.x * kPatchRound;
  const uint4 *codep = P.codes + (int64_t)dsc.x * kPatchRound;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  // FU/FA/FP rows: E_o = S_o W1_o^T on the FP64 tensor cores (mma m8n8k4): 2 x 21
  // n-tiles of 8 output rows over the warps, the B fragments (W1) in registers
  constexpr int kNT = 21, kMaxTW = 3;
  double bf[kMaxTW][4];
#pragma unroll
  for (int i = 0; i < kMaxTW; ++i) {
    const int t = warp + i * nwarps;
    const int o = t / kNT, n = (t % kNT) * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      bf[i][ks] = (t < 2 * kNT && n < 162 && kk < 14) ? P.w[(o * 162 + n) * 14 + kk] : 0.0;
    }
  }
  // Z_j, Z_A, Y rows: one product each (threads 0..215)
  int z_o = -1, z_q = 0, z_src = 0;
  double z_c = 0.0;
  if ((int)threadIdx.x < 216) {
    const int z = threadIdx.x, o = z / 108, v = z % 108, q = v % 36;
    z_o = o;
    z_q = 144 + v;
    if (v < 36) {  // ZJ[d][il][jl] = ga_d MX[il][jl]
      z_src = 14 + q / 18;
      z_c = P.mx[q % 18];
    } else if (v < 72) {  // ZA[d][il][jl] = jm(il) G1[o][jl][d]
      const int d = q / 18, il = (q / 3) % 6, jl = q % 3;
      z_src = 16 + il;
      z_c = P.g1[(o * 3 + jl) * 2 + d];
    } else {  // Y[c][il][jl] = ga_c MX[jl][il]
      const int c = q / 18, il = (q / 6) % 3, jl = q % 6;
      z_src = 14 + c;
      z_c = P.mx[jl * 3 + il];
    }
  }
  // software pipeline over the CTA's slab run, double-buffered state rows S and
  // element matrices E: iteration k writes the entries of slab k (B) from E[k&1] while
  // the tensor cores form E[(k+1)&1] (A1) and A0 stages the state rows of slab k+2;
  // the three are independent, so warps interleave them between two barriers
  const int k0 = blockIdx.y * P.kchunk, k1 = min(P.nt, k0 + P.kchunk);
  auto stage_A0 = [&](int k) {
    if (!(P.phases & 1) || k >= k1) return;
    const double *s = P.sc + (int64_t)k * P.slab;
    double *S = (k & 1) ? S1 : S0;
    for (int sl = threadIdx.x; sl < nsl; sl += blockDim.x) {
      const int e = P.slots[dsc.z + sl], o = e & 1;
      double *row = S + sl * kPatchSSZ;
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        const int g = P.elem_v[e * 6 + m];
        row[m] = s[g];
        row[6 + m] = s[P.nnv + g];
      }
      row[12] = 1.0;
      row[13] = 0.0;
      double av[3], jv[3];
#pragma unroll
      for (int n = 0; n < 3; ++n) {
        const int g = P.elem_1[e * 3 + n];
        av[n] = s[P.o_a + g];
        jv[n] = s[P.o_j + g];
      }
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        double ga = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) ga += av[n] * P.g1[(o * 3 + n) * 2 + d];
        row[14 + d] = ga;
      }
#pragma unroll
      for (int il = 0; il < 6; ++il) {
        double jm = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) jm += jv[n] * P.mx[il * 3 + n];
        row[16 + il] = jm;
      }
    }
  };
  auto stage_A1 = [&](int k) {
    if (!(P.phases & 1) || k >= k1) return;
    const double *S = (k & 1) ? S1 : S0;
    double *E = (k & 1) ? E1 : E0;
    // A1 (tensor cores): per tile, m-tiles of 8 elements x 4 k-steps
#pragma unroll
    for (int i = 0; i < kMaxTW; ++i) {
      const int t = warp + i * nwarps;
      if (t >= 2 * kNT) break;
      const int o = t / kNT, n = (t % kNT) * 8 + (lane & 3) * 2;
      const int no = o ? n1 : n0, sb = o ? n0 : 0;
      for (int m0 = 0; m0 < no; m0 += 8) {
        const int ra = m0 + (lane >> 2);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const double av = ra < no ? S[(sb + ra) * kPatchSSZ + ks * 4 + (lane & 3)] : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(d0), "+d"(d1)
                       : "d"(av), "d"(bf[i][ks]));
        }
        if (ra < no && n < 162) {
          const int q = n < 144 ? n : n + 108;
          *reinterpret_cast<double2 *>(E + (sb + ra) * kPatchESZ + q) = make_double2(d0, d1);
        }
      }
    }
    // A1 (scalar): Z_j, Z_A, Y
    if (z_o >= 0) {
      const int sb = z_o ? n0 : 0, se = z_o ? nsl : n0;
      for (int sl = sb; sl < se; ++sl) E[sl * kPatchESZ + z_q] = S[sl * kPatchSSZ + z_src] * z_c;
    }
  };
  auto stage_B = [&](int k) {
    const double *E = (k & 1) ? E1 : E0;
    // phase B: owned entries; 8 codes per entry in one 16-byte word; 4 entries per
    // thread in flight (table loads are L2 round trips)
    for (int i0 = threadIdx.x; i0 < ((P.phases & 2) ? ntab : 0); i0 += 4 * blockDim.x) {
      int w[4];
      uint4 cw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * blockDim.x;
        w[u] = i < ntab ? __ldg(outp + i) : -1;
        cw[u] = i < ntab ? __ldg(codep + i) : make_uint4(~0u, ~0u, ~0u, ~0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (w[u] < 0) continue;
        double v = 0.0;
        if (w[u] & (1 << 29)) {
          v = 1.0;
        } else {
          const unsigned c[8] = {cw[u].x & 0xffffu, cw[u].x >> 16, cw[u].y & 0xffffu, cw[u].y >> 16,
                                 cw[u].z & 0xffffu, cw[u].z >> 16, cw[u].w & 0xffffu, cw[u].w >> 16};
#pragma unroll
          for (int j = 0; j < kPatchMaxC; ++j)
            if (c[j] != 0xffffu) v += E[c[j]];
        }
        const int idx = w[u] & ((1 << 29) - 1);
        if (w[u] & (1 << 30)) P.fp[(int64_t)k * P.fp_stride + idx] = v;
        else P.js[(int64_t)k * P.js_stride + idx] = v;
      }
    }
  };
  if (P.pipe) {
    stage_A0(k0);
    __syncthreads();
    stage_A1(k0);
    stage_A0(k0 + 1);
    __syncthreads();
    for (int k = k0; k < k1; ++k) {
      stage_B(k);
      stage_A1(k + 1);
      stage_A0(k + 2);
      __syncthreads();
    }
  } else {
    for (int k = k0; k < k1; ++k) {
      stage_A0(k);
      __syncthreads();
      stage_A1(k);
      __syncthreads();
      stage_B(k);
      __syncthreads();
    }
  }
}

static void values_patch(stmhd_disc_s *d, const AsmArgs &a, cudaStream_t s, double *js, double *fp) {
  PatchArgs P{};
  P.nt = a.nt;
  P.npatch = (int)d->I("pa_npatch");
  P.nnv = a.nnv;
  P.o_j = a.n_u + a.n_p;
  P.o_a = P.o_j + a.n_j;
  P.slab = a.slab;
  P.sc = a.sc;
  P.elem_v = a.elem_v;
  P.elem_1 = a.elem_1;
  P.desc = d->D<int4>("pa_desc");
  P.slots = d->D<int>("pa_slots");
  P.out = d->D<int>("pa_out");
  P.codes = d->D<uint4>("pa_codes");
  P.w = d->D<double>("pa_w");
  {
    constexpr TOff O = toff(6, 3);
    P.g1 = d->D<double>("tensors") + O.G1;
    P.mx = d->D<double>("tensors") + O.MX;
  }
  P.js = js;
  P.fp = fp;
  {
    static const int ph = [] {
      const char *e = getenv("STMHD_PATCH_PHASES");
      return e ? atoi(e) : 3;
    }();
    P.phases = ph;
  }
  P.js_stride = d->I("nnz_js");
  P.fp_stride = d->I("nnz_fp");
  // double buffers when they fit (small patches), else the sequential phases; r01
  // measurements at C3: 6x5 sequential 1.65 ms, 4x3 pipelined 2.33 ms
  const size_t one = (size_t)d->I("pa_max_slots") * (kPatchESZ + kPatchSSZ) * sizeof(double);
  static const int pipe_env = [] {
    const char *e = getenv("STMHD_PATCH_PIPE");
    return e ? atoi(e) : 0;
  }();
  P.pipe = (pipe_env && 2 * one <= 225 * 1024) ? 1 : 0;
  const size_t smem = (P.pipe ? 2 : 1) * one;
  static bool attr = false;
  if (!attr) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(values_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          225 * 1024));
    attr = true;
  }
  require(smem <= 225 * 1024, "patch assembly: element matrices exceed shared memory");
  // slab runs per CTA: W rows loaded once per run, >= ~2 waves of one CTA per SM
  P.kchunk = std::max(1, std::min(16, (int)((int64_t)P.npatch * a.nt / (2 * num_sms()))));
  values_patch_kernel<<<dim3(P.npatch, cdiv(a.nt, P.kchunk)), kPatchThreads, smem, s>>>(P);
  STMHD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// Residual per patch (P2/P1; tables: asm_patches.build_residual_plan).  Phase A: the
// element residual vector RU[d][il] | RP | RJ | RA of every element the patch's rows
// touch (reference _slab_galerkin, spacetime.py:42-62, term by term as
// residual_kernel); phase B: each owned row is the sum of its node's element entries
// plus the row constant (-flux, e_load, -bc value; Dirichlet rows add the raw state).
struct ResConst {
  double TV[2][6][6][6][2];
  double MV[6][6], KV[2][6][6];
  double MX[6][3], G1[2][3][2], M1[3][3], K1[2][3][3];
  double BD[2][3][6][2];  // -int q_m d_c phi_n
};

struct ResArgs {
  ResConst c;
  int nt, nnv, o_p, o_j, o_a;
  int64_t slab;
  double idt, mu, ceta, imu0;
  const double *sc, *state, *ic_u, *ic_a, *add;
  const int *elem_v, *elem_p, *elem_1;
  const int4 *desc;
  const int *slots, *out;
  const uint4 *codes;
  double *res;
};

constexpr int kResSZ = 21;

// RU[d][il] for il in [R0, R0+3): mass/dt + mu K + pressure + (u.grad)u + Lorentz
template <int O, int R0>
__device__ __forceinline__ void res_part_u(const ResArgs &P, const double *s, const double *pu, const double *pa,
                                           int e, double *E) {
  const ResConst &C = P.c;
  double u[2][6], up[2][6];
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    const int g = P.elem_v[e * 6 + m];
    u[0][m] = s[g];
    u[1][m] = s[P.nnv + g];
    up[0][m] = pu[g];
    up[1][m] = pu[P.nnv + g];
  }
  double pv[3], av[3], jv[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    pv[n] = s[P.o_p + P.elem_p[e * 3 + n]];
    const int g = P.elem_1[e * 3 + n];
    av[n] = s[P.o_a + g];
    jv[n] = s[P.o_j + g];
  }
  (void)pa;
  double ga[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    ga[d] = 0.0;
#pragma unroll
    for (int n = 0; n < 3; ++n) ga[d] += av[n] * C.G1[O][n][d];
  }
#pragma unroll
  for (int il = R0; il < R0 + 3; ++il) {
    double w[6];
#pragma unroll
    for (int n = 0; n < 6; ++n) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int m = 0; m < 6; ++m) t = fma(u[c][m], C.TV[O][il][m][n][c], t);
      w[n] = t;
    }
    double jm = 0.0;
#pragma unroll
    for (int n = 0; n < 3; ++n) jm += jv[n] * C.MX[il][n];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      double mass = 0.0, visc = 0.0, pres = 0.0, adv = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        mass += C.MV[il][j] * (u[d][j] - up[d][j]);
        visc += C.KV[O][il][j] * u[d][j];
        adv += w[j] * u[d][j];
      }
#pragma unroll
      for (int n = 0; n < 3; ++n) pres += C.BD[O][n][il][d] * pv[n];
      E[d * 6 + il] = mass * P.idt + P.mu * visc + pres + adv + ga[d] * jm;
    }
  }
}

// RP (divergence), RJ (current definition), RA (induction)
template <int O>
__device__ __forceinline__ void res_part_s(const ResArgs &P, const double *s, const double *pa, int e, double *E) {
  const ResConst &C = P.c;
  double u[2][6];
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    const int g = P.elem_v[e * 6 + m];
    u[0][m] = s[g];
    u[1][m] = s[P.nnv + g];
  }
  double av[3], apv[3], jv[3];
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    const int g = P.elem_1[e * 3 + n];
    av[n] = s[P.o_a + g];
    apv[n] = pa[g];
    jv[n] = s[P.o_j + g];
  }
  double gx = 0.0, gy = 0.0;
#pragma unroll
  for (int n = 0; n < 3; ++n) {
    gx += av[n] * C.G1[O][n][0];
    gy += av[n] * C.G1[O][n][1];
  }
#pragma unroll
  for (int ml = 0; ml < 3; ++ml) {
    double rp = 0.0;
#pragma unroll
    for (int n = 0; n < 6; ++n)
#pragma unroll
      for (int c = 0; c < 2; ++c) rp += C.BD[O][ml][n][c] * u[c][n];
    double mj = 0.0, kj = 0.0, mass = 0.0, diff = 0.0;
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      mj += C.M1[ml][n] * jv[n];
      kj += C.K1[O][ml][n] * av[n];
      mass += C.M1[ml][n] * (av[n] - apv[n]);
      diff += C.K1[O][ml][n] * av[n];
    }
    double mx = 0.0, my = 0.0;
#pragma unroll
    for (int n = 0; n < 6; ++n) {
      mx += C.MX[n][ml] * u[0][n];
      my += C.MX[n][ml] * u[1][n];
    }
    E[12 + ml] = rp;
    E[15 + ml] = mj + kj * P.imu0;
    E[18 + ml] = mass * P.idt + P.ceta * diff + (gx * mx + gy * my);
  }
}

template <int O>
__device__ __noinline__ void res_part(const ResArgs &P, int part, const double *s, const double *pu,
                                      const double *pa, int e, double *E) {
  if (part == 0) res_part_u<O, 0>(P, s, pu, pa, e, E);
  else if (part == 1) res_part_u<O, 3>(P, s, pu, pa, e, E);
  else res_part_s<O>(P, s, pa, e, E);
}

__global__ void __launch_bounds__(256) residual_patch_kernel(const __grid_constant__ ResArgs P) {
  extern __shared__ double E[];
  const int pt = blockIdx.x, k = blockIdx.y;
  const int4 dsc = P.desc[pt];
  const int n0 = dsc.w & 0xffff, n1 = dsc.w >> 16;
  const int ch0 = (n0 + 31) / 32, nch = ch0 + (n1 + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double *s = P.sc + (int64_t)k * P.slab;
  const double *pu = k ? P.sc + (int64_t)(k - 1) * P.slab : P.ic_u;
  const double *pa = k ? P.sc + (int64_t)(k - 1) * P.slab + P.o_a : P.ic_a;
  for (int t = warp; t < 3 * nch; t += nwarps) {
    const int part = t % 3, ch = t / 3;
    const int o = ch < ch0 ? 0 : 1;
    const int loc = o == 0 ? ch * 32 + lane : (ch - ch0) * 32 + lane;
    if (loc >= (o == 0 ? n0 : n1)) continue;
    const int sl = o == 0 ? loc : n0 + loc;
    const int e = P.slots[dsc.z + sl];
    if (o == 0) res_part<0>(P, part, s, pu, pa, e, E + sl * kResSZ);
    else res_part<1>(P, part, s, pu, pa, e, E + sl * kResSZ);
  }
  __syncthreads();
  const int ntab = dsc.y * kPatchRound;
  const int *outp = P.out + (int64_t)dsc.x * kPatchRound;
  const uint4 *codep = P.codes + (int64_t)dsc.x * kPatchRound;
  const double *raw = P.state + (int64_t)k * P.slab;
  for (int i0 = threadIdx.x; i0 < ntab; i0 += 4 * blockDim.x) {
    int w[4];
    uint4 cw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      w[u] = i < ntab ? __ldg(outp + i) : -1;
      cw[u] = i < ntab ? __ldg(codep + i) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (w[u] < 0) continue;
      const int r = w[u] & ((1 << 29) - 1);
      double v = P.add[r];
      if (w[u] & (1 << 29)) {
        v = raw[r] + v;
      } else {
        const unsigned c[8] = {cw[u].x & 0xffffu, cw[u].x >> 16, cw[u].y & 0xffffu, cw[u].y >> 16,
                               cw[u].z & 0xffffu, cw[u].z >> 16, cw[u].w & 0xffffu, cw[u].w >> 16};
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < kPatchMaxC; ++j)
          if (c[j] != 0xffffu) acc += E[c[j]];
        v = acc + v;
      }
      P.res[(int64_t)k * P.slab + r] = v;
    }
  }
}

static void residual_patch(stmhd_disc_s *d, const AsmArgs &a, cudaStream_t s) {
  ResArgs P{};
  const HostArray &T = d->H("tensors");
  constexpr TOff O = toff(6, 3);
  require(T.count >= O.total, "patch residual: tensor blob too small");
  const double *t = T.as<double>();
  std::memcpy(P.c.MV, t + O.MV, sizeof(P.c.MV));
  std::memcpy(P.c.KV, t + O.KV, sizeof(P.c.KV));
  std::memcpy(P.c.TV, t + O.TV, sizeof(P.c.TV));
  std::memcpy(P.c.MX, t + O.MX, sizeof(P.c.MX));
  std::memcpy(P.c.G1, t + O.G1, sizeof(P.c.G1));
  std::memcpy(P.c.M1, t + O.M1, sizeof(P.c.M1));
  std::memcpy(P.c.K1, t + O.K1, sizeof(P.c.K1));
  std::memcpy(P.c.BD, t + O.BD, sizeof(P.c.BD));
  P.nt = a.nt;
  P.nnv = a.nnv;
  P.o_p = a.n_u;
  P.o_j = a.n_u + a.n_p;
  P.o_a = P.o_j + a.n_j;
  P.slab = a.slab;
  P.idt = 1.0 / a.dt;
  P.mu = a.mu;
  P.ceta = a.eta / a.mu0;
  P.imu0 = 1.0 / a.mu0;
  P.sc = a.sc;
  P.state = a.state;
  P.ic_u = a.ic_u;
  P.ic_a = a.ic_a;
  P.add = d->D<double>("pr_add");
  P.elem_v = a.elem_v;
  P.elem_p = a.elem_p;
  P.elem_1 = a.elem_1;
  P.desc = d->D<int4>("pr_desc");
  P.slots = d->D<int>("pr_slots");
  P.out = d->D<int>("pr_out");
  P.codes = d->D<uint4>("pr_codes");
  P.res = a.res;
  const size_t smem = (size_t)d->I("pr_max_slots") * kResSZ * sizeof(double);
  static bool attr = false;
  if (!attr) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(residual_patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          110 * 1024));
    attr = true;
  }
  require(smem <= 110 * 1024, "patch residual: element vectors exceed shared memory");
  residual_patch_kernel<<<dim3((unsigned)d->I("pr_npatch"), a.nt), 256, smem, s>>>(P);
  STMHD_LAUNCH_CHECK();
}

static AsmArgs make_args(const stmhd_disc_s *d) {
  AsmArgs a{};
  a.nt = (int)d->I("nt");
  a.n_u = (int)d->I("n_u");
  a.n_p = (int)d->I("n_p");
  a.n_j = (int)d->I("n_j");
  a.n_a = (int)d->I("n_a");
  a.nnv = (int)d->I("nnv");
  a.nn1 = (int)d->I("nn1");
  a.ne = (int)d->I("ne");
  a.p_pin = (int)d->I("p_pin");
  a.slab = d->slab();
  a.dt = d->R("dt");
  a.mu = d->R("mu");
  a.eta = d->R("eta");
  a.mu0 = d->R("mu0");
  a.tensors = d->D<double>("tensors");
  a.elem_v = d->D<int>("elem_v");
  a.elem_p = d->D<int>("elem_p");
  a.elem_1 = d->D<int>("elem_1");
  a.ne_v_ptr = d->D<int>("ne_v_ptr");
  a.ne_v = d->D<int>("ne_v");
  a.ne_p_ptr = d->D<int>("ne_p_ptr");
  a.ne_p = d->D<int>("ne_p");
  a.ne_1_ptr = d->D<int>("ne_1_ptr");
  a.ne_1 = d->D<int>("ne_1");
  a.u_bc_mask = d->D<int>("u_bc_mask");
  a.a_bc_mask = d->D<int>("a_bc_mask");
  a.u_bc_val = d->D<double>("u_bc_val");
  a.a_bc_val = d->D<double>("a_bc_val");
  a.flux = d->D<double>("flux");
  a.e_load = d->D<double>("e_load");
  return a;
}

template <int NV, int NP>
static void assemble_t(stmhd_disc_s *d, cudaStream_t s, const double *state, const double *ic_u,
                       const double *ic_a, double *res, double *js, double *fp, double *alf) {
  AsmArgs a = make_args(d);
  a.state = state;
  a.ic_u = ic_u;
  a.ic_a = ic_a;
  a.res = res;
  const int64_t N = (int64_t)a.nt * a.slab;
  if (d->clamped.bytes < (size_t)N * sizeof(double)) d->clamped.alloc(N * sizeof(double));
  double *sc = d->clamped.as<double>();
  a.sc = sc;
  clamp_kernel<<<std::min<int64_t>(cdiv(N, 256), 8 * num_sms()), 256, 0, s>>>(a, sc);
  STMHD_LAUNCH_CHECK();
  constexpr TOff O = toff(NV, NP);
  const size_t smem = O.total * sizeof(double);
  static bool attr = false;
  if (!attr) {
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(residual_kernel<NV, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(values_kernel<NV, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr = true;
  }
  static const bool patch_env = [] {
    const char *e = getenv("STMHD_PATCH_ASM");
    return !e || atoi(e) != 0;
  }();
  if (res) {
    if (NV == 6 && NP == 3 && patch_env && d->dev.count("pr_desc")) {
      residual_patch(d, a, s);
    } else {
      residual_kernel<NV, NP><<<dim3(cdiv(a.slab, 256), a.nt), 256, smem, s>>>(a);
      STMHD_LAUNCH_CHECK();
    }
    pin_row_kernel<<<a.nt, 256, 0, s>>>(state, d->D<double>("p_mean_row"), a.n_p, a.slab, a.n_u, a.p_pin,
                                         d->R("p_mean_target"), res);
    STMHD_LAUNCH_CHECK();
  }
  const int ychunks = std::max(1, std::min(a.nt, 8));
  if (NV == 6 && NP == 3 && js && fp && patch_env && d->dev.count("pa_desc")) {
    values_patch(d, a, s, js, fp);
    js = fp = nullptr;
  }
  if (js) {
    ValArgs v{};
    v.nnz = (int)d->I("nnz_js");
    v.nt = a.nt;
    v.kind = d->D<int>("js_kind");
    v.cptr = d->D<int>("js_cptr");
    v.contrib = d->D<int>("js_contrib");
    v.out_stride = v.nnz;
    v.out = js;
    v.is_fp = 0;
    values_kernel<NV, NP><<<dim3(cdiv(v.nnz, 256), ychunks), 256, smem, s>>>(a, v);
    STMHD_LAUNCH_CHECK();
  }
  if (fp) {
    ValArgs v{};
    v.nnz = (int)d->I("nnz_fp");
    v.nt = a.nt;
    v.kind = nullptr;
    v.cptr = d->D<int>("fp_cptr");
    v.contrib = d->D<int>("fp_contrib");
    v.out_stride = v.nnz;
    v.out = fp;
    v.is_fp = 1;
    values_kernel<NV, NP><<<dim3(cdiv(v.nnz, 256), ychunks), 256, smem, s>>>(a, v);
    STMHD_LAUNCH_CHECK();
  }
  if (alf) {
    alfven_kernel<<<a.nt, 256, 12 * sizeof(double), s>>>(a, a.tensors + O.G1, d->R("elem_area"), d->R("area"), alf);
    STMHD_LAUNCH_CHECK();
  }
}

void assemble(stmhd_disc_s *d, cudaStream_t s, const double *state, const double *ic_u, const double *ic_a,
              double *res, double *js, double *fp, double *alf) {
  require(state && ic_u && ic_a, "stmhd_assemble: state, ic_u and ic_a are required");
  int nv = (int)d->I("nv"), np = (int)d->I("npl");
  if (nv == 6 && np == 3)
    assemble_t<6, 3>(d, s, state, ic_u, ic_a, res, js, fp, alf);
  else if (nv == 10 && np == 6)
    assemble_t<10, 6>(d, s, state, ic_u, ic_a, res, js, fp, alf);
  else
    throw Error(STMHD_CONFIG, "unsupported element pair (need P2/P1 or P3/P2)");
}

}  // namespace stmhd
