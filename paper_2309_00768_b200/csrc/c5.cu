// Configuration-5 scalar advection-diffusion block (oracle/c5.py):
// per slab F_k = M/dt + eps K + W(u_k) on a P1 space (W: reference fem.py:430-462,
// lin_a with a P1 vector velocity), Dirichlet rows/columns -> identity, sub-diagonal -C with
// C = bc_zero(M/dt).  Device parts: entry-centric assembly of every slab's values in
// a fixed pattern, the block-bidiagonal batched SpMV, and the exact inverse by the
// cluster sweep over a batched LU (NDFactor::sweep).
#include <cstdint>

#include "capi_common.hpp"
#include "disc.hpp"
#include "nd.hpp"

namespace stmhd {

struct C5Args {
  int64_t nnz;
  const double *base;   // M/dt + eps K at the pattern entries (identity rows on BC rows)
  const int *cptr;      // nnz + 1: element contributions of each entry
  const int4 *cinfo;    // {element, local row, local col, orientation}
  const int *elem;      // 3 nodes per element
  const double *u;      // [slab][node][2]
  int64_t n_nodes;
  double m[3][3];       // P1 element mass (same on both orientations)
  double g[2][3][2];    // P1 basis gradients per orientation
  double *values;       // [slab][nnz]
};

// values[k][e] = base[e] + sum over the entry's element contributions of
//   int psi_i (u_k . grad psi_j) = sum_c g[o][j][c] sum_m M[i][m] u_k[node_m][c]
__global__ void c5_values_kernel(C5Args a) {
  const int k = blockIdx.y;
  const double *uk = a.u + (int64_t)k * a.n_nodes * 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < a.nnz; e += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = a.cptr[e]; j < a.cptr[e + 1]; ++j) {
      const int4 c = a.cinfo[j];
      const int *nd = a.elem + 3 * (int64_t)c.x;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double2 um = reinterpret_cast<const double2 *>(uk)[nd[m]];
        s0 = fma(a.m[c.y][m], um.x, s0);
        s1 = fma(a.m[c.y][m], um.y, s1);
      }
      acc = fma(a.g[c.w][c.z][0], s0, fma(a.g[c.w][c.z][1], s1, acc));
    }
    a.values[(int64_t)k * a.nnz + e] = a.base[e] + acc;
  }
}


// Advection fields of configuration 5: per slab, 8 Fourier modes
// (kx, ky, amplitude) of the stream function psi = sum a sin(pi kx (x+1)/2) sin(pi ky (y+1)/2),
// u = (d_y psi, -d_x psi) at the P1 nodes, rescaled to max |u| = 1 -- the same sums,
// in the same order, as the host generator c5.c5_velocity_fields.
__global__ void c5_velocity_kernel(const double *xy, int64_t n, const double *modes, double *u,
                                   unsigned long long *umax) {
  const int k = blockIdx.y;
  const double *md = modes + (int64_t)k * 24;
  const double h = 0.5 * 3.141592653589793;
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = xy[2 * i] + 1.0, y = xy[2 * i + 1] + 1.0;
    double ux = 0.0, uy = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double kx = md[3 * q], ky = md[3 * q + 1], a = md[3 * q + 2];
      double sx, cx, sy, cy;
      sincos(h * kx * x, &sx, &cx);
      sincos(h * ky * y, &sy, &cy);
      ux += a * sx * (h * ky) * cy;
      uy -= a * (h * kx) * cx * sy;
    }
    u[((int64_t)k * n + i) * 2] = ux;
    u[((int64_t)k * n + i) * 2 + 1] = uy;
    m = fmax(m, sqrt(ux * ux + uy * uy));
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomicMax(umax + k, __double_as_longlong(m));  // m >= 0: bit order = value order
}

__global__ void c5_velocity_scale_kernel(int64_t n, const unsigned long long *umax, double *u) {
  const int k = blockIdx.y;
  const double sc = __longlong_as_double(umax[k]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n; i += (int64_t)gridDim.x * blockDim.x)
    u[(int64_t)k * 2 * n + i] /= sc;
}

}  // namespace stmhd

using namespace stmhd;

extern "C" {

int stmhd_c5_values(void *stream, int64_t nnz, int nt, const double *base, const int32_t *cptr,
                    const int32_t *cinfo, const int32_t *elem, const double *u, int64_t n_nodes,
                    const double *mloc9, const double *grad12, double *values) {
  CAPI_BEGIN
  require(nnz >= 0 && nt >= 1 && base && cptr && cinfo && elem && u && mloc9 && grad12 && values,
          "stmhd_c5_values: bad arguments");
  C5Args a{};
  a.nnz = nnz;
  a.base = base;
  a.cptr = cptr;
  a.cinfo = reinterpret_cast<const int4 *>(cinfo);
  a.elem = elem;
  a.u = u;
  a.n_nodes = n_nodes;
  for (int i = 0; i < 9; ++i) a.m[i / 3][i % 3] = mloc9[i];
  for (int i = 0; i < 12; ++i) a.g[i / 6][(i / 2) % 3][i % 2] = grad12[i];
  a.values = values;
  c5_values_kernel<<<dim3((unsigned)std::min<int64_t>(cdiv(std::max<int64_t>(nnz, 1), 256), 1024), nt), 256, 0,
                     (cudaStream_t)stream>>>(a);
  STMHD_LAUNCH_CHECK();
  CAPI_END
}

int stmhd_c5_velocity(void *stream, int64_t n_nodes, int nt, const double *xy, const double *modes_host,
                      double *u) {
  CAPI_BEGIN
  require(n_nodes >= 1 && nt >= 1 && xy && modes_host && u, "stmhd_c5_velocity: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  DevBuf md((size_t)nt * 24 * sizeof(double)), mx((size_t)nt * sizeof(unsigned long long));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(md.ptr, modes_host, md.bytes, cudaMemcpyHostToDevice, s));
  STMHD_CUDA_CHECK(cudaMemsetAsync(mx.ptr, 0, mx.bytes, s));
  const unsigned gx = (unsigned)std::min<int64_t>(cdiv(n_nodes, 256), 64);
  c5_velocity_kernel<<<dim3(gx, nt), 256, 0, s>>>(xy, n_nodes, md.as<double>(), u, mx.as<unsigned long long>());
  STMHD_LAUNCH_CHECK();
  c5_velocity_scale_kernel<<<dim3(gx, nt), 256, 0, s>>>(n_nodes, mx.as<unsigned long long>(), u);
  STMHD_LAUNCH_CHECK();
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));  // scratch buffers die here
  CAPI_END
}

int stmhd_bidiag_spmv(void *stream, int64_t n, int nt, const int32_t *rowptr, const int32_t *col,
                      const double *vals, int64_t val_stride, const int32_t *c_rowptr, const int32_t *c_col,
                      const double *c_val, double c_coef, const double *x, double *y) {
  CAPI_BEGIN
  require(n >= 1 && nt >= 1 && rowptr && col && vals && x && y, "stmhd_bidiag_spmv: bad arguments");
  SpmvArgs a;
  a.nrows = (int)n;
  a.nslab = nt;
  a.y = y;
  a.y_stride = n;
  SpTerm f;
  f.beg = rowptr;
  f.col = col;
  f.val = vals;
  f.val_stride = val_stride;
  f.x = x;
  f.x_stride = n;
  a.t[0] = f;
  a.nterms = 1;
  if (c_rowptr) {
    SpTerm c;
    c.beg = c_rowptr;
    c.col = c_col;
    c.val = c_val;
    c.x = x;
    c.x_stride = n;
    c.lag = 1;
    c.alpha = c_coef;
    a.t[1] = c;
    a.nterms = 2;
  }
  spmv(a, (cudaStream_t)stream, 8);
  CAPI_END
}

}  // extern "C"
