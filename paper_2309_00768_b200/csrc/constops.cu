// State-independent operators on the device: mass, stiffness,
// divergence and mixed blocks of the uniform right-triangulated mesh, assembled from the
// two per-orientation element matrices (reference fem.py:211-271 assemble_mass /
// assemble_stiffness / assemble_divergence and their use in problems.py:185-204; the
// reference sums einsum element matrices through a COO -> CSR conversion).
//
// One thread owns one row node.  Pass 1 counts the distinct column nodes of the row's
// elements, an exclusive scan gives the row pointers, pass 2 writes the sorted columns
// and sums each entry's element contributions in ascending element order (a fixed
// order: the result is deterministic).  Runs once per discretisation.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>

#include "capi_common.hpp"

namespace stmhd {

constexpr int kConstMaxCols = 96;  // distinct columns of one row (P3 vertex: 37; P2: 19)

struct ConstArgs {
  int64_t n_rows;
  int nr, nc;
  const int *ne_ptr, *ne_code;  // elements of each row node: code = element * 16 + local row
  const int *elem_c;            // column nodes per element
  const double *local;          // [2][nr][nc], orientation = element & 1
  int *rowptr;                  // pass 1: counts (shifted by one); pass 2: pointers
  int *col;
  double *val;
  int *overflow;
};

// sorted distinct column nodes of row r into cols[], returns the count (or -1)
__device__ int const_row_columns(const ConstArgs &a, int64_t r, int *cols) {
  int n = 0;
  for (int q = a.ne_ptr[r]; q < a.ne_ptr[r + 1]; ++q) {
    const int e = a.ne_code[q] >> 4;
    for (int jl = 0; jl < a.nc; ++jl) {
      const int c = a.elem_c[(int64_t)e * a.nc + jl];
      int p = 0;
      while (p < n && cols[p] < c) ++p;
      if (p < n && cols[p] == c) continue;
      if (n == kConstMaxCols) return -1;
      for (int s = n; s > p; --s) cols[s] = cols[s - 1];
      cols[p] = c;
      ++n;
    }
  }
  return n;
}

__global__ void const_count_kernel(ConstArgs a) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= a.n_rows) return;
  int cols[kConstMaxCols];
  const int n = const_row_columns(a, r, cols);
  if (n < 0) {
    *a.overflow = 1;
    a.rowptr[r] = 0;
    return;
  }
  a.rowptr[r] = n;
}

__global__ void const_fill_kernel(ConstArgs a) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= a.n_rows) return;
  int cols[kConstMaxCols];
  double acc[kConstMaxCols];
  const int n = const_row_columns(a, r, cols);
  if (n < 0) return;
  for (int p = 0; p < n; ++p) acc[p] = 0.0;
  for (int q = a.ne_ptr[r]; q < a.ne_ptr[r + 1]; ++q) {
    const int code = a.ne_code[q], e = code >> 4, il = code & 15;
    const double *loc = a.local + ((int64_t)(e & 1) * a.nr + il) * a.nc;
    for (int jl = 0; jl < a.nc; ++jl) {
      const int c = a.elem_c[(int64_t)e * a.nc + jl];
      int lo = 0, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cols[mid] < c) lo = mid + 1;
        else hi = mid;
      }
      acc[lo] += loc[jl];
    }
  }
  const int base = a.rowptr[r];
  for (int p = 0; p < n; ++p) {
    a.col[base + p] = cols[p];
    a.val[base + p] = acc[p];
  }
}

}  // namespace stmhd

using namespace stmhd;

extern "C" int stmhd_const_assemble(void *stream, int64_t n_rows, int nr, int nc, int64_t ne,
                                    const int32_t *ne_ptr, const int32_t *ne_code, const int32_t *elem_c,
                                    const double *local, int32_t *rowptr, int32_t *col, double *val,
                                    int64_t capacity, int64_t *nnz) {
  CAPI_BEGIN
  require(n_rows > 0 && ne > 0 && nr > 0 && nr <= 16 && nc > 0, "const_assemble: bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  // incidence list length = ne_ptr[n_rows] (host)
  const int64_t n_inc = ne_ptr[n_rows];
  require(n_inc == ne * nr, "const_assemble: incidence list does not match ne * nr");
  DevBuf d_ptr((n_rows + 1) * sizeof(int)), d_code(n_inc * sizeof(int)), d_elem(ne * nc * sizeof(int));
  DevBuf d_rowptr((n_rows + 1) * sizeof(int)), d_loc((size_t)2 * nr * nc * sizeof(double)), d_flag(sizeof(int));
  DevBuf d_col, d_val, d_tmp;
  STMHD_CUDA_CHECK(cudaMemcpyAsync(d_ptr.ptr, ne_ptr, (n_rows + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(d_code.ptr, ne_code, (size_t)n_inc * sizeof(int), cudaMemcpyHostToDevice, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(d_elem.ptr, elem_c, (size_t)ne * nc * sizeof(int), cudaMemcpyHostToDevice, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(d_loc.ptr, local, (size_t)2 * nr * nc * sizeof(double), cudaMemcpyHostToDevice, s));
  STMHD_CUDA_CHECK(cudaMemsetAsync(d_flag.ptr, 0, sizeof(int), s));
  STMHD_CUDA_CHECK(cudaMemsetAsync(d_rowptr.ptr, 0, (n_rows + 1) * sizeof(int), s));
  ConstArgs a{};
  a.n_rows = n_rows, a.nr = nr, a.nc = nc;
  a.ne_ptr = d_ptr.as<int>(), a.ne_code = d_code.as<int>(), a.elem_c = d_elem.as<int>();
  a.local = d_loc.as<double>();
  a.rowptr = d_rowptr.as<int>(), a.overflow = d_flag.as<int>();
  const int threads = 128, blocks = (int)((n_rows + threads - 1) / threads);
  const_count_kernel<<<blocks, threads, 0, s>>>(a);
  STMHD_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  STMHD_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, a.rowptr, a.rowptr, (int)(n_rows + 1), s));
  d_tmp.alloc(std::max<size_t>(tmp_bytes, 1));
  STMHD_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(d_tmp.ptr, tmp_bytes, a.rowptr, a.rowptr, (int)(n_rows + 1), s));
  count_launch();
  int total = 0, flag = 0;
  STMHD_CUDA_CHECK(cudaMemcpyAsync(&total, a.rowptr + n_rows, sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(&flag, d_flag.ptr, sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  require(!flag, "const_assemble: a row has more distinct columns than the kernel holds");
  *nnz = total;
  require(total <= capacity, "const_assemble: output capacity too small");
  d_col.alloc((size_t)std::max(total, 1) * sizeof(int)), d_val.alloc((size_t)std::max(total, 1) * sizeof(double));
  a.col = d_col.as<int>(), a.val = d_val.as<double>();
  const_fill_kernel<<<blocks, threads, 0, s>>>(a);
  STMHD_LAUNCH_CHECK();
  STMHD_CUDA_CHECK(cudaMemcpyAsync(rowptr, a.rowptr, (n_rows + 1) * sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(col, a.col, (size_t)total * sizeof(int), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaMemcpyAsync(val, a.val, (size_t)total * sizeof(double), cudaMemcpyDeviceToHost, s));
  STMHD_CUDA_CHECK(cudaStreamSynchronize(s));
  CAPI_END
}
