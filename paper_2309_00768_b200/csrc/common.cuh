// Shared helpers for the stmhd_b200 native library (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/stmhd_b200.h"

namespace stmhd {

// Exception carrying a C-ABI status code; converted at the extern "C" boundary.
struct Error : std::runtime_error {
  int status;
  std::string block;
  Error(int s, const std::string &m, const std::string &b = "") : std::runtime_error(m), status(s), block(b) {}
};

void set_last_error(const std::string &msg, const std::string &block = "");

#define STMHD_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::stmhd::Error(STMHD_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// every kernel launch of the library goes through this check: it also counts
// launches (stmhd_launch_count) so benchmarks can report what ran natively
void count_launch();
#define STMHD_LAUNCH_CHECK()                    \
  do {                                          \
    ::stmhd::count_launch();                    \
    STMHD_CUDA_CHECK(cudaGetLastError());       \
  } while (0)

inline void require(bool cond, const std::string &msg) {
  if (!cond) throw Error(STMHD_CONFIG, msg);
}

// Owning device allocation.
// Device buffer.  alloc() uses cudaMalloc; alloc_async() takes the block from the
// device's default stream-ordered pool (kept, not returned to the driver), which is
// what the per-Newton-step preconditioner storage uses: a new preconditioner reuses
// the blocks of the previous one without cudaMalloc/cudaFree round trips.
inline void ensure_pool_retained() {
  static bool done = false;
  if (!done) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = true;
  }
}

struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;  // pooled buffers: freed in order on this stream
  bool pooled = false;
  DevBuf() = default;
  explicit DevBuf(size_t b) { alloc(b); }
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  DevBuf(DevBuf &&o) noexcept : ptr(o.ptr), bytes(o.bytes), stream(o.stream), pooled(o.pooled) {
    o.ptr = nullptr;
    o.bytes = 0;
  }
  DevBuf &operator=(DevBuf &&o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      bytes = o.bytes;
      stream = o.stream;
      pooled = o.pooled;
      o.ptr = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t b) {
    release();
    bytes = b;
    pooled = false;
    if (b) STMHD_CUDA_CHECK(cudaMalloc(&ptr, b));
  }
  void alloc_async(size_t b, cudaStream_t s) {
    release();
    ensure_pool_retained();
    bytes = b;
    stream = s;
    pooled = true;
    if (b) STMHD_CUDA_CHECK(cudaMallocAsync(&ptr, b, s));
  }
  void release() {
    if (ptr) {
      if (pooled) cudaFreeAsync(ptr, stream);
      else cudaFree(ptr);
    }
    ptr = nullptr;
    bytes = 0;
  }
  template <class T> T *as() const { return static_cast<T *>(ptr); }
};

template <class T>
inline DevBuf upload_vec(const std::vector<T> &v, cudaStream_t s) {
  DevBuf b(v.size() * sizeof(T));
  if (!v.empty()) STMHD_CUDA_CHECK(cudaMemcpyAsync(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return b;
}

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// ---- device helpers ----
#if defined(__CUDACC__)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction (fixed tree); `sh` holds >= blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double *sh) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  int nw = (blockDim.x + 31) >> 5;
  double r = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}
#endif  // __CUDACC__

}  // namespace stmhd
