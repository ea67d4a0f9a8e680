// Micro-benchmarks of the synchronisation primitives the sweep kernel uses
// (diagnostics only; exported as stmhd_bench_barrier).
#include "nd.hpp"

namespace stmhd {

__device__ __forceinline__ void mb_barrier(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    unsigned g = *gen;
    __threadfence();
    unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void barrier_kernel(unsigned *bar, int n) {
  for (int i = 0; i < n; ++i) mb_barrier(bar);
}

// dependent-load chain (pointer chase) + cluster barriers inside one cluster
__global__ void chase_kernel(const int *next, int steps, int nbar, unsigned long long *out) {
  unsigned long long t0, t1, t2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  int p = (int)((threadIdx.x * 997ll + blockIdx.x * 131ll) % 1021);
  for (int i = 0; i < steps; ++i) p = next[p];
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  for (int i = 0; i < nbar; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = (unsigned long long)p;
  }
}

// one warp per CTA of a cluster chases pointers; optionally a cluster barrier
// (release/acquire) between consecutive loads
__global__ void chase2_kernel(const int *next, int steps, int with_bar, int64_t nelem, unsigned long long *out) {
  long long c0 = clock64();
  int p = (int)((threadIdx.x * 7919ll + blockIdx.x * 104729ll) % nelem);
  for (int i = 0; i < steps; ++i) {
    p = next[p];
    if (with_bar) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
  }
  long long c1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (unsigned long long)(c1 - c0);
    out[1] = (unsigned long long)p;
  }
}

}  // namespace stmhd

using namespace stmhd;

extern "C" int stmhd_bench_chase2(int64_t nelem, int steps, int cluster, int threads, int with_bar,
                                  double *cycles_per_step) {
  try {
    std::vector<int> perm(nelem), h(nelem);
    for (int64_t i = 0; i < nelem; ++i) perm[i] = (int)i;
    uint64_t st = 88172645463325252ull;
    for (int64_t i = nelem - 1; i > 0; --i) {
      st ^= st << 13; st ^= st >> 7; st ^= st << 17;
      int64_t j = st % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    for (int64_t i = 0; i < nelem; ++i) h[perm[i]] = perm[(i + 1) % nelem];
    DevBuf d = upload_vec(h, 0);
    DevBuf out(2 * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(chase2_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int *dp = d.as<int>();
    unsigned long long *op = out.as<unsigned long long>();
    void *args[] = {&dp, &steps, &with_bar, &nelem, &op};
    for (int rep = 0; rep < 2; ++rep) STMHD_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void *)chase2_kernel, args));
    unsigned long long r[2];
    STMHD_CUDA_CHECK(cudaMemcpy(r, out.ptr, sizeof(r), cudaMemcpyDeviceToHost));
    *cycles_per_step = (double)r[0] / steps;
    return 0;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.status;
  }
}

extern "C" int stmhd_bench_chase(int64_t nelem, int steps, int cluster, int threads, int nbar, double *ns_per_load,
                                 double *ns_per_barrier) {
  try {
    std::vector<int> h(nelem);
    // random cyclic permutation
    std::vector<int> perm(nelem);
    for (int64_t i = 0; i < nelem; ++i) perm[i] = (int)i;
    uint64_t st = 88172645463325252ull;
    for (int64_t i = nelem - 1; i > 0; --i) {
      st ^= st << 13; st ^= st >> 7; st ^= st << 17;
      int64_t j = st % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    for (int64_t i = 0; i < nelem; ++i) h[perm[i]] = perm[(i + 1) % nelem];
    DevBuf d = upload_vec(h, 0);
    DevBuf out(3 * sizeof(unsigned long long));
    STMHD_CUDA_CHECK(cudaFuncSetAttribute(chase_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int *dp = d.as<int>();
    unsigned long long *op = out.as<unsigned long long>();
    void *args[] = {&dp, &steps, &nbar, &op};
    for (int rep = 0; rep < 2; ++rep)
      STMHD_CUDA_CHECK(cudaLaunchKernelExC(&cfg, (const void *)chase_kernel, args));
    unsigned long long r[3];
    STMHD_CUDA_CHECK(cudaMemcpy(r, out.ptr, sizeof(r), cudaMemcpyDeviceToHost));
    *ns_per_load = (double)r[0] / steps;
    *ns_per_barrier = nbar ? (double)r[1] / nbar : 0.0;
    return 0;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.status;
  }
}

extern "C" int stmhd_bench_barrier(int blocks_per_sm, int threads, int nbar, double *us_per_barrier) {
  try {
    DevBuf bar(2 * sizeof(unsigned));
    STMHD_CUDA_CHECK(cudaMemset(bar.ptr, 0, 2 * sizeof(unsigned)));
    int grid = blocks_per_sm * num_sms();
    unsigned *b = bar.as<unsigned>();
    void *args[] = {&b, &nbar};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    STMHD_CUDA_CHECK(cudaLaunchCooperativeKernel((void *)barrier_kernel, dim3(grid), dim3(threads), args, 0, 0));
    cudaEventRecord(e0);
    STMHD_CUDA_CHECK(cudaLaunchCooperativeKernel((void *)barrier_kernel, dim3(grid), dim3(threads), args, 0, 0));
    cudaEventRecord(e1);
    STMHD_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *us_per_barrier = 1e3 * ms / nbar;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
  } catch (const Error &e) {
    set_last_error(e.what());
    return e.status;
  }
}
