// Per-SM streaming rate of a per-warp cp.async.bulk ring (the sweep's factor path):
// G CTAs x W warps, every warp streams its own contiguous range in chunks of S
// doubles through D shared-memory slots, summing each chunk (GEMV stand-in).
// Diagnostics only: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_ring_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void ring_kernel(const double *src, long long per_warp, int S, int D, int use_ldg, double *out, int wmode, int P) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long mbar[32][4];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int W = blockDim.x >> 5;
  const double *base = src + ((long long)blockIdx.x * W + wl) * per_warp;
  double *slots = sm + (long long)wl * D * S;
  const int nch = (int)(per_warp / S);
  double acc = 0.0;
  long long t_arrive = 0, t_issue = 0;
  if (use_ldg == 2) {
    auto issue = [&](int c) {
      if (c < nch) {
        const double *g = base + (long long)c * S;
        double *d = slots + (c % D) * S;
        for (int i = 2 * lane; i < S; i += 64)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(d + i)), "l"(g + i) : "memory");
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    for (int d = 0; d < D; ++d) issue(d);
    for (int c = 0; c < nch; ++c) {
      if (D == 2) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else asm volatile("cp.async.wait_group 3;\n" ::: "memory");
      __syncwarp();
      const double *b = slots + (c % D) * S;
      if (wmode != 4)
        for (int i = lane; i < S; i += 32) acc += b[i];
      __syncwarp();
      issue(c + D);
    }
  } else if (use_ldg) {
    for (int c = 0; c < nch; ++c) {
      const double *p = base + (long long)c * S;
      for (int i = lane; i < S; i += 32) acc += __ldg(p + i);
    }
  } else {
    if (lane == 0) {
      for (int d = 0; d < D; ++d)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[wl][d])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    for (int d = 0; d < D && d < nch; ++d) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar[wl][d])),
                     "r"(S * 8)
                     : "memory");
      __syncwarp();
      if (lane < P) {
        const int ps = S / P;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_u32(slots + d * S + lane * ps)),
            "l"(base + (long long)d * S + lane * ps), "r"(ps * 8), "r"(smem_u32(&mbar[wl][d]))
            : "memory");
      }
    }
    for (int c = 0; c < nch; ++c) {
      const int sl = c % D;
      const unsigned ph = (unsigned)(c / D) & 1u;
      unsigned done = 0;
      if (wmode == 0) {
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(done)
              : "r"(smem_u32(&mbar[wl][sl])), "r"(ph)
              : "memory");
        } while (!done);
      } else if (wmode == 1) {
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(done)
              : "r"(smem_u32(&mbar[wl][sl])), "r"(ph)
              : "memory");
        } while (!done);
      } else {
        do {
          asm volatile(
              "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(done)
              : "r"(smem_u32(&mbar[wl][sl])), "r"(ph), "r"(20)
              : "memory");
        } while (!done);
      }
      const double *b = slots + sl * S;
      if (wmode == 3) {
        double a4[4] = {0, 0, 0, 0};
        for (int i = lane; i < S; i += 128) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (i + 32 * u < S) a4[u] += b[i + 32 * u];
        }
        acc += (a4[0] + a4[1]) + (a4[2] + a4[3]);
      } else if (wmode != 4) {
        for (int i = lane; i < S; i += 32) acc += b[i];
      }
      __syncwarp();
      if (c + D < nch) {
        long long q0 = clock64();
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar[wl][sl])),
                       "r"(S * 8)
                       : "memory");
        __syncwarp();
        long long q1 = clock64();
        if (lane == 0) { t_arrive += q1 - q0; }
        if (lane < P) {
          const int ps = S / P;
          if (wmode == 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  smem_u32(slots + sl * S + lane * ps)),
              "l"(base + (long long)(c + D) * S + lane * ps), "r"(ps * 8), "r"(smem_u32(&mbar[wl][sl]))
              : "memory");
          else if (wmode == 1)
          asm volatile(
              "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                  smem_u32(slots + sl * S + lane * ps)),
              "l"(base + (long long)(c + D) * S + lane * ps), "r"(ps * 8), "r"(smem_u32(&mbar[wl][sl]))
              : "memory");
          else
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
                  smem_u32(slots + sl * S + lane * ps)),
              "l"(base + (long long)(c + D) * S + lane * ps), "r"(ps * 8), "r"(smem_u32(&mbar[wl][sl])), "l"(0x14F0000000000000ull)
              : "memory");
        }
        __syncwarp();
        if (lane == 0) t_issue += clock64() - q1;
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
  if (lane == 0 && blockIdx.x == 0 && wl == 0) {
    out[1] = (double)t_arrive / nch;
    out[2] = (double)t_issue / nch;
  }
}

int main(int argc, char **argv) {
  const long long total = 1LL << 27;  // doubles (1 GB)
  double *src, *out;
  cudaMalloc(&src, total * 8);
  cudaMalloc(&out, 64);
  cudaMemset(src, 0, total * 8);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int Gs[] = {16};
  const int Ws[] = {8, 16};
  const int Ss[] = {320, 640};
  const int Ds[] = {2, 4};
  const int Ps[] = {1};
  for (int P : Ps)
  for (int wmode = 0; wmode < 3; wmode += 1)
  for (int l2 = 0; l2 < 1; ++l2)
    for (int G : Gs)
      for (int W : Ws)
        for (int S : Ss)
          for (int D : Ds)
            for (int ldg = 0; ldg < 1; ldg += 2) {
              const size_t smem = (size_t)W * D * S * 8;
              if (smem > 200 * 1024) continue;
              // l2 = 1: each warp re-reads a small range (L2 resident: 32 MB total)
              long long per_warp = l2 ? (32LL << 20) / 8 / ((long long)G * W) : total / ((long long)G * W);
              per_warp = per_warp / S * S;
              if (per_warp < 4 * S) continue;
              for (int it = 0; it < 2; ++it) ring_kernel<<<G, W * 32, smem>>>(src, per_warp, S, D, ldg, out, wmode, P);
              cudaEventRecord(e0);
              const int reps = 5;
              for (int it = 0; it < reps; ++it) ring_kernel<<<G, W * 32, smem>>>(src, per_warp, S, D, ldg, out, wmode, P);
              cudaEventRecord(e1);
              cudaEventSynchronize(e1);
              float ms;
              cudaEventElapsedTime(&ms, e0, e1);
              const double bytes = (double)per_warp * 8 * G * W * reps;
              double ho[3];
              cudaMemcpy(ho, out, 24, cudaMemcpyDeviceToHost);
              printf("arrive %.0f cyc issue %.0f cyc | ", ho[1], ho[2]);
              printf("P=%d mode%d %s G=%3d W=%2d S=%4d D=%d %s : %8.1f GB/s total  %6.1f GB/s per SM\n", P, wmode, l2 ? "L2 " : "HBM", G, W,
                     S, D, ldg ? "ldgsts" : "tma", bytes / ms / 1e6, bytes / ms / 1e6 / G);
            }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
