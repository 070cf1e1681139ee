// tcgen05.mma issue-rate microbenchmark: ./umma_rate <kind 0=tf32 1=f16 2=tf32-TS 3=bf16-TS> <N> <iters>
// One CTA per SM, one thread issues `iters` MMAs (M=128, K-major SW128 operands
// already in smem, same accumulator), timed with clock64 around commit/wait.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k(int kind, int N, int iters, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  for (int e = threadIdx.x; e < 65536 / 4; e += blockDim.x) ((float*)base)[e] = 0.001f * (e & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t fmt = kind == 1 ? 0u : kind == 3 ? 1u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                           ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t da = mk(su32(base)), db = mk(su32(base + 32768));
    long long t0 = clock64();
    if (kind == 0) {
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tb), "l"(da + (uint64_t)((u & 3) * 2)), "l"(db + (uint64_t)((u & 3) * 2)), "r"(idesc), "r"(1u) : "memory");
      }
    } else if (kind == 2) {  // A from TMEM (columns 256..), B from smem
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tb), "r"(tb + 256 + (u & 3) * 8), "l"(db + (uint64_t)((u & 3) * 2)), "r"(idesc), "r"(1u) : "memory");
      }
    } else if (kind == 3) {  // bf16, A from TMEM
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tb), "r"(tb + 256 + (u & 3) * 8), "l"(db + (uint64_t)((u & 3) * 2)), "r"(idesc), "r"(1u) : "memory");
      }
    } else {
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tb), "l"(da + (uint64_t)((u & 3) * 2)), "l"(db + (uint64_t)((u & 3) * 2)), "r"(idesc), "r"(1u) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512) : "memory");
}

int main(int argc, char** argv) {
  const int kind = atoi(argv[1]), N = atoi(argv[2]), iters = atoi(argv[3]);
  long long* cyc; cudaMallocManaged(&cyc, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<148, 128, 100000>>>(kind, N, iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  const double c = (double)cyc[0] / iters;
  const int K = (kind == 1 || kind == 3) ? 16 : 8;
  printf("kind %s N %d: %.1f cycles/MMA, %.0f MAC/cycle/SM (%s)\n", kind == 0 ? "tf32" : kind == 2 ? "tf32-TS" : kind == 3 ? "bf16-TS" : "f16", N, c,
         128.0 * N * K / c, cudaGetErrorString(e));
}
