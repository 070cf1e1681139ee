// Two issuer warps, bf16 TS MMAs into one accumulator, the NCHW tensor-core
// kernel's pattern: warp 0 issues N=n0 (A = x1 columns), warp 1 N=n1 (A = x2
// columns), A advancing 8 columns per k-step over 4 k-steps, B advancing 32 B.
// ./umma_dual n0 n1 iters  -> cycles per k-step (both MMAs)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(1u) : "memory");
}

__global__ void k(int n0, int n1, int iters, long long* out, int fill, int boff) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar[2];
  for (int e = threadIdx.x; e < 16384 / 4; e += blockDim.x) {
    uint32_t hsh = (uint32_t)e * 2654435761u;
    hsh ^= hsh >> 13;
    ((uint32_t*)base)[e] = fill ? (0x3c003c00u ^ (hsh & 0x03ff03ffu)) : 0u;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
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
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (fill) {  // A in TMEM (lane quarter of this warp... only warps 0,1 -> quarters 0,1; good enough)
    for (int c = 256; c < 512; c += 8) {
      uint32_t v[8];
      for (int i = 0; i < 8; ++i) {
        uint32_t hsh = (uint32_t)(c * 8 + i + lane * 977) * 2654435761u;
        v[i] = 0x3c003c00u ^ ((hsh >> 7) & 0x03ff03ffu);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + ((32 * (warp & 3)) << 16) + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int n = warp == 0 ? n0 : n1;
  if (warp < 2 && lane == 0 && n > 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t db = mk(su32(base) + boff);
    const uint32_t a0 = tb + 256 + warp * 32;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) mma(tb, a0 + 8 * ks, db + 2 * ks, idesc);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar[warp])) : "memory");
    out[warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512) : "memory");
}

int main(int argc, char** argv) {
  const int n0 = atoi(argv[1]), n1 = atoi(argv[2]), iters = argc > 3 ? atoi(argv[3]) : 4000;
  long long* d;
  cudaMallocManaged(&d, 16);
  d[0] = d[1] = 0;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  const int fill = argc > 4 ? atoi(argv[4]) : 0;
  const int boff = argc > 5 ? atoi(argv[5]) : 0;
  k<<<148, 128, 20000>>>(n0, n1, iters, d, fill, boff);
  cudaError_t e = cudaDeviceSynchronize();
  printf("boff=%d fill=%d n0=%d n1=%d (%s): warp0 %.1f warp1 %.1f cycles per k-step\n", argc > 5 ? atoi(argv[5]) : 0, fill, n0, n1, cudaGetErrorString(e),
         (double)d[0] / iters, (double)d[1] / iters);
}
