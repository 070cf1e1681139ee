// Two (or four) warps issue bf16 TS MMAs (M128 N128 K16, all-ones operands)
// into the SAME accumulator: are updates lost?  Expect D = iters*warps*16.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k(float* out, int iters, int nw, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar[4];
  for (int e = threadIdx.x; e < 32768 / 4; e += blockDim.x) ((uint32_t*)base)[e] = 0x3f803f80u;  // bf16 1.0 pairs
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
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
  // A (TMEM cols 256..263) = ones: every warp writes its lane quarter
  if (warp < 4) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = 0x3f803f80u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + ((32 * warp) << 16) + 256),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t db = mk(su32(base));
  if (warp == 0 && lane == 0) {  // zero D first
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(tb), "r"(tb + 256), "l"(db), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[3])) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar[3])) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  long long t0 = clock64();
  if (warp < nw && lane == 0) {
    for (int i = 0; i < iters; ++i)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tb), "r"(tb + 256), "l"(db), "r"(idesc), "r"(1u) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp])) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar[warp])) : "memory");
    cyc[warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    uint32_t r[8];
    for (int c0 = 0; c0 < 128; c0 += 8) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tb + ((32 * warp) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 8; ++i) out[(32 * warp + lane) * 128 + c0 + i] = __uint_as_float(r[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512) : "memory");
}

int main() {
  float* d;
  long long* cyc;
  cudaMallocManaged(&d, 128 * 128 * 4);
  cudaMallocManaged(&cyc, 4 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int nw : {1, 2, 4}) {
    for (int rep = 0; rep < 3; ++rep) {
      const int iters = 4000;
      k<<<1, 128, 40000>>>(d, iters, nw, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      const float expect = 16.0f * iters * nw;  // exact in fp32 (< 2^24)
      int bad = 0;
      float mn = 1e30f, mx = -1e30f;
      for (int i = 0; i < 128 * 128; ++i) {
        bad += d[i] != expect;
        mn = d[i] < mn ? d[i] : mn;
        mx = d[i] > mx ? d[i] : mx;
      }
      printf("warps %d rep %d (%s): expect %.0f min %.0f max %.0f bad %d  cycles/MMA/warp %.1f\n", nw, rep,
             cudaGetErrorString(e), expect, mn, mx, bad, (double)cyc[0] / iters);
    }
  }
}
