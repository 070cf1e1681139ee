// tcgen05.mma kind::f16 TS-form issue/execution rate for the slide-MMA conv
// (csrc/conv2d_mma.cu): M128 x N x K16, A in TMEM, B in smem (no swizzle).
//   ./ts_rate <N> <iters> <issuers> <dmode> <ldwarps>
//   dmode 0: every MMA into the same D; 1: D steps by 8 columns per MMA over a
//   256-column ring (mask, no division); 2: three MMAs per "row" into the same
//   D, then the next row's D 8 columns later (the conv kernel's pattern)
//   ldwarps: extra warps that tcgen05.ld / st other TMEM columns meanwhile
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t mk(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)(lay & 7) << 61);
}

__global__ void k(int N, int iters, int issuers, int dmode, int ldwarps, long long* cyc, int* cnt, int commits, int amode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sb = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar, bar2[4];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) reinterpret_cast<uint32_t*>(sb)[e] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(issuers));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar2[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tb))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((128u >> 4) << 24);
  if (warp < issuers) {
    const uint64_t db = mk(su32(sb), 128, 256, 0);
    const uint32_t a0 = tb + 320;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        uint32_t d;
        if (dmode == 0) d = tb;
        else if (dmode == 1) d = tb + (((it * 3 + r) * 8) & 255);
        else if (dmode == 2) d = tb + ((it * 8) & 255);
        else if (dmode == 3) d = tb + (warp & 1) * 160 + ((it * 16) & 63);   // own ring, window shifts 16 cols per row
        else d = tb + warp * 160 + ((it * 64) & 63);                   // own ring, disjoint windows
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.eq.u32 p, 1, 1;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(amode ? a0 + 16 * (uint32_t)((it * 2 + warp) % 12) + (r == 2 ? 8u : 0u) : a0 + 16 * warp), "l"(db), "r"(idesc)
            : "memory");
      }
      if (commits)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                su32(&bar2[warp]))
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            su32(&bar))
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], "
          "0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&bar))
          : "memory");
    if (threadIdx.x == 0) {
      *cyc = clock64() - t0;
      stop = 1;
    }
  } else if (warp >= 4 && warp < 4 + ldwarps) {
    // TMEM traffic on columns 256..383 of this warp's lane quarter
    const uint32_t base = tb + ((uint32_t)(32 * (warp & 3)) << 16) + 256;
    int n = 0;
    while (!stop) {
      uint32_t v[8];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7])
          : "r"(base + (n & 15) * 8));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
              base + ((n + 3) & 15) * 8),
          "r"(v[0] & 0u)
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      ++n;
    }
    if (lane == 0) atomicAdd(cnt, n);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 64, iters = argc > 2 ? atoi(argv[2]) : 2000;
  const int issuers = argc > 3 ? atoi(argv[3]) : 1, dmode = argc > 4 ? atoi(argv[4]) : 0;
  const int ldw = argc > 5 ? atoi(argv[5]) : 0, commits = argc > 6 ? atoi(argv[6]) : 0;
  const int amode = argc > 7 ? atoi(argv[7]) : 0;
  long long* cyc;
  cudaMalloc(&cyc, 8);
  int* cnt;
  cudaMalloc(&cnt, 4);
  cudaMemset(cnt, 0, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<<<1, 256, 32768>>>(N, iters, issuers, dmode, ldw, cyc, cnt, commits, amode);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  int hc = 0;
  cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost);
  if (ldw) printf("  ld/st warp iterations: %.0f cycles each\n", (double)c * ldw / (hc ? hc : 1));
  printf("amode %d commits %d TS N %d issuers %d dmode %d ldwarps %d: %s %.1f cycles/MMA (ideal %d)\n", amode, commits, N, issuers,
         dmode, ldw, cudaGetErrorString(e), (double)c / (3.0 * iters * issuers), N / 2);
  return 0;
}
