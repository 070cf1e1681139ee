// How many tcgen05.mma (bf16, TS form, M128 N128 K16) can one thread issue
// before the issue blocks: clock64 after each of 24 back-to-back issues.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k(long long* out, int n, int nw) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  for (int e = threadIdx.x; e < 32768 / 4; e += blockDim.x) ((float*)base)[e] = 0.f;
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
  if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < nw) {
    const int wi = threadIdx.x >> 5;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t db = mk(su32(base));
    long long t[24];
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 24; ++i) {
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tb + wi * 128), "r"(tb + 256 + wi * 64 + (i & 3) * 8), "l"(db + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(1u) : "memory");
      t[i] = clock64();
    }
    long long tc = clock64(), te = tc;
    if (wi == 0) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      tc = clock64();
      uint32_t ok = 0;
      while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
      te = clock64();
    }
    for (int i = 0; i < 24; ++i) out[wi * 26 + i] = t[i] - t0;
    out[wi * 26 + 24] = tc - t0;
    out[wi * 26 + 25] = te - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512) : "memory");
}

int main() {
  long long* d;
  cudaMallocManaged(&d, 4 * 26 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int nw : {1, 2, 4}) {
    k<<<1, 128, 40000>>>(d, 128, nw);
    cudaError_t e = cudaDeviceSynchronize();
    for (int wi = 0; wi < nw; ++wi) {
      printf("warps=%d w%d (%s): issue clocks:", nw, wi, cudaGetErrorString(e));
      for (int i = 0; i < 24; i += 4) printf(" %lld", d[wi * 26 + i]);
      printf(" last %lld | commit %lld done %lld\n", d[wi * 26 + 23], d[wi * 26 + 24], d[wi * 26 + 25]);
    }
  }
}
