// Round-trip latency of mbarrier hand-offs between two warps, with the
// forward signal a plain mbarrier.arrive (mode 0), a tcgen05.commit with no
// MMA outstanding (mode 1), or a commit after one tf32 M128 N64 K8 MMA
// (mode 2).  Also the self latency commit -> try_wait in one thread (mode 3).
// ./commit_lat <mode> <iters>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool tryw(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
               "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void waitb(uint64_t* b, uint32_t ph) { while (!tryw(b, ph)) {} }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k(int mode, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t X, Y;
  for (int e = threadIdx.x; e < 32768 / 4; e += blockDim.x) ((float*)base)[e] = 0.001f * (e & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&X)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&Y)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = mk(su32(base)), db = mk(su32(base + 16384));
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (mode == 0) arrive(&X);
      else if (mode == 1 || mode == 3) commit(&X);
      else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tb), "l"(da), "l"(db), "r"(idesc), "r"(1) : "memory");
        commit(&X);
      }
      if (mode == 3) waitb(&X, i & 1);
      else waitb(&Y, i & 1);
    }
    out[0] = clock64() - t0;
  } else if (threadIdx.x == 32 && mode != 3) {
    for (int i = 0; i < iters; ++i) {
      waitb(&X, i & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      arrive(&Y);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(128) : "memory");
  }
}

int main(int argc, char** argv) {
  int iters = argc > 2 ? atoi(argv[2]) : 10000;
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    k<<<1, 64, 33 * 1024>>>(mode, iters, d);
    long long c = 0;
    cudaError_t e = cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: %s  %.1f cycles per round trip\n", mode, cudaGetErrorString(e), (double)c / iters);
  }
  return 0;
}
