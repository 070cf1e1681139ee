// tcgen05.mma kind::tf32 TS form with M = 64: which TMEM lanes of A are read
// and which lanes of D are written?  D is pre-filled with a sentinel; each
// written D element is matched against dot(A[m], B[n]) for every m.  Also
// times M = 64 vs M = 128 (bf16, N = 112) issue throughput.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__global__ void k(const float* A, const float* B, float* D, uint32_t idesc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sb = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int n = e / 32, kk = e % 32;
    *reinterpret_cast<float*>(sb + n * 128 + (((kk >> 2) ^ (n & 7)) << 4) + (kk & 3) * 4) = kk < 8 ? B[n * 8 + kk] : 0.f;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(128) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int m = 32 * warp + lane;
    uint32_t a[8];
    for (int kk = 0; kk < 8; ++kk) a[kk] = __float_as_uint(A[m * 8 + kk]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(tb + ((uint32_t)(32 * warp) << 16) + 64), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]),
                   "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]) : "memory");
    const uint32_t s = __float_as_uint(-999.0f);
    for (int c = 0; c < 64; c += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};"
                   ::"r"(tb + ((uint32_t)(32 * warp) << 16) + c), "r"(s) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(tb), "r"(tb + 64), "l"(mk(su32(sb))), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  __syncwarp();
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < 64; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tb + ((uint32_t)(32 * warp) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[(32 * warp + lane) * 64 + c] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(128) : "memory");
}

int main() {
  float hA[128 * 8], hB[64 * 8], hD[128 * 64];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7 + i / 8 * 3) % 13) - 6 + 0.25f * (i / 8);
  for (int i = 0; i < 64 * 8; ++i) hB[i] = (float)((i * 5) % 11) - 5;
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((64u >> 4) << 24);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<1, 128, 16384>>>(A, B, D, idesc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  printf("M=64 probe: %s\n", cudaGetErrorString(e));
  for (int L = 0; L < 128; L += 1) {
    int written = 0, match_m = -1, nmatch = 0;
    for (int n = 0; n < 64; ++n) written += hD[L * 64 + n] != -999.0f;
    if (!written) continue;
    for (int m = 0; m < 128; ++m) {
      bool all = true;
      for (int n = 0; n < 64 && all; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 8; ++kk) ref += (double)hA[m * 8 + kk] * hB[n * 8 + kk];
        all = fabs(ref - hD[L * 64 + n]) < 1e-3;
      }
      if (all) { match_m = m; ++nmatch; }
    }
    if (L % 8 == 0 || match_m != L) printf("  D lane %3d: %d cols written, = A row %d (%d matches)\n", L, written, match_m, nmatch);
  }
}
