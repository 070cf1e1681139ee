// Minimal tcgen05.mma kind::tf32 test: D(128x64) = A(128x8) * B(8x64).
// variant 0: A K-major SW128, B K-major SW128; variant 1: A MN-major SW64 (16-elem groups)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t mk(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)(lay & 7) << 61);
}

__global__ void k(int variant, const float* A, const float* B, float* D, uint32_t idesc, uint32_t lboA, uint32_t sboA) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  unsigned char* sa = base;           // 16 KiB
  unsigned char* sb = base + 16384;   // 8 KiB
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  // fill A (128 x 32 floats, only k < 8 nonzero used) and B (64 x 32)
  for (int e = threadIdx.x; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, kk = e % 32;
    const float v = kk < 8 ? A[m * 8 + kk] : 0.f;
    uint32_t off;
    if (variant == 0) off = m * 128 + ((((kk >> 2) ^ (m & 7))) << 4) + (kk & 3) * 4;
    else if (variant == 2) {
      const int g = m / 32, ee = m % 32, c = kk;
      const uint32_t raw = g * 4096 + c * 128 + ee * 4;   // LBO = 4096 (32 K-rows * 128B)
      off = raw ^ (((raw >> 7) & 7) << 4);
    } else {  // MN-major SW64: (h = m/16, c = kk, w = m%16): h*2048 + c*64 + swz
      const int hh = m / 16, ww = m % 16, c = kk;
      const uint32_t raw = hh * 2048 + c * 64 + ww * 4;
      off = raw ^ (((raw >> 7) & 3) << 4);
    }
    *reinterpret_cast<float*>(sa + off) = v;
  }
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int n = e / 32, kk = e % 32;
    const float v = kk < 8 ? B[n * 8 + kk] : 0.f;
    const uint32_t off = n * 128 + ((((kk >> 2) ^ (n & 7))) << 4) + (kk & 3) * 4;
    *reinterpret_cast<float*>(sb + off) = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(64) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint64_t da = variant == 0 ? mk(su32(sa), 16, 1024, 2)
                      : variant == 2 ? mk(su32(sa), lboA, sboA, 2) : mk(su32(sa), lboA, sboA, 4);
    const uint64_t db = mk(su32(sb), 16, 1024, 2);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tb), "l"(da), "l"(db), "r"(idesc), "r"(0u) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  __syncwarp();
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < 64; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tb + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[(32 * warp + (threadIdx.x & 31)) * 64 + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(64) : "memory");
}

int main(int argc, char** argv) {
  const int variant = atoi(argv[1]);
  const uint32_t lbo = argc > 2 ? atoi(argv[2]) : 2048, sbo = argc > 3 ? atoi(argv[3]) : 512;
  float hA[128 * 8], hB[64 * 8], hD[128 * 64];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 13) - 6;
  for (int i = 0; i < 64 * 8; ++i) hB[i] = (float)((i * 5) % 11) - 5;
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(D, 0, sizeof hD);
  const uint32_t amaj = variant == 0 ? 0 : 1;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (amaj << 15) | (0u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<<<1, 128, 32768>>>(variant, A, B, D, idesc, lbo, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0; int bad = 0;
  for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n) {
    double ref = 0; for (int kk = 0; kk < 8; ++kk) ref += (double)hA[m * 8 + kk] * hB[n * 8 + kk];
    const double d = fabs(ref - hD[m * 64 + n]); maxerr = d > maxerr ? d : maxerr; maxref = fabs(ref) > maxref ? fabs(ref) : maxref;
    if (d > 1e-3 && bad++ < 3) printf("  m=%d n=%d got %g want %g\n", m, n, hD[m * 64 + n], ref);
  }
  printf("variant %d lbo %u sbo %u: %s maxerr %g (maxref %g) bad %d\n", variant, lbo, sbo, cudaGetErrorString(e), maxerr, maxref, bad);
}
