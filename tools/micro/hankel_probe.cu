// Probe for the tensor-core single-channel conv (csrc/conv2d_mma.cu):
// tcgen05.mma kind::f16, SS form, A = a PLAIN bf16 row x read through a
// no-swizzle K-major descriptor with LBO = 16 B and SBO = 128 B, so that
// A[m][k] = x[8m + k] for k < 16 (core matrices overlap: the (m-group, k-half 1)
// matrix is the (m-group, k-half 0) matrix shifted by one 16-byte row).
// B = [N x 16] bf16, no-swizzle K-major (LBO 128, SBO 256).
//   ./hankel_probe check <N>        -> D == sum_k x[8m+k] B[n][k] ?
//   ./hankel_probe rate <N> <iters> -> cycles per MMA (3 back-to-back per iter)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t mk(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)(lay & 7) << 61);
}

__global__ void kcp(const __nv_bfloat16* X, const __nv_bfloat16* B, float* D, int N) {
  // tcgen05.cp.128x256b of the Hankel-described bf16 row into TMEM columns
  // 256..263, then a TS MMA with A from those columns
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(base);
  unsigned char* sb = base + 4096;
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 1040; e += blockDim.x) sx[e] = X[e];
  for (int e = threadIdx.x; e < N * 16; e += blockDim.x) {
    const int n = e / 16, kk = e % 16;
    const uint32_t off = (n / 8) * 256 + (kk / 8) * 128 + (n % 8) * 16 + (kk % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = B[n * 16 + kk];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tb)), "n"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t da = mk(su32(sx), 16, 128, 0);
    const uint64_t db = mk(su32(sb), 128, 256, 0);
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 256), "l"(da) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                 ::"r"(tb), "r"(tb + 256), "l"(db), "r"(idesc) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tb + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[(32 * warp + (threadIdx.x & 31)) * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(512) : "memory");
}

__global__ void k(const __nv_bfloat16* X, const __nv_bfloat16* B, float* D, int N, int iters,
                  long long* cyc, int issuers, int rot, int elect) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(base);           // 1040 bf16
  unsigned char* sb = base + 4096;                                      // N x 16 bf16
  __shared__ uint32_t tb;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 1040; e += blockDim.x) sx[e] = X[e];
  for (int e = threadIdx.x; e < N * 16; e += blockDim.x) {
    const int n = e / 16, kk = e % 16;
    const uint32_t off = (n / 8) * 256 + (kk / 8) * 128 + (n % 8) * 16 + (kk % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sb + off) = B[n * 16 + kk];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(issuers));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&tb)),
                 "n"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((128u >> 4) << 24);
  if (elect && warp < issuers) {
    // whole warp runs the loop (warp-uniform operands), one elected lane issues
    const uint64_t da = mk(su32(sx), 16, 128, 0);
    const uint64_t db = mk(su32(sb), 128, 256, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const uint32_t acc = (it | r) ? 1u : 0u;
        const uint32_t d = tb + (rot ? (uint32_t)(((it * 3 + r) * issuers + warp) % rot) * N : 0u);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc)
            : "memory");
      }
    }
    if ((threadIdx.x & 31) == 0) {
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              su32(&bar))
          : "memory");
    }
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], "
          "0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&bar))
          : "memory");
    if (threadIdx.x == 0) *cyc = clock64() - t0;
  }
  if (!elect && (threadIdx.x & 31) == 0 && warp < issuers) {
    const uint64_t da = mk(su32(sx), 16, 128, 0);
    const uint64_t db = mk(su32(sb), 128, 256, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int r = 0; r < 3; ++r) {
        const uint32_t acc = (it | r) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + (rot ? (uint32_t)(((it * 3 + r) * issuers + warp) % rot) * N : 0u)),
            "l"(da), "l"(db), "r"(idesc), "r"(iters == 1 ? 0u : acc)
            : "memory");
        if (iters == 1) break;
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
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
    if (warp == 0) *cyc = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                   : "=r"(r)
                   : "r"(tb + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[(32 * warp + (threadIdx.x & 31)) * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(256)
                 : "memory");
}

int main(int argc, char** argv) {
  const bool rate = argc > 1 && !strcmp(argv[1], "rate");
  const bool cp = argc > 1 && !strcmp(argv[1], "cpcheck");
  const int N = argc > 2 ? atoi(argv[2]) : 64;
  const int iters = rate ? (argc > 3 ? atoi(argv[3]) : 1000) : 1;
  const int issuers = argc > 4 ? atoi(argv[4]) : 1, rot = argc > 5 ? atoi(argv[5]) : 0;
  const int elect = argc > 6 ? atoi(argv[6]) : 0;
  static __nv_bfloat16 hx[1040], hb[256 * 16];
  static float fx[1040], fb[256 * 16], hd[128 * 256];
  for (int i = 0; i < 1040; ++i) {
    fx[i] = (float)((i * 7) % 13 - 6);
    hx[i] = __float2bfloat16(fx[i]);
  }
  for (int i = 0; i < N * 16; ++i) {
    fb[i] = (float)((i * 5) % 11 - 5);
    hb[i] = __float2bfloat16(fb[i]);
  }
  __nv_bfloat16 *X, *B;
  float* D;
  long long* cyc;
  cudaMalloc(&X, sizeof hx);
  cudaMalloc(&B, sizeof hb);
  cudaMalloc(&D, sizeof hd);
  cudaMalloc(&cyc, 8);
  cudaMemcpy(X, hx, sizeof hx, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb, sizeof hb, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  if (cp) {
    cudaFuncSetAttribute(kcp, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    kcp<<<1, 128, 32768>>>(X, B, D, N);
  } else {
    k<<<1, 128, 32768>>>(X, B, D, N, iters, cyc, issuers, rot, elect);
  }
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(hd, D, sizeof(float) * 128 * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  if (rate) {
    printf("elect %d N %d issuers %d rot %d: %s %lld cycles for %d MMAs = %.1f cycles/MMA (ideal %d)\n", elect, N, issuers, rot,
           cudaGetErrorString(e), c, 3 * iters * issuers, (double)c / (3 * iters * issuers), N / 2);
    return 0;
  }
  int bad = 0;
  double maxerr = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int kk = 0; kk < 16; ++kk) ref += (double)fx[8 * m + kk] * fb[n * 16 + kk];
      const double d = fabs(ref - hd[m * N + n]);
      maxerr = d > maxerr ? d : maxerr;
      if (d > 1e-3 && bad++ < 4) printf("  m=%d n=%d got %g want %g\n", m, n, hd[m * N + n], ref);
    }
  printf("%s N %d: %s maxerr %g bad %d\n", cp ? "cpcheck" : "check", N, cudaGetErrorString(e), maxerr, bad);
  return bad != 0;
}
