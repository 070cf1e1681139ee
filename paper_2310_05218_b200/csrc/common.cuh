// Shared helpers for the slideconv_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/slideconv_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "slideconv_b200 is built for sm_100a only"
#endif

namespace sc {

// ---------------------------------------------------------------- status
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SC_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return sc::cuda_fail(_e, #call); \
  } while (0)

#define SC_LAUNCH_CHECK(what)                                    \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return sc::cuda_fail(_e, what);       \
  } while (0)

constexpr int kNumSMs = 148;

constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & (kMaxDevices - 1);
}

// SM count of the current device (cached per device)
inline int sm_count() {
  static int n[kMaxDevices] = {};
  const int dev = current_device();
  if (n[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = kNumSMs;
    n[dev] = v;
  }
  return n[dev];
}

// Stream-ordered scratch for the few paths that need one (weight packing,
// split partial planes, exact-mode passes).  The device's default memory
// pool keeps up to 1 GiB of freed blocks (release threshold raised once per
// device): with
// the default threshold of 0 every synchronisation returns them to the
// driver and the next call pays a fresh allocation (~tens of us).
inline cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static bool pool_set[kMaxDevices] = {};
  const int dev = current_device();
  if (!pool_set[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 1ull << 30;  // keep up to 1 GiB (large exact-mode scratch is released)
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_set[dev] = true;
  }
  return cudaMallocAsync(p, bytes, st);
}

// Raise a kernel's dynamic shared-memory limit once per device
// (cudaFuncSetAttribute applies to the current device only); `done` is the
// caller's per-kernel bit set of devices already configured.
template <typename F>
cudaError_t set_smem_limit_once(F* func, size_t bytes, uint64_t* done, int carveout = -1) {
  const uint64_t bit = 1ull << current_device();
  if (__atomic_load_n(done, __ATOMIC_ACQUIRE) & bit) return cudaSuccess;
  cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  // carveout (percent of the unified L1 / shared array given to shared
  // memory): the driver otherwise may pick a configuration that fits only
  // one CTA per SM (a 100 KB carveout for two 85 KB CTAs, say)
  if (e == cudaSuccess && carveout >= 0)
    e = cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  if (e == cudaSuccess) __atomic_fetch_or(done, bit, __ATOMIC_RELEASE);
  return e;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// once its predecessor in the stream has triggered (griddepcontrol.
// launch_dependents) and must execute griddepcontrol.wait before touching
// memory the predecessor may read or write.  Kernels launched this way
// trigger their own dependents early, so back-to-back calls overlap launch
// latency and prologue with the predecessor's tail.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool off = [] {
    const char* e = getenv("SC_PDL");  // SC_PDL=0: plain stream order (A/B knob)
    return e && e[0] == '0';
  }();
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------ arithmetic
// np.maximum(a, b): NaN if either operand is NaN, b on ties (so +0/-0 ties
// return the later operand); pooling.py:70,75 with numpy's ufunc semantics.
__device__ __forceinline__ float np_max(float a, float b) {
  return (a > b || a != a) ? a : b;
}

// Reference tap update, reference.py:22: acc + (f * x), two roundings.
template <bool kExact>
__device__ __forceinline__ float mac(float acc, float f, float x) {
  if constexpr (kExact) {
    return __fadd_rn(acc, __fmul_rn(f, x));
  } else {
    return fmaf(f, x, acc);
  }
}

template <bool kExact>
__device__ __forceinline__ double mac(double acc, double f, double x) {
  if constexpr (kExact) {
    return __dadd_rn(acc, __dmul_rn(f, x));
  } else {
    return fma(f, x, acc);
  }
}

__device__ __forceinline__ float max_nan(float a, float b) {
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

// Correctly rounded a / k from the correctly rounded reciprocal r = RN(1/k):
// q = RN(a r) is within an ulp of a/k, the FMA residual a - k q is exact, and
// RN(q + r (a - k q)) is RN(a/k) (Markstein's theorem).  Tiny or non-finite
// numerators take the IEEE division (underflow voids the theorem).
__device__ __forceinline__ float div_by_k_fast(float a, float k, float r) {
  const float q = a * r;
  const float e = fmaf(-k, q, a);
  return fmaf(e, r, q);
}

// true when the numerator is outside the range the theorem covers
__device__ __forceinline__ bool div_needs_ieee(float a) {
  return !(fabsf(a) >= 1e-30f && fabsf(a) < 3.0e38f);
}

// In-place v[j] /= k for N values: branch-free reciprocal path, one warp
// vote, and the IEEE division only for the (rare) flagged values.
template <int N>
__device__ __forceinline__ void div_all_by_k(float (&v)[N], float k, float r) {
  bool slow = false;
  float a[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    a[j] = v[j];
    slow |= div_needs_ieee(v[j]);
    v[j] = div_by_k_fast(v[j], k, r);
  }
  if (__any_sync(0xffffffffu, slow)) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (div_needs_ieee(a[j])) v[j] = __fdiv_rn(a[j], k);
  }
}

// Output stores of the FP32-bound conv kernels.  A lane stores C
// consecutive outputs per row.  The column range check is hoisted out of the
// row loop into a store mode computed from warp-uniform values only (kernel
// parameters and the warp's first column), so the per-row test compiles to a
// uniform branch: a divergent per-row branch splits the unrolled row bodies
// into separate scheduling regions, a copy of the row loop per mode thrashes
// the instruction cache when warps of one SM run different copies, and
// 64-bit per-column compares with predicated stores cost ~25 instructions
// per row (ISETP.EX pairs and an R2UR descriptor copy per predicated STG).
//   pairs:     the warp's 32 C columns are in range and the row pitch and
//              base are 8-byte aligned -> C / 2 STG.64;
//   otherwise: the lane's count of in-range columns, predicated STG.32.
struct OutCols {
  bool pairs;  // warp-uniform (broadcast by a shuffle so the compiler knows it)
  int nv;      // this lane's in-range columns (used when !pairs)
};
template <int C>
__device__ __forceinline__ OutCols out_cols(const float* y, int64_t ow, int64_t wcol0,
                                            int64_t gcol) {
  const bool pairs = C % 2 == 0 && wcol0 + 32 * C <= ow &&
                     ((reinterpret_cast<uintptr_t>(y) | (uintptr_t)(ow * 4)) & 7) == 0;
  return {__shfl_sync(0xffffffffu, (int)pairs, 0) != 0,
          (int)max((int64_t)0, min((int64_t)C, ow - gcol))};
}

template <int C>
__device__ __forceinline__ void store_cols(float* p, const OutCols& m, const float (&v)[C]) {
  if (m.pairs) {
#pragma unroll
    for (int c = 0; c < C; c += 2) *reinterpret_cast<float2*>(p + c) = make_float2(v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c)
      if (c < m.nv) p[c] = v[c];
  }
}

// The pair (p[0], p[1]) of a shared-memory row at an odd float offset, as a
// register pair for packed FFMA2.  Volatile scalar loads: ptxas merges plain
// ones with the neighbouring aligned vector loads and then rebuilds the pair
// with moves at every use.
__device__ __forceinline__ float2 lds_pair_unaligned(const float* p) {
  float a, b;
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(a) : "r"(
      static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(b) : "r"(
      static_cast<uint32_t>(__cvta_generic_to_shared(p + 1))));
  return make_float2(a, b);
}

// ------------------------------------------------------ mbarrier / TMA PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Non-blocking probe: returns at once (mbarrier.try_wait may suspend the
// thread for a while before reporting an incomplete phase).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Spin on the non-blocking probe (for latency-critical waiters whose phase is
// usually already complete).
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  while (!mbar_test_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// For producer / bookkeeping threads that run ahead of the math warps: back
// off with __nanosleep between probes so the spin loop does not steal issue
// slots from the FMA / tensor warps sharing the SM sub-partition (ncu on the
// 7x7 conv: 490 M SYNCS + 514 M BRA + 486 M YIELD vs 828 M FFMA2 executed).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity,
                                                uint32_t ns0 = 32, uint32_t ns_max = 512) {
  uint32_t ns = ns0;
  while (!mbar_try_wait(bar, parity)) {
    __nanosleep(ns);
    ns = ns < ns_max ? ns * 2 : ns_max;
  }
}

// 4-byte cp.async global -> shared (zero-fill when pred is false)
__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool pred) {
  const int n = pred ? 4 : 0;  // zero-fill when predicated off
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 3-D tiled TMA load global -> shared, completion on an mbarrier.
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

}  // namespace sc
