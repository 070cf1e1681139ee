// Multi-channel NCHW 3x3 / pad 1 convolution on the 5th-generation tensor
// cores (tcgen05, kind::tf32) with 3xTF32 split precision.
//
// BASELINE config 4 (N16 Cin64 Cout64 112x112) has ~144 flop/byte: it is
// FP32-pipe bound on CUDA cores (ncu: nchw3x3_kernel FMA pipe 55 %, 0.45 ms;
// cuDNN FP32 0.17 ms), so the contraction moves to the tensor cores as an
// implicit GEMM per filter tap:
//     out[p, co] += sum_ci  X[ci, p + (j-1, i-1)] * W[co, ci, j, i]
// * A = shifted input window, M = 128 output pixels (8 rows x 16 cols), K = 32
//   channels per k-block, loaded straight from the NCHW tensor by a 4-D TMA
//   box {16 w, 32 c, 8 h, 1 n} whose (w, h) origin is shifted by the tap:
//   out-of-bounds rows / columns are zero-filled by TMA = the zero padding.
//   In shared memory this is an MN-major, 64-byte-swizzled UMMA operand.
// * B = weights of the tap, N = 64 output channels, K-major 128-byte swizzle,
//   pre-split on the device into tf32 hi / lo parts ([tap][co][ci]).
// * 3xTF32: D += A_hi B_hi + A_hi B_lo + A_lo B_hi with A_hi = rna_tf32(A),
//   A_lo = A - A_hi (split in shared memory by 4 worker warps), fp32
//   accumulation in TMEM (128 lanes x 64 columns).  Error ~2^-21 per product:
//   far inside 1e-5 * k * sqrt(Cin) (plain TF32 would not be).
// * Warp roles: warp 0 TMA producer, warp 1 TMEM owner + single-thread MMA
//   issuer, warps 2..5 split workers then the epilogue (tcgen05.ld -> NCHW
//   stores).  A 4-deep TMA ring (A box + B hi/lo) and a 2-deep split ring
//   (A hi/lo, K-major) with full / split / split_free / empty mbarriers; the
//   empty barriers are armed by tcgen05.commit so a slot is refilled as soon
//   as the MMAs that read it retire.
// * Measured (B200, config 4): 0.20 ms vs 0.455 ms for the FFMA kernel and
//   0.17 ms for cuDNN's FP32 algorithm.  The kernel is shared-memory-bandwidth
//   bound: per k-block TMA writes 32 KB, the split moves 48 KB and the 12
//   MMAs (N = Cout = 64 is small) read 72 KB of operands (~1.2 k cycles at
//   128 B/clk vs ~0.6 k cycles of MMA issue).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {

constexpr int kTileH = 8, kTileW = 16;         // M = 128 pixels
constexpr int kM = kTileH * kTileW;
constexpr int kN = 64;                          // output channels per CTA
constexpr int kKB = 32;                         // input channels per k-block
constexpr int kLoadStages = 4;                  // TMA ring: A box + B hi/lo
constexpr int kSplitStages = 2;                 // split ring: A hi/lo (K-major)
constexpr int kABytes = kM * kKB * 4;           // 16 KiB
constexpr int kBBytes = kN * kKB * 4;           // 8 KiB
constexpr int kLoadBytes = kABytes + 2 * kBBytes;   // [A box (MN-major SW64)][B_hi][B_lo]
constexpr int kSplitBytes = 2 * kABytes;            // [A_hi][A_lo] (K-major SW128)
constexpr int kThreads = 192;

__device__ __forceinline__ uint64_t make_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// kind::tf32, D f32, A K-major, B K-major, M = 128, N = 64.  (An MN-major
// tf32 A operand returned all-zero products on sm_100a in
// tools/micro/umma_probe.cu, so the split workers transpose A to K-major.)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                            ((uint32_t)(kN >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float a) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(kThreads, 1)
    nchw3x3_tc_kernel(const __grid_constant__ CUtensorMap tmx,
                      const __grid_constant__ CUtensorMap tmw_hi,
                      const __grid_constant__ CUtensorMap tmw_lo, const float* __restrict__ x,
                      float* __restrict__ y, int cin, int h, int w, int cout) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kLoadStages], empty_bar[kLoadStages];
  __shared__ __align__(8) uint64_t split_bar[kSplitStages], split_free[kSplitStages];
  __shared__ __align__(8) uint64_t tmem_full;
  __shared__ uint32_t tmem_base_sh;
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* load_ring = base;
  unsigned char* split_ring = base + kLoadStages * kLoadBytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w0 = blockIdx.x * kTileW, h0 = blockIdx.y * kTileH;
  const int co_tiles = cout / kN;
  const int n = blockIdx.z / co_tiles, co0 = (blockIdx.z % co_tiles) * kN;
  const int cchunks = cin / kKB;
  const int kblocks = 9 * cchunks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kLoadStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kSplitStages; ++s) {
      mbar_init(&split_bar[s], 4);
      mbar_init(&split_free[s], 1);
    }
    mbar_init(&tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: 128 lanes x 64 fp32 columns for the accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(kN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_d = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmw_hi);
      prefetch_tmap(&tmw_lo);
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % kLoadStages;
        if (kb >= kLoadStages) mbar_wait(&empty_bar[s], ((kb / kLoadStages) - 1) & 1);
        const int tap = kb / cchunks, ci0 = (kb % cchunks) * kKB;
        const int dj = tap / 3 - 1;
        unsigned char* st = load_ring + s * kLoadBytes;
        mbar_arrive_expect_tx(&full_bar[s], kLoadBytes);
        // The innermost TMA coordinate must be 16-byte aligned (measured on
        // sm_100a: an unaligned or negative w origin is an illegal
        // instruction), so every tap loads the aligned 16-column block at w0;
        // the split workers shift it by the tap's column offset and supply
        // the halo column.  Rows (dim 2) may start at -1: TMA zero-fills.
        tma_load_4d(st, &tmx, &full_bar[s], w0, ci0, h0 + dj, n);
        tma_load_3d(st + kABytes, &tmw_hi, &full_bar[s], ci0, co0, tap);
        tma_load_3d(st + kABytes + kBBytes, &tmw_lo, &full_bar[s], ci0, co0, tap);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int ls = kb % kLoadStages, ss = kb % kSplitStages;
        mbar_wait(&split_bar[ss], (kb / kSplitStages) & 1);  // implies the TMA landed
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // K-major SW128 descriptors (128-byte rows of 32 channels, SBO = 1 KiB
        // between 8-row groups); a k-step of 8 tf32 advances the start by 32 B
        // = 2 in the descriptor's 16-byte address units
        const uint64_t dah = make_desc(smem_u32(split_ring + ss * kSplitBytes), 16, 1024, 2);
        const uint64_t dal = dah + (kABytes >> 4);
        const uint64_t dbh = make_desc(smem_u32(load_ring + ls * kLoadBytes) + kABytes, 16, 1024, 2);
        const uint64_t dbl = dbh + (kBBytes >> 4);
#pragma unroll
        for (int ks = 0; ks < kKB / 8; ++ks) {
          const uint64_t o = (uint64_t)(2 * ks);
          mma_tf32(tmem_d, dal + o, dbh + o, (kb | ks) ? 1u : 0u);  // small terms first
          mma_tf32(tmem_d, dah + o, dbl + o, 1u);
          mma_tf32(tmem_d, dah + o, dbh + o, 1u);
        }
        umma_commit(&empty_bar[ls]);    // B slot (and its A box) free once these retire
        umma_commit(&split_free[ss]);   // A hi / lo slot free
      }
      umma_commit(&tmem_full);
    }
  } else {
    // ------------------------------------------------ split workers (128 thr)
    // thread t: pixel row hh = t / 16 of the tile, channel pair 2*(t % 16)
    const int t = threadIdx.x - 64;
    const int hh = t >> 4, cp = (t & 15) * 2;
    // halo column of the shifted taps (the TMA block is aligned at w0): loaded
    // one k-block ahead so the global-load latency hides behind the MMAs
    auto fetch_halo = [&](int kb2, float (&hv)[2]) {
      hv[0] = hv[1] = 0.0f;
      if (kb2 >= kblocks) return;
      const int tap2 = kb2 / cchunks, c2 = (kb2 % cchunks) * kKB;
      const int dj2 = tap2 / 3 - 1, di2 = tap2 % 3 - 1;
      if (di2 == 0) return;
      const int gw = di2 < 0 ? w0 - 1 : w0 + kTileW, gh = h0 + dj2 + hh;
      if (gw >= 0 && gw < w && gh >= 0 && gh < h) {
        const float* src = x + (((int64_t)n * cin + c2 + cp) * h + gh) * w + gw;
        hv[0] = __ldg(src);
        hv[1] = __ldg(src + (int64_t)h * w);
      }
    };
    float halo_next[2];
    fetch_halo(0, halo_next);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int ls = kb % kLoadStages, ss = kb % kSplitStages;
      const int tap = kb / cchunks;
      const int di = tap % 3 - 1;
      float halo[2] = {halo_next[0], halo_next[1]};
      fetch_halo(kb + 1, halo_next);
      mbar_wait(&full_bar[ls], (kb / kLoadStages) & 1);
      if (kb >= kSplitStages) mbar_wait(&split_free[ss], ((kb / kSplitStages) - 1) & 1);
      const unsigned char* box = load_ring + ls * kLoadBytes;  // MN-major SW64
      unsigned char* ahi = split_ring + ss * kSplitBytes;      // K-major SW128
      unsigned char* alo = ahi + kABytes;
      float v[2][16];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int cc = cp + r;
        const int rbase = hh * (kKB * 64) + cc * 64;
        const int sw = (cc >> 1) & 3;  // SW64: 16-byte chunk ^= address bits [7,9)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = *reinterpret_cast<const float4*>(box + rbase + ((q ^ sw) << 4));
          v[r][4 * q] = f.x;
          v[r][4 * q + 1] = f.y;
          v[r][4 * q + 2] = f.z;
          v[r][4 * q + 3] = f.w;
        }
      }
      // transpose to K-major: pixel m = hh*16 + e owns a 128-byte row of 32
      // channels, 16-byte chunk (c/4) ^ (m & 7); this thread writes channels
      // (cp, cp+1) as one 8-byte store -- a warp fills two whole rows per step.
      // The tap's column offset DI is applied here: pixel e takes sample e+DI.
      auto emit = [&](auto di_tag) {
        constexpr int DI = decltype(di_tag)::value;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int src = e + DI;
          const bool edge = src < 0 || src > 15;
          const int sc_ = edge ? 0 : src;
          const float f0 = edge ? halo[0] : v[0][sc_];
          const float f1 = edge ? halo[1] : v[1][sc_];
          const int m = hh * kTileW + e;
          const int off = m * 128 + ((((cp >> 2) ^ (m & 7))) << 4) + ((cp & 3) << 2);
          const float h0v = tf32_hi(f0), h1v = tf32_hi(f1);
          *reinterpret_cast<float2*>(ahi + off) = make_float2(h0v, h1v);
          *reinterpret_cast<float2*>(alo + off) = make_float2(f0 - h0v, f1 - h1v);
        }
      };
      if (di < 0) emit(std::integral_constant<int, -1>{});
      else if (di > 0) emit(std::integral_constant<int, 1>{});
      else emit(std::integral_constant<int, 0>{});
      fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05.mma
      __syncwarp();
      if (lane == 0) mbar_arrive(&split_bar[ss]);
    }
    // ------------------------------------------------ epilogue
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    uint32_t r[64];
    const uint32_t taddr = tmem_d + ((uint32_t)(32 * ew) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
        "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
        "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]),
          "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),
          "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]),
          "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]),
          "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = 32 * ew + lane;  // output pixel of this TMEM lane
    const int oh = h0 + m / kTileW, ow = w0 + m % kTileW;
    if (oh < h && ow < w) {
      float* yp = y + (((int64_t)n * cout + co0) * h + oh) * w + ow;
      const int64_t plane = (int64_t)h * w;
#pragma unroll
      for (int c = 0; c < kN; ++c) yp[c * plane] = __uint_as_float(r[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "n"(kN)
                 : "memory");
  }
}

// w[co][ci][3][3] -> hi / lo [tap][co][ci] (K-major B operand per tap)
__global__ void split_weights_kernel(const float* __restrict__ w, float* __restrict__ hi,
                                     float* __restrict__ lo, int cin, int cout) {
  const int total = 9 * cout * cin;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int ci = e % cin, co = (e / cin) % cout, tap = e / (cin * cout);
    const float v = w[((int64_t)co * cin + ci) * 9 + tap];
    const float hv = tf32_hi(v);
    hi[e] = hv;
    lo[e] = v - hv;
  }
}

}  // namespace

// Returns SC_OK / an error if the tensor-core path ran, 1 if it does not apply.
int nchw3x3_tc(const float* x, int64_t nb, int64_t cin, int64_t h, int64_t w, const float* wt,
               int64_t cout, float* y, cudaStream_t st) {
  if (cin % kKB != 0 || cout % kN != 0 || w % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      nb * (cout / kN) > 65535 || h > 65535 * kTileH || cin * h * w >= ((int64_t)1 << 31))
    return 1;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap mx, mwh, mwl;
  {
    // dims (w, c, h, n) -- permuted so channels sit between w and h in the box
    cuuint64_t dims[4] = {(cuuint64_t)w, (cuuint64_t)cin, (cuuint64_t)h, (cuuint64_t)nb};
    cuuint64_t strides[3] = {(cuuint64_t)(h * w * 4), (cuuint64_t)(w * 4),
                             (cuuint64_t)(cin * h * w * 4)};
    cuuint32_t box[4] = {kTileW, kKB, kTileH, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "nchw tc: x tensor map failed");
  }
  float* wsplit = nullptr;
  const size_t wbytes = (size_t)9 * cout * cin * sizeof(float);
  SC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wsplit), 2 * wbytes, st));
  float* whi = wsplit;
  float* wlo = wsplit + (size_t)9 * cout * cin;
  split_weights_kernel<<<(unsigned)std::min<int64_t>(1024, (9 * cout * cin + 255) / 256), 256, 0,
                         st>>>(wt, whi, wlo, (int)cin, (int)cout);
  SC_LAUNCH_CHECK("split_weights_kernel");
  for (int i = 0; i < 2; ++i) {
    cuuint64_t dims[3] = {(cuuint64_t)cin, (cuuint64_t)cout, 9};
    cuuint64_t strides[2] = {(cuuint64_t)(cin * 4), (cuuint64_t)(cin * cout * 4)};
    cuuint32_t box[3] = {kKB, kN, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(i ? &mwl : &mwh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, i ? wlo : whi, dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "nchw tc: weight tensor map failed");
  }
  const size_t smem = 1024 + (size_t)kLoadStages * kLoadBytes + (size_t)kSplitStages * kSplitBytes;
  static bool attr = false;
  if (!attr) {
    SC_CUDA(cudaFuncSetAttribute(nchw3x3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)((w + kTileW - 1) / kTileW), (unsigned)((h + kTileH - 1) / kTileH),
            (unsigned)(nb * (cout / kN)));
  nchw3x3_tc_kernel<<<grid, kThreads, smem, st>>>(mx, mwh, mwl, x, y, (int)cin, (int)h, (int)w,
                                                   (int)cout);
  SC_LAUNCH_CHECK("nchw3x3_tc_kernel");
  SC_CUDA(cudaFreeAsync(wsplit, st));
  return SC_OK;
}

}  // namespace sc
