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
constexpr int kNC = 2 * kN;                     // MMA N: [B_hi | B_lo] concatenated
constexpr int kKB = 32;                         // input channels per k-block
constexpr int kLoadStages = 3;                  // TMA ring: A box + B hi/lo
constexpr int kSplitStages = 2;                 // split ring: A hi/lo (K-major)
constexpr int kABytes = kM * kKB * 4;           // 16 KiB
constexpr int kBBytes = kNC * kKB * 4;          // 16 KiB: rows 0..63 hi, 64..127 lo
constexpr int kLoadBytes = kABytes + kBBytes;       // [A box (MN-major SW64)][B_hi ; B_lo]
// A hi / lo live in TMEM (TS-form MMA): per split stage 32 + 32 columns
constexpr int kTmemD = 0;                        // D: columns [0, 128)
constexpr int kTmemA = kNC;                      // A stages: columns [128, 256)
constexpr int kTmemCols = 256;
constexpr int kSplitWarps = 8;                  // split workers, then epilogue
constexpr int kThreads = 64 + 32 * kSplitWarps;

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

// kind::tf32, D f32, A K-major, B K-major, M = 128, N = 128 ([B_hi | B_lo]).  (An MN-major
// tf32 A operand returned all-zero products on sm_100a in
// tools/micro/umma_probe.cu, so the split workers transpose A to K-major.)
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                            ((uint32_t)(kNC >> 3) << 17) | ((uint32_t)(kM >> 4) << 24);

// A from TMEM (lane = output pixel, column = k), B from shared memory
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(kIdesc), "r"(accumulate)
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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float a) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(a));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(kThreads, 2)
    nchw3x3_tc_kernel(const __grid_constant__ CUtensorMap tmx,
                      const __grid_constant__ CUtensorMap tmw, const float* __restrict__ x,
                      float* __restrict__ y, int cin, int h, int w, int cout) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kLoadStages], empty_bar[kLoadStages];
  __shared__ __align__(8) uint64_t split_bar[kSplitStages], split_free[kSplitStages];
  __shared__ __align__(8) uint64_t tmem_full;
  __shared__ uint32_t tmem_base_sh;
  unsigned char* load_ring = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

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
      mbar_init(&split_bar[s], kSplitWarps);
      mbar_init(&split_free[s], 1);
    }
    mbar_init(&tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: D (128 lanes x 128 fp32 columns) + two A hi/lo stages
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmw);
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
        // the split workers apply the tap's column offset and supply the halo
        // column.  Rows (dim 2) may start at -1: TMA zero-fills them.
        tma_load_4d(st, &tmx, &full_bar[s], w0, ci0, h0 + dj, n);
        tma_load_3d(st + kABytes, &tmw, &full_bar[s], ci0, 2 * co0, tap);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int ls = kb % kLoadStages, ss = kb % kSplitStages;
        mbar_wait(&split_bar[ss], (kb / kSplitStages) & 1);  // implies the TMA landed
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a_hi = tmem + kTmemA + ss * 64;
        const uint32_t a_lo = a_hi + 32;
        // B: K-major SW128 (128-byte rows of 32 channels, SBO = 1 KiB between
        // 8-row groups); a k-step of 8 tf32 advances the start by 32 B
        const uint64_t dbc = make_desc(smem_u32(load_ring + ls * kLoadBytes) + kABytes, 16, 1024, 2);
#pragma unroll
        for (int ks = 0; ks < kKB / 8; ++ks) {
          // D[:, 0:64] += A * B_hi, D[:, 64:128] += A * B_lo, A = A_lo then A_hi
          // (4-term split product; the epilogue adds the two halves)
          mma_tf32_ts(tmem + kTmemD, a_lo + 8 * ks, dbc + 2 * ks, (kb | ks) ? 1u : 0u);
          mma_tf32_ts(tmem + kTmemD, a_hi + 8 * ks, dbc + 2 * ks, 1u);
        }
        umma_commit(&empty_bar[ls]);    // A box + B slot free once these retire
        umma_commit(&split_free[ss]);   // TMEM A stage free
      }
      umma_commit(&tmem_full);
    }
  } else {
    // ------------------------------------------------ split workers (8 warps)
    // warp -> TMEM lane quarter q = warp % 4 (pixels m = 32q + lane) and half
    // of the 32 channels of a k-block; each thread splits its pixel's 16
    // channels into tf32 hi / lo and stores them to TMEM (tcgen05.st)
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int m = 32 * q + lane;
    const int hh = m / kTileW, e = m % kTileW;
    const int c_lo = 16 * half;
    float halo_next[16];
    auto fetch_halo = [&](int kb2, float (&hv)[16]) {
#pragma unroll
      for (int c = 0; c < 16; ++c) hv[c] = 0.0f;
      if (kb2 >= kblocks) return;
      const int tap2 = kb2 / cchunks, c2 = (kb2 % cchunks) * kKB;
      const int dj2 = tap2 / 3 - 1, di2 = tap2 % 3 - 1;
      if (!((di2 < 0 && e == 0) || (di2 > 0 && e == kTileW - 1))) return;
      const int gw = di2 < 0 ? w0 - 1 : w0 + kTileW, gh = h0 + dj2 + hh;
      if (gw < 0 || gw >= w || gh < 0 || gh >= h) return;
      const float* src = x + (((int64_t)n * cin + c2 + c_lo) * h + gh) * w + gw;
#pragma unroll
      for (int c = 0; c < 16; ++c) hv[c] = __ldg(src + (int64_t)c * h * w);
    };
    fetch_halo(0, halo_next);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int ls = kb % kLoadStages, ss = kb % kSplitStages;
      const int tap = kb / cchunks;
      const int di = tap % 3 - 1;
      float halo[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) halo[c] = halo_next[c];
      fetch_halo(kb + 1, halo_next);
      mbar_wait(&full_bar[ls], (kb / kLoadStages) & 1);
      if (kb >= kSplitStages) mbar_wait(&split_free[ss], ((kb / kSplitStages) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* box = load_ring + ls * kLoadBytes;  // MN-major SW64
      const int ee = e + di;
      const bool edge = ee < 0 || ee >= kTileW;
      const int eec = edge ? 0 : ee;
      uint32_t vh[16], vl[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int cc = c_lo + c;
        // box element (hh, cc, eec): 64-byte row (hh, cc), SW64 chunk swizzle
        const int off = hh * (kKB * 64) + cc * 64 + ((((eec >> 2) ^ ((cc >> 1) & 3))) << 4) +
                        ((eec & 3) << 2);
        const float f = edge ? halo[c] : *reinterpret_cast<const float*>(box + off);
        const float hv = tf32_hi(f);
        vh[c] = __float_as_uint(hv);
        vl[c] = __float_as_uint(f - hv);
      }
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + kTmemA + ss * 64 + c_lo;
      tmem_st16(ta, vh);
      tmem_st16(ta + 32, vl);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&split_bar[ss]);
    }
    // ------------------------------------------------ epilogue
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int ch0 = half * 32;
    uint32_t r[32], rl[32];
    const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + kTmemD + ch0;
    tmem_ld32(taddr, r);
    tmem_ld32(taddr + kN, rl);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int oh = h0 + hh, ow = w0 + e;
    if (oh < h && ow < w) {
      float* yp = y + (((int64_t)n * cout + co0 + ch0) * h + oh) * w + ow;
      const int64_t plane = (int64_t)h * w;
#pragma unroll
      for (int c = 0; c < 32; ++c) yp[c * plane] = __uint_as_float(r[c]) + __uint_as_float(rl[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// w[co][ci][3][3] -> [tap][2*cout][ci]: for every 64-channel tile, rows
// 0..63 are the tf32 hi parts, rows 64..127 the lo parts (K-major B operand
// of one N = 128 MMA per tap)
__global__ void split_weights_kernel(const float* __restrict__ w, float* __restrict__ out,
                                     int cin, int cout) {
  const int total = 9 * cout * cin;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int ci = e % cin, co = (e / cin) % cout, tap = e / (cin * cout);
    const float v = w[((int64_t)co * cin + ci) * 9 + tap];
    const float hv = tf32_hi(v);
    const int tile = co / kN, cl = co % kN;
    float* base = out + ((int64_t)tap * 2 * cout + (int64_t)tile * kNC) * cin;
    base[(int64_t)cl * cin + ci] = hv;
    base[(int64_t)(kN + cl) * cin + ci] = v - hv;
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
  CUtensorMap mx;
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
  const size_t wbytes = (size_t)9 * 2 * cout * cin * sizeof(float);
  SC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wsplit), wbytes, st));
  split_weights_kernel<<<(unsigned)std::min<int64_t>(1024, (9 * cout * cin + 255) / 256), 256, 0,
                         st>>>(wt, wsplit, (int)cin, (int)cout);
  SC_LAUNCH_CHECK("split_weights_kernel");
  CUtensorMap mw;
  {
    cuuint64_t dims[3] = {(cuuint64_t)cin, (cuuint64_t)(2 * cout), 9};
    cuuint64_t strides[2] = {(cuuint64_t)(cin * 4), (cuuint64_t)(2 * cin * cout * 4)};
    cuuint32_t box[3] = {kKB, kNC, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, wsplit, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "nchw tc: weight tensor map failed");
  }
  const size_t smem = 1024 + (size_t)kLoadStages * kLoadBytes;
  static bool attr = false;
  if (!attr) {
    SC_CUDA(cudaFuncSetAttribute(nchw3x3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr = true;
  }
  dim3 grid((unsigned)((w + kTileW - 1) / kTileW), (unsigned)((h + kTileH - 1) / kTileH),
            (unsigned)(nb * (cout / kN)));
  nchw3x3_tc_kernel<<<grid, kThreads, smem, st>>>(mx, mw, x, y, (int)cin, (int)h, (int)w,
                                                   (int)cout);
  SC_LAUNCH_CHECK("nchw3x3_tc_kernel");
  SC_CUDA(cudaFreeAsync(wsplit, st));
  return SC_OK;
}

}  // namespace sc
