// Multi-channel NCHW 3x3 / pad 1 convolution, weights-stationary form, for
// Cin <= 64 (BASELINE config 4: N16 Cin64 Cout64 112x112).
//
// The pixel-stationary kernel (nchw_tc.cu) streams the weights through shared
// memory for every 128-pixel tile and copies the shifted pixel window into
// TMEM for every tap; both cost shared-memory bandwidth, which is what bounds
// it.  Here the roles flip:
//   * A (M = 128 TMEM lanes) = the 64 output channels' weights, split
//     w = w1 + w2 (bf16, as in nchw_tc.cu): in lane quarter q, lanes 0-15
//     hold w1 of channels 16q..16q+15 and lanes 16-31 their w2; K = 9 taps x
//     Cin in TMEM columns -- loaded ONCE per CTA and resident for all its rows
//     (288 columns).
//   * B (N = a row segment of Wt <= 112 pixels) = the input, split
//     x = x1 + x2, read by the MMA straight from shared memory: each input
//     row is converted once into a 128-byte-swizzled K-major [pixel][channel]
//     slot (the canonical UMMA layout, 8-pixel core groups 1024 B apart), and
//     the tap (dj, di) is just a descriptor at slot(r+dj) + (1+di) pixels.
//   * Issuer 1: D += A x x1 with M = 128 (w1 x1 and w2 x1).  Issuer 2:
//     D += A x x2 with M = 64, which reads / writes only lanes 0-15 of every
//     quarter (measured, tools/micro/umma_m64_probe.cu) = the w1 rows: w1 x2
//     at half the tensor time of an M = 128 product, and no wasted w2 x2.
//     The epilogue adds lanes j and j + 16 with one shuffle:
//     out = w1 x1 + w1 x2 + w2 x1, error ~2^-16 per product as in nchw_tc.cu.
//   * A CTA walks a segment of output rows of one image with a rolling window
//     of four split input-row slots: row r needs input rows r-1, r, r+1, and
//     row r+2 is converted while row r's MMAs run.  TMA brings each input row
//     (+ 4-column halo boxes when the tile is not the whole width) into a
//     2-deep fp32 staging ring.
// Warp roles: 0 TMA producer; 1 TMEM owner + x1 issuer; 2-9 split; 10-13
// epilogue (+ the one-time A load); 14 x2 issuer.  TMEM: D0 [0,112),
// D1 [112,224), A [224,512).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {
using namespace tc;

constexpr int kCo = 64;                       // output channels per CTA (M = 2 x 64)
constexpr int kMaxCin = 64;
constexpr int kMaxWt = 112;                   // pixels per row segment (N)
constexpr int kDStride = 112;                 // TMEM columns per accumulator
constexpr int kTmemA = 2 * kDStride;          // 224
constexpr int kTmemCols = 512;
constexpr int kSlots = 4;                     // split input-row ring
constexpr int kStages = 3;                    // fp32 staging ring
constexpr int kPixBytes = 128;                // one pixel's 64 bf16 channels
constexpr int kXRegion = ((kMaxWt + 2) * kPixBytes + 1023) / 1024 * 1024;  // 15 KiB
constexpr int kSlotBytes = 2 * kXRegion;                                     // x1 | x2
constexpr int kHaloW = 4;
constexpr int kStageBoxBytes = kMaxWt * kMaxCin * 4;                         // 28 KiB
constexpr int kStageBytes = kStageBoxBytes + 2 * kHaloW * kMaxCin * 4;      // + halos
constexpr size_t kSmem = 1024 + (size_t)kSlots * kSlotBytes + (size_t)kStages * kStageBytes;
constexpr int kSplitWarps = 8, kEpiWarps = 4;
constexpr int kIssuer2 = 2 + kSplitWarps + kEpiWarps;   // 14
constexpr int kThreads = 32 * (kIssuer2 + 1);
static_assert(kTmemA + 9 * kMaxCin / 2 <= kTmemCols, "TMEM budget");

// Optional timeline of every CTA (tools/micro/ws_trace.cu builds this file
// with -DSC_WS_TRACE): globaltimer stamps per CTA at fixed events.
#ifdef SC_WS_TRACE
__device__ unsigned long long g_ws_trace[160][13];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
  return t;
}
#define WS_TRACE(ev) g_ws_trace[blockIdx.x][ev] = gtime()
// global-clock stamps (%globaltimer, ns): conv CTA start / end, pack start
__device__ unsigned long long g_ws_gt[160][2], g_pack_gt[2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define WS_GT(ev) g_ws_gt[blockIdx.x][ev] = gtimer()
#else
#define WS_TRACE(ev) \
  do {               \
  } while (0)
#define WS_GT(ev) \
  do {            \
  } while (0)
#endif

struct WsArgs {
  int nb, cin, h, w, cout;
  int wt, col_tiles, seg_rows, segs;   // row segments of seg_rows rows per (image, column tile)
  int items_per_co, ctas_per_co;
};

template <int kKSteps>  // Cin / 16
__global__ void __launch_bounds__(kThreads, 1)
    nchw3x3_ws_kernel(const __grid_constant__ CUtensorMap tmx,
                      const __grid_constant__ CUtensorMap tmh, const uint32_t* __restrict__ apack,
                      float* __restrict__ y, const WsArgs args, const float* __restrict__ xraw,
                      const float* __restrict__ wraw) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (threadIdx.x == 0) {
    WS_TRACE(0);
    WS_GT(0);
  }
  __shared__ __align__(8) uint64_t stage_full[kStages], stage_empty[kStages];
  __shared__ __align__(8) uint64_t slot_full[kSlots], slot_free[kSlots];
  __shared__ __align__(8) uint64_t d_full[2], d_empty[2];
  __shared__ __align__(8) uint64_t a_ready;  // weights + zeroed D in TMEM
  __shared__ uint32_t tmem_base_sh;
  __shared__ float zero_word;
  unsigned char* slots = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* stages = slots + kSlots * kSlotBytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cin = args.cin, h = args.h, w = args.w, wt = args.wt;
  const int co_tiles = (args.cout + kCo - 1) / kCo;  // last tile zero-padded
  const int co_tile = blockIdx.x % co_tiles;
  const int cta_in_co = blockIdx.x / co_tiles;
  const int a_cols = 9 * cin / 2;
  constexpr int ksteps = kKSteps;
  const uint32_t idesc128 = idesc_bf16(128, wt), idesc64 = idesc_bf16(64, wt);

  // item -> (image, column tile, first row, row count)
  auto item_of = [&](int it, int& n, int& w0, int& r0, int& nr) {
    const int seg = it % args.segs;
    const int rest = it / args.segs;
    w0 = (rest % args.col_tiles) * wt;
    n = rest / args.col_tiles;
    r0 = seg * args.seg_rows;
    nr = min(args.seg_rows, h - r0);
  };

  if (threadIdx.x == 0) {
    zero_word = 0.0f;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&stage_full[s], 1);
      mbar_init(&stage_empty[s], kSplitWarps);
    }
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&slot_full[s], kSplitWarps);
      mbar_init(&slot_free[s], 2);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&d_full[s], 2);
      mbar_init(&d_empty[s], kEpiWarps);
    }
    mbar_init(&a_ready, kSplitWarps + kEpiWarps);
    fence_mbar_init();
  }
  if (warp == 1) {
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
  if (warp >= 2 && warp < kIssuer2) {
    // one-time setup by the 12 split + epilogue warps (3 per TMEM lane
    // quarter q = warp % 4): zero both accumulators and load this CTA's
    // weights (A) into TMEM.  Each warp owns a third of the A columns and
    // issues all its 16-byte loads before storing (one L2 round trip).
    const int q = warp & 3, third = (warp - 2) >> 2;  // 0..2
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    // launched as a programmatic dependent of the weight-packing kernel: only
    // this load needs its result; barrier setup, TMEM allocation and the
    // first input rows overlap it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (warp == 2 && lane == 0) WS_TRACE(12);
    if (third == 0) {
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
      for (int c = 0; c < kTmemA; c += 16) tmem_st16(lane_base + c, z);
    }
    const int chunks = a_cols / 16;                // 18 for Cin 64, 9 for Cin 32
    const int per = (chunks + 2) / 3;
    const int c_lo = third * per, c_hi = min(chunks, c_lo + per);
    // apack is [tile][16-column chunk][4 x 16 B][128 lanes]: a warp's load of
    // one 16-byte piece is 512 contiguous bytes
    const uint4* abase = reinterpret_cast<const uint4*>(apack) +
                         (size_t)co_tile * chunks * 4 * 128 + 32 * q + lane;
    uint4 buf[6][4];
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (c_lo + k < c_hi)
#pragma unroll
        for (int v = 0; v < 4; ++v) buf[k][v] = __ldg(abase + ((c_lo + k) * 4 + v) * 128);
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if (c_lo + k < c_hi) tmem_st16(lane_base + kTmemA + (c_lo + k) * 16,
                                     *reinterpret_cast<const uint32_t(*)[16]>(&buf[k][0]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&a_ready);
  }
  // no CTA-wide barrier here: the producer and split warps start on the
  // first input rows while the A load is in flight; only the issuers wait
  // inputs the bf16 split cannot carry (inf / NaN, |x| >= 2^127: x - bf16(x)
  // would be NaN or overflow), seen by the split warps
  // (tracked as the largest |x| bit pattern: >= 2^127, inf and NaN all
  // compare above 0x7f000000)
  uint32_t mag = 0;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer: input rows
    if (lane == 0) {
      prefetch_tmap(&tmx);
      prefetch_tmap(&tmh);
      int s = 0;
      for (int it = cta_in_co; it < args.items_per_co; it += args.ctas_per_co) {
        int n, w0, r0, nr;
        item_of(it, n, w0, r0, nr);
        // innermost TMA coordinates must be 16-byte aligned and in range, so
        // halo columns come from 4-wide boxes, skipped at the image edge
        const bool left = w0 > 0, right = w0 + wt < w;
        const uint32_t bytes = (uint32_t)(wt * cin * 4) + (left ? kHaloW * cin * 4 : 0) +
                               (right ? kHaloW * cin * 4 : 0);
        for (int rho = r0 - 1; rho <= r0 + nr; ++rho, ++s) {
          const int st = s % kStages;
          if (s >= kStages) mbar_wait(&stage_empty[st], ((s / kStages) - 1) & 1);
          unsigned char* dst = stages + st * kStageBytes;
          mbar_arrive_expect_tx(&stage_full[st], bytes);
          // rows -1 and h are outside the image: TMA zero-fills them (padding)
          if (s == 0) WS_TRACE(10);
          tma_load_4d(dst, &tmx, &stage_full[st], w0, rho, 0, n);
          if (s == 0) WS_TRACE(11);
          if (left)
            tma_load_4d(dst + kStageBoxBytes, &tmh, &stage_full[st], w0 - kHaloW, rho, 0, n);
          if (right)
            tma_load_4d(dst + kStageBoxBytes + kHaloW * cin * 4, &tmh, &stage_full[st], w0 + wt,
                        rho, 0, n);
        }
      }
    }
  } else if (warp == 1 || warp == kIssuer2) {
    // ------------------------------------------------ MMA issuers (x1 / x2)
    // whole warp, warp-uniform operands (shuffled), one elected lane issues
    const int part = __shfl_sync(0xffffffffu, warp == 1 ? 0 : 1, 0);  // which split product
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t idesc = part ? idesc64 : idesc128;
    const uint32_t slots_u = __shfl_sync(0xffffffffu, smem_u32(slots), 0) + part * kXRegion;
    mbar_wait(&a_ready, 0);
    if (part == 0 && threadIdx.x % 32 == 0) WS_TRACE(1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int s = 0, o = 0;
    for (int it = cta_in_co; it < args.items_per_co; it += args.ctas_per_co) {
      int n, w0, r0, nr;
      item_of(it, n, w0, r0, nr);
      const int base = s;  // seq of input row r0 - 1
      for (int rr = 0; rr < nr; ++rr, ++o) {
        const int acc = o & 1;
        if (o >= 2) mbar_wait(&d_empty[acc], ((o >> 1) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // input rows r-1, r, r+1 are waited for right before the taps that
        // read them, so at an item's first row the MMAs of row r-1 overlap
        // the split of rows r and r+1; later rows only wait for the new row
        // r+1 (rows r-1 and r were confirmed by the previous output row: a
        // slot cannot be refilled before this row frees it)
        const uint32_t d = tmem_u + acc * kDStride;
        const uint32_t a_base = tmem_u + kTmemA;
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
          const int sq = base + rr + dj;
          if (rr == 0 || dj == 2) {
            mbar_wait(&slot_full[sq % kSlots], (sq / kSlots) & 1);
            if (o == 0 && part == 0 && threadIdx.x % 32 == 0) {
              if (dj == 0) WS_TRACE(8);
              if (dj == 2) WS_TRACE(9);
            }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          }
          // tap column offset di: the window starts at slot pixel 1 + di.
          // Measured on sm_100a (tools/ws_debug.py): with this 128-byte
          // swizzled K-major B operand the MMA's first row is the one after
          // the descriptor start, so the start is one pixel earlier.  Fully
          // unrolled: operands are compile-time offsets (tap column di =
          // 128 B, k step = 32 B in the descriptor's 16-byte units).
          const uint64_t db = make_desc(slots_u + (sq % kSlots) * kSlotBytes, 16, 1024, 2);
#pragma unroll
          for (int di = 0; di < 3; ++di)
#pragma unroll
            for (int kk = 0; kk < ksteps; ++kk)
              mma_bf16_ts_elect(d, a_base + (dj * 3 + di) * (ksteps * 8) + kk * 8,
                                db + (uint64_t)(di * 8 + kk * 2), idesc);
        }
        if (part == 0 && threadIdx.x % 32 == 0) {
          if (o == 0) WS_TRACE(2);
          WS_TRACE(3);
        }
        umma_commit_elect(&d_full[acc]);
        // input row r-1 is not read by any later output row of this item
        umma_commit_elect(&slot_free[(base + rr) % kSlots]);
        if (rr == nr - 1) {
          umma_commit_elect(&slot_free[(base + rr + 1) % kSlots]);
          umma_commit_elect(&slot_free[(base + rr + 2) % kSlots]);
        }
        __syncwarp();
      }
      s = base + nr + 2;
    }
  } else if (warp < 2 + kSplitWarps) {
    // ------------------------------------------------ split warps
    const int tid = threadIdx.x - 64;  // 0 .. 255
    int s = 0;
    for (int it = cta_in_co; it < args.items_per_co; it += args.ctas_per_co) {
      int n, w0, r0, nr;
      item_of(it, n, w0, r0, nr);
      const bool left = w0 > 0, right = w0 + wt < w;
      for (int rho = r0 - 1; rho <= r0 + nr; ++rho, ++s) {
        const int st = s % kStages, sl = s % kSlots;
        mbar_wait(&stage_full[st], (s / kStages) & 1);
        if (s == 0 && tid == 0) WS_TRACE(7);
        if (s >= kSlots) mbar_wait(&slot_free[sl], ((s / kSlots) - 1) & 1);
        const unsigned char* src_box = stages + st * kStageBytes;
        unsigned char* xs = slots + sl * kSlotBytes;
        const int groups = cin / 8, pix = wt + 2;
        // unit = (8-channel group g, slot pixel p): p = 0 is column w0-1,
        // p = wt+1 is column w0+wt (halo or zero padding)
        for (int u = tid; u < groups * pix; u += 32 * kSplitWarps) {
          const int g = u / pix, p = u - g * pix;
          const unsigned char* src;
          int stride;
          if (p >= 1 && p <= wt) {
            src = src_box + (p - 1) * 4;
            stride = wt * 4;
          } else if (p == 0 ? left : right) {
            src = src_box + kStageBoxBytes + (p == 0 ? 3 * 4 : kHaloW * cin * 4);
            stride = kHaloW * 4;
          } else {
            src = reinterpret_cast<const unsigned char*>(&zero_word);
            stride = 0;
          }
          src += 8 * g * stride;
          uint4 w1, w2;
          uint32_t* p1 = &w1.x;
          uint32_t* p2 = &w2.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float f0 = *reinterpret_cast<const float*>(src + (2 * j) * stride);
            const float f1 = *reinterpret_cast<const float*>(src + (2 * j + 1) * stride);
            mag = max(mag, max(__float_as_uint(f0) & 0x7fffffffu, __float_as_uint(f1) & 0x7fffffffu));
            const uint32_t a1 = pack_bf16x2(f0, f1);  // channel 2j in the low half
            p1[j] = a1;
            p2[j] = pack_bf16x2(f0 - __uint_as_float(a1 << 16),
                                f1 - __uint_as_float(a1 & 0xffff0000u));
          }
          // 128-byte swizzle: 16-byte chunk g of pixel p at chunk g ^ (p & 7)
          const int off = p * kPixBytes + ((g ^ (p & 7)) << 4);
          *reinterpret_cast<uint4*>(xs + off) = w1;
          *reinterpret_cast<uint4*>(xs + kXRegion + off) = w2;
        }
        // generic-proxy smem writes -> read by the tensor core (async proxy)
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&slot_full[sl]);
          mbar_arrive(&stage_empty[st]);
        }
      }
    }
  } else if (warp < kIssuer2) {
    // ------------------------------------------------ epilogue (4 warps)
    const int q = warp & 3;
    const int c = 16 * q + (lane & 15);  // lanes j, j + 16: w1 / w2 rows of channel c
    uint32_t z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0u;
    const int64_t plane = (int64_t)h * w;
    int o = 0;
    for (int it = cta_in_co; it < args.items_per_co; it += args.ctas_per_co) {
      int n, w0, r0, nr;
      item_of(it, n, w0, r0, nr);
      const bool c_live = co_tile * kCo + c < args.cout;  // padded channels are dropped
      float* ybase = y + ((int64_t)n * args.cout + co_tile * kCo + c) * plane + w0;
      for (int rr = 0; rr < nr; ++rr, ++o) {
        const int acc = o & 1;
        mbar_wait_sleep(&d_full[acc], (o >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + acc * kDStride;
        float* yr = ybase + (int64_t)(r0 + rr) * w;
        for (int p0 = 0; p0 < wt; p0 += 16) {
          uint32_t v[16];
          tmem_ld16(taddr + p0, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          tmem_st16(taddr + p0, z);  // re-arm the accumulator
          float sum[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            sum[i] = __uint_as_float(v[i]) + __shfl_xor_sync(0xffffffffu, __uint_as_float(v[i]), 16);
          // lanes j and j + 16 both hold channel c: each stores half the pixels
          const bool odd = lane >= 16;
          float hv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) hv[i] = odd ? sum[8 + i] : sum[i];
          float* dst = yr + p0 + (odd ? 8 : 0);
          // pixels of this half in the image (W % 16 != 0 pads the tile to
          // 16 pixels); none for a padded output channel
          const int live = c_live ? w - w0 - p0 - (odd ? 8 : 0) : 0;
          if (live < 8) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i < live) dst[i] = hv[i];
          } else if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            reinterpret_cast<float4*>(dst)[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
            reinterpret_cast<float4*>(dst)[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = hv[i];
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[acc]);
        if (q == 0 && lane == 0) {
          if (o == 0) WS_TRACE(6);
          WS_TRACE(4);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  const int redo = __syncthreads_or(mag >= 0x7f000000u);
  if (threadIdx.x == 0) {
    WS_TRACE(5);
    WS_GT(1);
  }
  if (redo) {
    // a non-finite or huge input in this CTA's rows: recompute its outputs
    // with fp32 FMAs (ci, dj, di ascending), overwriting the tensor-core
    // results (the barrier above orders the two sets of global stores), so
    // inf / NaN come out as the reference's pattern instead of the split's
    // NaN.  Rare and slow (~0.2 ms per CTA), never taken on finite inputs.
    const int64_t plane = (int64_t)h * w;
    for (int it = cta_in_co; it < args.items_per_co; it += args.ctas_per_co) {
      int n, w0, r0, nr;
      item_of(it, n, w0, r0, nr);
      const int cols = min(wt, w - w0);
      const int64_t total = (int64_t)kCo * nr * cols;
      for (int64_t e = threadIdx.x; e < total; e += kThreads) {
        const int cc = (int)(e % cols), rr = (int)((e / cols) % nr), cl = (int)(e / ((int64_t)cols * nr));
        const int co = co_tile * kCo + cl;
        if (co >= args.cout) continue;
        const int r = r0 + rr, c = w0 + cc;
        const float* xn = xraw + (int64_t)n * cin * plane;
        const float* wc = wraw + (int64_t)co * cin * 9;
        float acc = 0.0f;
        for (int ci = 0; ci < cin; ++ci)
          for (int dj = 0; dj < 3; ++dj) {
            const int rin = r + dj - 1;
            if (rin < 0 || rin >= h) continue;
            for (int di = 0; di < 3; ++di) {
              const int cin_c = c + di - 1;
              if (cin_c < 0 || cin_c >= w) continue;
              acc = fmaf(wc[ci * 9 + dj * 3 + di], xn[ci * plane + (int64_t)rin * w + cin_c], acc);
            }
          }
        y[((int64_t)n * args.cout + co) * plane + (int64_t)r * w + c] = acc;
      }
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols)
                 : "memory");
  }
}

// w[co][ci][3][3] -> A for each 64-channel tile (stored chunk-major for
// coalesced loads, see the A load above): row 32q + j holds channel
// 16q + (j & 15), bf16 w1 for j < 16 and bf16 w2 = bf16(w - w1) for j >= 16;
// column k2 packs K elements (2 k2, 2 k2 + 1) with K = tap * Cin + ci (low
// half = even element)
__global__ void pack_weights_kernel(const float* __restrict__ wt, uint32_t* __restrict__ apack,
                                    int cin, int cout) {
  // let the dependent conv kernel launch now (it waits for this grid's
  // completion before reading apack)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef SC_WS_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_pack_gt[0] = gtimer();
#endif
  const int a_cols = 9 * cin / 2;
  const int total = (cout + kCo - 1) / kCo * 128 * a_cols;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int k2 = e % a_cols;
    const int m = (e / a_cols) % 128;
    const int tile = e / (a_cols * 128);
    const int co = tile * kCo + 16 * (m >> 5) + (m & 15), hlf = (m >> 4) & 1;
    uint32_t packed = 0;
    for (int t = 0; t < 2; ++t) {
      const int kidx = 2 * k2 + t;
      const int tap = kidx / cin, ci = kidx % cin;
      const float v = co < cout ? wt[((int64_t)co * cin + ci) * 9 + tap] : 0.0f;
      const __nv_bfloat16 v1 = __float2bfloat16_rn(v);
      const __nv_bfloat16 part = hlf ? __float2bfloat16_rn(v - __bfloat162float(v1)) : v1;
      packed |= (uint32_t)__bfloat16_as_ushort(part) << (16 * t);
    }
    // [tile][chunk = k2 / 16][piece = (k2 % 16) / 4][lane m][word k2 % 4]
    const int chunk = k2 >> 4, piece = (k2 >> 2) & 3, word = k2 & 3;
    apack[((((size_t)tile * (a_cols / 16) + chunk) * 4 + piece) * 128 + m) * 4 + word] = packed;
  }
}

int pick_tile_width(int64_t w) {
  for (int t = kMaxWt / 16; t >= 1; --t)
    if ((w / 16) % t == 0) return 16 * t;
  return 16;
}

}  // namespace

// Returns SC_OK / an error if it ran, 1 if the shape is outside its range.
int nchw3x3_ws(const float* x, int64_t nb, int64_t cin, int64_t h, int64_t w, const float* wt,
               int64_t cout, float* y, cudaStream_t st) {
  // W % 16 != 0 (e.g. 56, 28): one column tile padded to the next multiple
  // of 16 pixels (TMA zero-fills the columns past W, the epilogue masks
  // them); the x rows must still be 16-byte aligned for TMA (W % 4 == 0)
  const bool padded = w % 16 != 0;
  if (cin > kMaxCin || cin % 32 != 0 || cout < 1 || w % 4 != 0 ||
      (padded && w > kMaxWt) ||
      (reinterpret_cast<uintptr_t>(x) & 15) || nb * cin * h * w >= ((int64_t)1 << 31) ||
      nb * cout * h * w >= ((int64_t)1 << 31) || h < 1)
    return 1;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int tw = padded ? (int)((w + 15) / 16 * 16) : pick_tile_width(w);
  WsArgs a;
  a.nb = (int)nb, a.cin = (int)cin, a.h = (int)h, a.w = (int)w, a.cout = (int)cout;
  a.wt = tw;
  a.col_tiles = padded ? 1 : (int)(w / tw);
  const int co_tiles = (int)((cout + kCo - 1) / kCo);
  const int sms = sm_count();
  a.ctas_per_co = std::max(1, sms / co_tiles);
  // Segment length: the CTAs (one per SM) walk items of seg_rows output rows
  // (one image, one column tile) in a grid-stride loop, so the kernel lasts
  // ceil(items / ctas) items.  Pick seg_rows minimising that x (seg_rows + 2)
  // (+2: the per-item pipeline fill).  Splitting rows_total evenly and
  // rounding per image made 160 items for 148 CTAs at N = 32 (kernel 2.5x
  // the N = 16 time instead of 2x).
  const int64_t units = nb * a.col_tiles;
  int64_t best = -1;
  a.seg_rows = (int)h;
  for (int64_t sr = 4; sr <= h; ++sr) {
    const int64_t items = units * ((h + sr - 1) / sr);
    const int64_t cost = (items + a.ctas_per_co - 1) / a.ctas_per_co * (sr + 2);
    if (best < 0 || cost < best) best = cost, a.seg_rows = (int)sr;
  }
  a.segs = (int)((h + a.seg_rows - 1) / a.seg_rows);
  a.items_per_co = (int)(nb * a.col_tiles * a.segs);
  a.ctas_per_co = std::min(a.ctas_per_co, a.items_per_co);

  cuuint64_t dims[4] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)cin, (cuuint64_t)nb};
  cuuint64_t strides[3] = {(cuuint64_t)(w * 4), (cuuint64_t)(h * w * 4),
                           (cuuint64_t)(cin * h * w * 4)};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMap mx, mh;
  {
    cuuint32_t box[4] = {(cuuint32_t)tw, 1, (cuuint32_t)cin, 1};
    CUresult r = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "nchw ws: x tensor map failed");
  }
  {
    cuuint32_t box[4] = {kHaloW, 1, (cuuint32_t)cin, 1};
    CUresult r = enc(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides,
                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "nchw ws: halo tensor map failed");
  }
  uint32_t* apack = nullptr;
  const size_t abytes = (size_t)co_tiles * 128 * (9 * cin / 2) * sizeof(uint32_t);
  SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&apack), abytes, st));
  pack_weights_kernel<<<(unsigned)std::min<int64_t>(1024, (int64_t)(abytes / 4 + 255) / 256), 256,
                        0, st>>>(wt, apack, (int)cin, (int)cout);
  SC_LAUNCH_CHECK("pack_weights_kernel");
  static uint64_t attr = 0;  // devices whose limit is set
  auto kern = cin == 64 ? nchw3x3_ws_kernel<4> : nchw3x3_ws_kernel<2>;
  static uint64_t attr2 = 0;
  SC_CUDA(set_smem_limit_once(kern, (int)kSmem, cin == 64 ? &attr : &attr2));
  const unsigned grid = (unsigned)(a.ctas_per_co * co_tiles);
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    SC_CUDA(cudaLaunchKernelEx(&cfg, kern, mx, mh, (const uint32_t*)apack, y, a, x, wt));
  }
  SC_LAUNCH_CHECK("nchw3x3_ws_kernel");
  SC_CUDA(cudaFreeAsync(apack, st));
  return SC_OK;
}

}  // namespace sc
