// 2-D single-channel valid convolution (and batched 1-D as a 1 x k filter).
//
// Replaces _accumulate_taps (reference.py:15-23) behind conv2d_reference,
// conv2d_slide_generic / _compound, conv2d_custom3 / 5 and conv1d_slide
// (kernels.py:220-275).
//
// conv2d_tma_kernel<KH, KW> -- the filter-size-specialised path, the GPU form
// of the paper's custom kernels (kernels.py:185-206: each input row's slid
// vectors are built once and reused for every output row that touches it).
//   * A CTA owns a column strip of TW = 32*NW output columns and RC output
//     rows.  A producer warp streams the strip's input rows (TW + KW - 1
//     columns, RS rows per stage) into an NST-deep shared-memory ring with
//     cp.async.bulk.tensor (TMA) and mbarrier complete_tx.
//   * Each consumer warp owns 32 output columns (lane-striped, so every
//     global store is one coalesced 128-byte line -- output rows are not
//     16-byte aligned, SURVEY 7 hard part 1).  Walking input rows once, a lane
//     reads its KW taps of the row from shared memory and folds them into KH
//     register-resident rolling accumulators (output rows t-KH+1 .. t).
//   * Taps live in the launch parameters (constant bank), so FFMA / FMUL read
//     them as constant operands; KH x KW is fully unrolled.
//   * kExact: __fmul_rn + __fadd_rn in ascending (j, i) order from 0 ->
//     bit-identical to the reference; otherwise one FFMA per tap.
// conv2d_generic_kernel<T> -- runtime (kh, kw), float or double (the latter
// backs oracle_conv2d, reference.py:42-47); direct, L1-cached loads.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace sc {
namespace {

template <int KH, int KW>
struct Taps {
  float f[KH * KW];
};
// (f, f) pairs for the packed fp32x2 FMA of the fast path
template <int KH, int KW>
struct TapPairs {
  unsigned long long f[KH * KW];
};

constexpr int kConsumerWarps = 2;
constexpr int kColsPerLane = 2;                                // cols lane and lane + 32
constexpr int kColsPerWarp = 32 * kColsPerLane;
constexpr int kColsPerCta = kColsPerWarp * kConsumerWarps;     // 128 output columns
constexpr int kStages = 4;

template <int KH>
struct RowsPerStage {
  // a multiple of KH so the rolling-accumulator phase is static per stage
  static constexpr int value = KH == 1 ? 8 : (KH == 3 ? 12 : (KH == 5 ? 10 : 14));
};

__host__ __device__ constexpr int box_cols(int kw) { return ((kColsPerCta + kw - 1) + 3) / 4 * 4; }
__host__ __device__ constexpr int stage_floats(int rs, int bw) { return (rs * bw + 31) / 32 * 32; }

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Fast path: packed FFMA2 over the lane's column pair.  Exact path: scalar
// __fmul_rn/__fadd_rn (ptxas contracts mul/add.rn.f32x2 into FFMA2, so the
// packed forms cannot be used for the reference's two-rounding order).
template <int KH, int KW, bool kExact>
__global__ void __launch_bounds__(32 * (kConsumerWarps + 1))
    conv2d_tma_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                      int64_t oh, int64_t ow, int rows_per_cta, const Taps<KH, KW> taps,
                      const TapPairs<KH, KW> pairs) {
  constexpr int RS = RowsPerStage<KH>::value;
  constexpr int BW = box_cols(KW);
  constexpr int kStageFloats = stage_floats(RS, BW);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // TMA destinations must be 128-byte aligned: align the dynamic base and
  // round every stage up to a multiple of 32 floats
  float* smem = reinterpret_cast<float*>(
      smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  __shared__ __align__(8) uint64_t full_bar[kStages];
  __shared__ __align__(8) uint64_t empty_bar[kStages];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * kColsPerCta;
  const int r0 = blockIdx.y * rows_per_cta;
  const int b = blockIdx.z;
  const int rc = (int)min((int64_t)rows_per_cta, oh - r0);  // output rows here
  const int n_in = rc + KH - 1;                              // input rows needed
  const int n_stage = (n_in + RS - 1) / RS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: one elected lane issues the TMA ring
    if (lane == 0) {
      prefetch_tmap(&tmap);
      for (int s = 0; s < n_stage; ++s) {
        const int slot = s % kStages;
        if (s >= kStages) mbar_wait_sleep(&empty_bar[slot], ((s / kStages) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[slot], RS * BW * (uint32_t)sizeof(float));
        tma_load_3d(smem + slot * kStageFloats, &tmap, &full_bar[slot], c0, r0 + s * RS, b);
      }
    }
    return;
  }

  // ---------------- consumers: lane owns columns col and col + 32
  const int col = warp * kColsPerWarp + lane;
  const int64_t gcol = (int64_t)c0 + col;
  const bool ok0 = gcol < ow, ok1 = gcol + 32 < ow;
  // address of output row (t - KH + 1) for the input row t being consumed
  float* ynext = y + ((int64_t)b * oh + r0 - (KH - 1)) * ow + gcol;

  float a0[KH], a1[KH];                 // exact path accumulators
  unsigned long long ap[KH];            // fast path packed accumulators
#pragma unroll
  for (int j = 0; j < KH; ++j) {
    a0[j] = a1[j] = 0.0f;
    ap[j] = 0ull;
  }

  for (int s = 0; s < n_stage; ++s) {
    const int slot = s % kStages;
    mbar_wait(&full_bar[slot], (s / kStages) & 1);
    const float* buf = smem + slot * kStageFloats + col;
    // software pipeline over the stage's rows: the taps of row r+1 are read
    // from shared memory while row r's FMAs run (hides the LDS latency)
    float c0v[KW], c1v[KW];
#pragma unroll
    for (int i = 0; i < KW; ++i) {
      c0v[i] = buf[i];
      c1v[i] = buf[32 + i];
    }
#pragma unroll 1
    for (int g = 0; g < RS / KH; ++g) {
#pragma unroll
      for (int u = 0; u < KH; ++u) {
        const int rr = g * KH + u;  // row within the stage
        float n0v[KW], n1v[KW];
        if (u < KH - 1 || rr + 1 < RS) {
          const float* nx = buf + (rr + 1) * BW;
#pragma unroll
          for (int i = 0; i < KW; ++i) {
            n0v[i] = nx[i];
            n1v[i] = nx[32 + i];
          }
        }
        // output row t - j lives in slot (u - j) mod KH; RS % KH == 0 keeps
        // (t mod KH) == u, so every index below is a compile-time constant.
        if constexpr (kExact) {
#pragma unroll
          for (int j = 0; j < KH; ++j) {
            const int sl = ((u - j) % KH + KH) % KH;
            float p = (j == 0) ? 0.0f : a0[sl];
            float q = (j == 0) ? 0.0f : a1[sl];
#pragma unroll
            for (int i = 0; i < KW; ++i) {
              p = mac<true>(p, taps.f[j * KW + i], c0v[i]);
              q = mac<true>(q, taps.f[j * KW + i], c1v[i]);
            }
            a0[sl] = p;
            a1[sl] = q;
          }
        } else {
          unsigned long long v[KW];
#pragma unroll
          for (int i = 0; i < KW; ++i) v[i] = pack2(c0v[i], c1v[i]);
#pragma unroll
          for (int j = 0; j < KH; ++j) {
            const int sl = ((u - j) % KH + KH) % KH;
            unsigned long long p = (j == 0) ? 0ull : ap[sl];
#pragma unroll
            for (int i = 0; i < KW; ++i) p = ffma2(v[i], pairs.f[j * KW + i], p);
            ap[sl] = p;
          }
        }
#pragma unroll
        for (int i = 0; i < KW; ++i) {
          c0v[i] = n0v[i];
          c1v[i] = n1v[i];
        }
        // output row t - KH + 1 is complete; ynext tracks its address
        const int t = s * RS + rr;  // input row relative to r0
        if ((unsigned)(t - (KH - 1)) < (unsigned)rc) {
          const int sl = (u + 1) % KH;
          float r0v, r1v;
          if constexpr (kExact) {
            r0v = a0[sl];
            r1v = a1[sl];
          } else {
            const float2 pr = unpack2(ap[sl]);
            r0v = pr.x;
            r1v = pr.y;
          }
          if (ok0) ynext[0] = r0v;
          if (ok1) ynext[32] = r1v;
        }
        ynext += ow;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
  }
}

// ------------------------------------------------ 4-column rolling kernel
// conv2d_cols4_kernel<K>: the FP32-bound 7 x 7 (config 5).  A lane owns FOUR
// consecutive output columns and K rolling accumulator rows (4K registers).
// Per input row it reads its K + 3 inputs (two LDS.128 + one LDS.64 ... as
// float4 / float2, conflict-free) and issues 4 K^2 FFMAs with the taps as
// constant-bank operands: ~97 % of the issued instructions are FMAs (the
// column-pair kernel above spends ~30 % on loads and packing).  Each consumer
// warp covers 128 columns with its own TMA box per stage.
constexpr int kC4Warps = 4;                        // consumer warps per CTA (one TMA box each)
constexpr int kC4Cols = 128;                       // output columns per warp
#ifndef SC_C4_STAGES
#define SC_C4_STAGES 4
#endif
constexpr int kC4Stages = SC_C4_STAGES;
// input rows per stage: a multiple of K (static rolling slots), ~7-10 rows
#ifndef SC_C4_PACKED
#define SC_C4_PACKED 1
#endif
#ifndef SC_ROT4_PACKED
#define SC_ROT4_PACKED 1
#endif
__host__ __device__ constexpr int c4_rs(int k) { return k >= 7 ? k : 2 * k; }
__host__ __device__ constexpr int c4_box(int k) { return (kC4Cols + k - 1 + 3) / 4 * 4; }
__host__ __device__ constexpr int c4_sub(int k) {  // one warp's box, 128-byte aligned
  return (c4_rs(k) * c4_box(k) + 31) / 32 * 32;
}

template <int K, bool kExact>
__global__ void __launch_bounds__(32 * (kC4Warps + 1))
    conv2d_cols4_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                        int64_t oh, int64_t ow, int rows_per_cta, const Taps<K, K> taps) {
  constexpr int BW = c4_box(K);
  constexpr int SUB = c4_sub(K);
  constexpr int STAGE = kC4Warps * SUB;
  constexpr int kC4RS = c4_rs(K);
  static_assert(kC4RS % K == 0, "rows per stage must be a multiple of K");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  __shared__ __align__(8) uint64_t full_bar[kC4Stages];
  __shared__ __align__(8) uint64_t empty_bar[kC4Stages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * (kC4Warps * kC4Cols);
  const int r0 = blockIdx.y * rows_per_cta;
  const int b = blockIdx.z;
  const int rc = (int)min((int64_t)rows_per_cta, oh - r0);
  const int n_in = rc + K - 1;
  const int n_stage = (n_in + kC4RS - 1) / kC4RS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kC4Stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kC4Warps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kC4Warps) {
    if (lane == 0) {
      prefetch_tmap(&tmap);
      for (int s = 0; s < n_stage; ++s) {
        const int slot = s % kC4Stages;
        if (s >= kC4Stages) mbar_wait_sleep(&empty_bar[slot], ((s / kC4Stages) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[slot], kC4Warps * kC4RS * BW * (uint32_t)sizeof(float));
        for (int wv = 0; wv < kC4Warps; ++wv)
          tma_load_3d(smem + slot * STAGE + wv * SUB, &tmap, &full_bar[slot], c0 + wv * kC4Cols,
                      r0 + s * kC4RS, b);
      }
    }
    return;
  }

  const int col = warp * kC4Cols + 4 * lane;       // first of the lane's 4 columns
  const int64_t gcol = (int64_t)c0 + col;
  float* ynext = y + ((int64_t)b * oh + r0 - (K - 1)) * ow + gcol;
  const OutCols nvc = out_cols<4>(y, ow, c0 + warp * kC4Cols, gcol);
  // fast mode: packed FFMA2 on column pairs (0,1), (2,3) with the tap as a
  // broadcast uniform-register operand; the odd tap offsets read a second,
  // shifted pair view of the input row (K / 2 + 1 pairs rebuilt once per
  // row, shared by all K x K taps).  Half the FMA issue slots of scalar
  // FFMA.  Exact mode: scalar FMUL + FADD in the reference order.
  constexpr bool kPacked = !kExact && SC_C4_PACKED && K >= 7;  // 5x5: HBM-bound, scalar 1 % faster
  float acc[K][4];
  float2 acc2[K][2];
#pragma unroll
  for (int j = 0; j < K; ++j) {
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[j][c] = 0.0f;
    acc2[j][0] = acc2[j][1] = make_float2(0.0f, 0.0f);
  }

  for (int s = 0; s < n_stage; ++s) {
    const int slot = s % kC4Stages;
    mbar_wait(&full_bar[slot], (s / kC4Stages) & 1);
    const float* buf = smem + slot * STAGE + warp * SUB + 4 * lane;
    auto load = [&](int rr, float (&v)[K + 3]) {
      const float* p = buf + rr * BW;
#pragma unroll
      for (int q = 0; q < (K + 3) / 4; ++q) {
        const float4 t = reinterpret_cast<const float4*>(p)[q];
        v[4 * q] = t.x, v[4 * q + 1] = t.y, v[4 * q + 2] = t.z, v[4 * q + 3] = t.w;
      }
#pragma unroll
      for (int q = (K + 3) / 4 * 4; q < K + 3; ++q) v[q] = p[q];
    };
    // packed path: the row as aligned pairs pe = (x0,x1),(x2,x3).. (LDS.128 /
    // LDS.64) and shifted pairs po = (x1,x2),(x3,x4).. loaded straight into
    // register pairs (scalar LDS: building them from pe costs ~8 moves per
    // row that ptxas multiplies by re-materialising); two row buffers
    // alternate with the (unrolled) row index, so the prefetch needs no copy
    constexpr int kPe = (K + 3) / 2, kPo = K / 2 + 1;
    float2 pe[2][kPe], po[2][kPo];
    auto loadp = [&](int rr, int bsel) {
      const float* p = buf + rr * BW;
#pragma unroll
      for (int q = 0; q < kPe / 2; ++q) {
        const float4 t = reinterpret_cast<const float4*>(p)[q];
        pe[bsel][2 * q] = make_float2(t.x, t.y);
        pe[bsel][2 * q + 1] = make_float2(t.z, t.w);
      }
      if constexpr (kPe % 2) pe[bsel][kPe - 1] = reinterpret_cast<const float2*>(p)[kPe - 1];
#pragma unroll
      for (int q = 0; q < kPo; ++q) po[bsel][q] = lds_pair_unaligned(p + 2 * q + 1);
    };
    float cur[K + 3];
    if constexpr (kPacked) loadp(0, 0);
    else load(0, cur);
#pragma unroll 1
    for (int g = 0; g < kC4RS / K; ++g) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int rr = g * K + u;
        float nxt[K + 3];
        if constexpr (kPacked) {
          if (rr + 1 < kC4RS) loadp(rr + 1, (u + 1) & 1);
        } else {
          if (rr + 1 < kC4RS) load(rr + 1, nxt);
        }
        // output row t - j lives in slot (u - j) mod K (kC4RS % K == 0)
        if constexpr (kPacked) {
          const float2(&pe_u)[kPe] = pe[u & 1];
          const float2(&po_u)[kPo] = po[u & 1];
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int sl = ((u - j) % K + K) % K;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp) {
              float2 a = (j == 0) ? make_float2(0.0f, 0.0f) : acc2[sl][pp];
#pragma unroll
              for (int i = 0; i < K; ++i) {
                const float tv = taps.f[j * K + i];
                a = __ffma2_rn(make_float2(tv, tv), (i & 1) ? po_u[pp + i / 2] : pe_u[pp + i / 2],
                               a);
              }
              acc2[sl][pp] = a;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j) {
            const int sl = ((u - j) % K + K) % K;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              float a = (j == 0) ? 0.0f : acc[sl][c];
#pragma unroll
              for (int i = 0; i < K; ++i) a = mac<kExact>(a, taps.f[j * K + i], cur[c + i]);
              acc[sl][c] = a;
            }
          }
        }
        if constexpr (!kPacked) {
#pragma unroll
          for (int q = 0; q < K + 3; ++q) cur[q] = nxt[q];
        }
        const int t = s * kC4RS + rr;  // input row relative to r0
        if ((unsigned)(t - (K - 1)) < (unsigned)rc) {
          if constexpr (kPacked) {
            const int sl = (u + 1) % K;
            const float o[4] = {acc2[sl][0].x, acc2[sl][0].y, acc2[sl][1].x, acc2[sl][1].y};
            store_cols<4>(ynext, nvc, o);
          } else {
            store_cols<4>(ynext, nvc, acc[(u + 1) % K]);
          }
        }
        ynext += ow;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
  }
}

// ------------------------------------------- rotating 4-column kernel
// conv2d_rot4_kernel<K>: the same lane tiling for the paper's larger square
// filters (K = 9 .. 29): 4 columns x K accumulator rows per lane, taps in the
// constant bank, but instead of unrolling K input rows to make the rolling
// slot indices static, the accumulator rows are shifted by one after each
// input row (4 (K - 1) moves against 4 K^2 FFMAs), so the code size is one
// row body (4 K^2 FFMAs) and the stage depth is independent of K.
constexpr int kR4RS = 8;
template <int K>
struct BigSquareTaps {
  float f[K * K];
};

// C = columns per lane (4; a 2-column variant for K = 29..37 measured slower
// than conv2d_big, 18-25 vs 36 TFLOP/s); a warp covers 32 C columns.
__host__ __device__ constexpr int rot_box(int k, int c) { return (32 * c + k - 1 + 3) / 4 * 4; }

template <int K, int C, bool kExact>
__global__ void __launch_bounds__(32 * (kC4Warps + 1))
    conv2d_rot4_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                       int64_t oh, int64_t ow, int rows_per_cta,
                       const __grid_constant__ BigSquareTaps<K> taps) {
  constexpr int BW = rot_box(K, C);
  constexpr int SUB = (kR4RS * BW + 31) / 32 * 32;
  constexpr int STAGE = kC4Warps * SUB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127));
  __shared__ __align__(8) uint64_t full_bar[kC4Stages];
  __shared__ __align__(8) uint64_t empty_bar[kC4Stages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * (kC4Warps * 32 * C);
  const int r0 = blockIdx.y * rows_per_cta;
  const int b = blockIdx.z;
  const int rc = (int)min((int64_t)rows_per_cta, oh - r0);
  const int n_in = rc + K - 1;
  const int n_stage = (n_in + kR4RS - 1) / kR4RS;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kC4Stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kC4Warps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kC4Warps) {
    if (lane == 0) {
      prefetch_tmap(&tmap);
      for (int s = 0; s < n_stage; ++s) {
        const int slot = s % kC4Stages;
        if (s >= kC4Stages) mbar_wait_sleep(&empty_bar[slot], ((s / kC4Stages) - 1) & 1);
        mbar_arrive_expect_tx(&full_bar[slot], kC4Warps * kR4RS * BW * (uint32_t)sizeof(float));
        for (int wv = 0; wv < kC4Warps; ++wv)
          tma_load_3d(smem + slot * STAGE + wv * SUB, &tmap, &full_bar[slot],
                      c0 + wv * 32 * C, r0 + s * kR4RS, b);
      }
    }
    return;
  }

  const int col = warp * 32 * C + C * lane;
  const int64_t gcol = (int64_t)c0 + col;
  float* ynext = y + ((int64_t)b * oh + r0 - (K - 1)) * ow + gcol;
  const OutCols nvc = out_cols<C>(y, ow, c0 + warp * 32 * C, gcol);
  // acc[j]: output row t - (K - 1) + j for the input row t just consumed.
  // Fast mode with C = 4: packed FFMA2 on column pairs as in
  // conv2d_cols4_kernel (aligned pairs by LDS.128, shifted pairs by volatile
  // scalar loads, taps broadcast from uniform registers).
  // (measured per K: 4 x 2048^2 k = 9 / 13 / 15 / 17: 33 / 37 / 36 / 35 -> 40 /
  // 43 / 43 / 44 TFLOP/s, 32 x 512^2 even or better; K = 11 (spills) and 21
  // lose 7-10 % on the small images, so they stay scalar)
  constexpr bool kPk = !kExact && C == 4 && SC_ROT4_PACKED && K != 11 && K != 21;
  float acc[K][C];
  float2 ap[K][2];
#pragma unroll
  for (int j = 0; j < K; ++j) {
#pragma unroll
    for (int c = 0; c < C; ++c) acc[j][c] = 0.0f;
    ap[j][0] = ap[j][1] = make_float2(0.0f, 0.0f);
  }

  int t = 0;  // input row relative to r0
  for (int s = 0; s < n_stage; ++s) {
    const int slot = s % kC4Stages;
    mbar_wait(&full_bar[slot], (s / kC4Stages) & 1);
    const float* buf = smem + slot * STAGE + warp * SUB + C * lane;
    const int rows_here = min(kR4RS, n_in - s * kR4RS);
#pragma unroll 1
    for (int rr = 0; rr < rows_here; ++rr, ++t) {
      constexpr int NW = K + C - 1;  // the lane's input window
      float cur[NW];
      const float* p = buf + rr * BW;
      if constexpr (kPk) {
        constexpr int kPe = (K + 3) / 2, kPo = K / 2 + 1;  // (x0,x1).. / (x1,x2)..
        float2 pe[kPe], po[kPo];
#pragma unroll
        for (int q = 0; q < kPe / 2; ++q) {
          const float4 v = reinterpret_cast<const float4*>(p)[q];
          pe[2 * q] = make_float2(v.x, v.y);
          pe[2 * q + 1] = make_float2(v.z, v.w);
        }
        if constexpr (kPe % 2) pe[kPe - 1] = reinterpret_cast<const float2*>(p)[kPe - 1];
#pragma unroll
        for (int q = 0; q < kPo; ++q) po[q] = lds_pair_unaligned(p + 2 * q + 1);
#pragma unroll
        for (int j = 0; j < K; ++j) {
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            float2 a = ap[j][pp];
#pragma unroll
            for (int i = 0; i < K; ++i) {
              const float tv = taps.f[(K - 1 - j) * K + i];
              a = __ffma2_rn(make_float2(tv, tv), (i & 1) ? po[pp + i / 2] : pe[pp + i / 2], a);
            }
            ap[j][pp] = a;
          }
        }
        if ((unsigned)(t - (K - 1)) < (unsigned)rc) {
          const float o[4] = {ap[0][0].x, ap[0][0].y, ap[0][1].x, ap[0][1].y};
          store_cols<4>(ynext, nvc, o);
        }
        ynext += ow;
#pragma unroll
        for (int j = 0; j < K - 1; ++j) ap[j][0] = ap[j + 1][0], ap[j][1] = ap[j + 1][1];
        ap[K - 1][0] = ap[K - 1][1] = make_float2(0.0f, 0.0f);
        continue;
      }
      if constexpr (C == 4) {
#pragma unroll
        for (int q = 0; q < NW / 4; ++q) {
          const float4 v = reinterpret_cast<const float4*>(p)[q];
          cur[4 * q] = v.x, cur[4 * q + 1] = v.y, cur[4 * q + 2] = v.z, cur[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int q = NW / 4 * 4; q < NW; ++q) cur[q] = p[q];
      } else {
#pragma unroll
        for (int q = 0; q < NW / 2; ++q) {
          const float2 v = reinterpret_cast<const float2*>(p)[q];
          cur[2 * q] = v.x, cur[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int q = NW / 2 * 2; q < NW; ++q) cur[q] = p[q];
      }
      // input row t feeds output rows t - j' for filter row j' = K-1 .. 0:
      // acc[j] holds output row t - (K-1) + j, i.e. filter row K-1-j
#pragma unroll
      for (int j = 0; j < K; ++j) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          float a = acc[j][c];
#pragma unroll
          for (int i = 0; i < K; ++i) a = mac<kExact>(a, taps.f[(K - 1 - j) * K + i], cur[c + i]);
          acc[j][c] = a;
        }
      }
      // acc[0] (output row t - K + 1) is complete
      if ((unsigned)(t - (K - 1)) < (unsigned)rc) {
        store_cols<C>(ynext, nvc, acc[0]);
      }
      ynext += ow;
#pragma unroll
      for (int j = 0; j < K - 1; ++j)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[j][c] = acc[j + 1][c];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[K - 1][c] = 0.0f;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
  }
}

// --------------------------------------------------------------- generic
template <typename T, bool kExact>
__global__ void conv2d_generic_kernel(const T* __restrict__ x, int64_t batch, int64_t h,
                                      int64_t w, const T* __restrict__ f, int kh, int kw,
                                      T* __restrict__ y, int64_t oh, int64_t ow) {
  const int64_t total = batch * oh * ow;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx % ow;
    const int64_t rb = idx / ow;
    const int64_t r = rb % oh;
    const int64_t b = rb / oh;
    const T* xp = x + (b * h + r) * w + c;
    T acc = T(0);
    for (int j = 0; j < kh; ++j) {
      const T* xr = xp + (int64_t)j * w;
      const T* fr = f + j * kw;
      for (int i = 0; i < kw; ++i) acc = mac<kExact>(acc, __ldg(fr + i), __ldg(xr + i));
    }
    y[idx] = acc;
  }
}

// ---------------------------------------------------------- tensor maps
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap(CUtensorMap* map, const float* x, int64_t batch, int64_t h, int64_t w, int bw,
              int rs) {
  auto enc = get_encode();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)w * sizeof(float), (cuuint64_t)(h * w) * sizeof(float)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)rs, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return SC_OK;
}

template <int KH, int KW, bool kExact>
int launch_tma(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, float* y,
               cudaStream_t st) {
  constexpr int RS = RowsPerStage<KH>::value;
  constexpr int BW = box_cols(KW);
  const int64_t oh = h - KH + 1, ow = w - KW + 1;
  CUtensorMap map;
  int rc = make_tmap(&map, x, batch, h, w, BW, RS);
  if (rc) return rc;
  Taps<KH, KW> taps;
  TapPairs<KH, KW> pairs;
  for (int i = 0; i < KH * KW; ++i) {
    taps.f[i] = f[i];
    unsigned int bits;
    std::memcpy(&bits, &f[i], 4);
    pairs.f[i] = ((unsigned long long)bits << 32) | bits;
  }
  // rows per CTA: enough CTAs for >= ~8 waves of 148 SMs, RS-aligned
  const int64_t strips = (ow + kColsPerCta - 1) / kColsPerCta;
  int64_t rows;
  static const int env_rows = [] {
    const char* e = getenv("SC_CONV_ROWS");
    return e ? atoi(e) : 0;
  }();
  if (env_rows > 0) {
    rows = env_rows;
  } else {
    // measured on B200 (tools/conv_sweep.py): short row segments keep the
    // concurrently streamed rows adjacent in HBM for the bandwidth-bound
    // sizes; the FP32-bound 7x7 prefers long segments (less halo re-work).
    // Segment length = RS*m - (KH-1) so the last stage carries no waste.
    const int m = KH >= 7 ? 64 : (KH == 1 ? 7 : (KH == 3 ? 3 : 6));  // 3x3: 34 rows (58: +2.5 %)
    rows = (int64_t)RS * m - (KH - 1);
  }
  rows = std::min<int64_t>(rows, oh);
  const int64_t segs = (oh + rows - 1) / rows;
  if (strips > 0x7fffffff || segs > 65535 || batch > 65535)
    return fail(SC_ERR_UNSUPPORTED, "conv2d: grid too large");
  const size_t smem = (size_t)kStages * stage_floats(RS, BW) * sizeof(float) + 128;
  static uint64_t attr = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(conv2d_tma_kernel<KH, KW, kExact>, (int)smem, &attr));
  dim3 grid((unsigned)strips, (unsigned)segs, (unsigned)batch);
  conv2d_tma_kernel<KH, KW, kExact><<<grid, 32 * (kConsumerWarps + 1), smem, st>>>(
      map, y, oh, ow, (int)rows, taps, pairs);
  SC_LAUNCH_CHECK("conv2d_tma_kernel");
  return SC_OK;
}

// Row-segment length (output rows per CTA) of the 4-column kernel for this
// grid; shared by the launch and by sc_conv2d_segment_rows (test / tooling
// introspection of where CTA segment boundaries fall).
template <int K, bool kExact>
int cols4_rows(int64_t batch, int64_t h, int64_t w, int64_t* rows_out) {
  const int64_t oh = h - K + 1, ow = w - K + 1;
  const int64_t strips = (ow + kC4Warps * kC4Cols - 1) / (kC4Warps * kC4Cols);
  static const int env_rows = [] {
    const char* e = getenv("SC_CONV_ROWS");
    return e ? atoi(e) : 0;
  }();
  // measured (tools/conv_sweep.py): long segments for the FP32-bound 7 x 7
  // (then refined by the wave model below); 96-row segments for the
  // bandwidth-bound 5 x 5 (config 3: 446 rows 0.707 ms -> 96 rows 0.654 ms,
  // i.e. 1.0 of the HBM copy peak: many short CTAs keep the streams adjacent
  // and the last wave short)
  const int64_t seg_rows = K >= 7 ? 896 : 100;
  int64_t rows = env_rows > 0 ? env_rows : (int64_t)c4_rs(K) * (seg_rows / c4_rs(K)) - (K - 1);
  const size_t smem = (size_t)kC4Stages * kC4Warps * c4_sub(K) * sizeof(float) + 128;
  static uint64_t attr = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(conv2d_cols4_kernel<K, kExact>, smem, &attr));
  static int slots_dev[kMaxDevices] = {};  // resident CTAs on the whole GPU
  int& slots = slots_dev[current_device()];
  if (!slots) {
    int occ = 0;
    SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, conv2d_cols4_kernel<K, kExact>, 32 * (kC4Warps + 1), smem));
    slots = std::max(1, occ) * sm_count();
  }
  if (env_rows <= 0 && K >= 7) {
    // FP32-bound: every CTA costs ~(segment stages) and the grid runs in
    // waves of `slots` CTAs, so pick the segment length (whole stages, no
    // tail waste) minimising waves x stages per CTA over 40..200 stages.
    // Whole 65,536^2 image: 14.99 waves instead of 21.3 (-3.6 % modelled);
    // an 8,192-row band (row-band config 5 at G = 8): 6.9 waves instead of
    // 2.9 (-9 %).
    int64_t best = -1;
    for (int64_t m = 40; m <= 200; ++m) {
      const int64_t r = (int64_t)c4_rs(K) * m - (K - 1);
      const int64_t n = strips * ((oh + r - 1) / r) * batch;
      const int64_t cost = (n + slots - 1) / slots * m;
      if (best < 0 || cost < best) best = cost, rows = r;
    }
  }
  *rows_out = std::min<int64_t>(rows, oh);
  return SC_OK;
}


template <int K, bool kExact>
int launch_cols4(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, float* y,
                 cudaStream_t st) {
  constexpr int BW = c4_box(K);
  const int64_t oh = h - K + 1, ow = w - K + 1;
  CUtensorMap map;
  int rc = make_tmap(&map, x, batch, h, w, BW, c4_rs(K));
  if (rc) return rc;
  Taps<K, K> taps;
  for (int i = 0; i < K * K; ++i) taps.f[i] = f[i];
  const int64_t strips = (ow + kC4Warps * kC4Cols - 1) / (kC4Warps * kC4Cols);
  const size_t smem = (size_t)kC4Stages * kC4Warps * c4_sub(K) * sizeof(float) + 128;
  int64_t rows = 0;
  if ((rc = cols4_rows<K, kExact>(batch, h, w, &rows))) return rc;
  rows = std::min<int64_t>(rows, oh);
  const int64_t segs = (oh + rows - 1) / rows;
  if (strips > 0x7fffffff || segs > 65535 || batch > 65535)
    return fail(SC_ERR_UNSUPPORTED, "conv2d: grid too large");
  dim3 grid((unsigned)strips, (unsigned)segs, (unsigned)batch);
  conv2d_cols4_kernel<K, kExact><<<grid, 32 * (kC4Warps + 1), smem, st>>>(map, y, oh, ow,
                                                                         (int)rows, taps);
  SC_LAUNCH_CHECK("conv2d_cols4_kernel");
  return SC_OK;
}

template <int K, int C, bool kExact>
int launch_rot4(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, float* y,
                cudaStream_t st) {
  constexpr int BW = rot_box(K, C);
  const int64_t oh = h - K + 1, ow = w - K + 1;
  CUtensorMap map;
  int rc = make_tmap(&map, x, batch, h, w, BW, kR4RS);
  if (rc) return rc;
  BigSquareTaps<K> taps;
  for (int i = 0; i < K * K; ++i) taps.f[i] = f[i];
  const int64_t strips = (ow + kC4Warps * 32 * C - 1) / (kC4Warps * 32 * C);
  const size_t smem =
      (size_t)kC4Stages * kC4Warps * ((kR4RS * BW + 31) / 32 * 32) * sizeof(float) + 128;
  static uint64_t attr = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(conv2d_rot4_kernel<K, C, kExact>, (int)smem, &attr));
  static int slots_dev[kMaxDevices] = {};  // resident CTAs on the whole GPU
  int& slots = slots_dev[current_device()];
  if (!slots) {
    int occ = 0;
    SC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, conv2d_rot4_kernel<K, C, kExact>, 32 * (kC4Warps + 1), smem));
    slots = std::max(1, occ) * sm_count();
  }
  // rows per CTA: FP32-bound, a CTA costs ~(rows + K - 1) input rows and the
  // grid runs in waves of `slots` CTAs -- minimise waves x (rows + K - 1)
  // (the old rule, halve from 1,024 until >= 2 waves, gave 64-row segments
  // with 31 % halo re-work for K = 21 on 4 x 2048^2)
  // Measured against the old rule: 4 x 2048^2 / 1 x 4096^2 +5-30 % for
  // K = 9..21, 32 x 512^2 +10 % for K = 15 / 17; K = 21 on 512^2 / 1024^2
  // images loses 7 % (a floor on the grid fill did not recover it).
  int64_t rows = 64, best = -1;
  for (int64_t r = 16; r <= 1024; r += 8) {
    const int64_t n = batch * strips * ((oh + r - 1) / r);
    const int64_t cost = (n + slots - 1) / slots * (std::min<int64_t>(r, oh) + K - 1);
    if (best < 0 || cost < best) best = cost, rows = r;
    if (r >= oh) break;
  }
  rows = std::min<int64_t>(rows, oh);
  const int64_t segs = (oh + rows - 1) / rows;
  if (strips > 0x7fffffff || segs > 65535 || batch > 65535)
    return fail(SC_ERR_UNSUPPORTED, "conv2d: grid too large");
  dim3 grid((unsigned)strips, (unsigned)segs, (unsigned)batch);
  conv2d_rot4_kernel<K, C, kExact><<<grid, 32 * (kC4Warps + 1), smem, st>>>(map, y, oh, ow,
                                                                        (int)rows, taps);
  SC_LAUNCH_CHECK("conv2d_rot4_kernel");
  return SC_OK;
}

template <int K>
int try_rot4(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, bool exact,
             float* y, cudaStream_t st, bool* done) {
  constexpr int C = K <= 21 ? 4 : 2;
  *done = false;
  if ((reinterpret_cast<uintptr_t>(x) % 16) || (w % 4) || w < rot_box(K, C) || h < K) return SC_OK;
  // 512-column CTAs: for a grid smaller than ~one wave (one 512^2 image) the
  // register-blocked conv2d_big kernel, with its smaller tiles, is faster
  const int64_t oh = h - K + 1, ow = w - K + 1;
  const int64_t ctas = batch * ((ow + kC4Warps * 32 * C - 1) / (kC4Warps * 32 * C)) *
                       ((oh + 63) / 64);
  if (ctas < sm_count()) return SC_OK;
  *done = true;
  return exact ? launch_rot4<K, C, true>(x, batch, h, w, f, y, st)
               : launch_rot4<K, C, false>(x, batch, h, w, f, y, st);
}

template <typename T>
int launch_generic(const T* x, int64_t batch, int64_t h, int64_t w, const T* f, int64_t kh,
                   int64_t kw, bool exact, T* y, cudaStream_t st) {
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  T* fd = nullptr;
  const size_t fb = (size_t)(kh * kw) * sizeof(T);
  SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&fd), fb, st));
  SC_CUDA(cudaMemcpyAsync(fd, f, fb, cudaMemcpyHostToDevice, st));
  const int64_t total = batch * oh * ow;
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32));
  if (exact)
    conv2d_generic_kernel<T, true><<<(unsigned)blocks, 256, 0, st>>>(x, batch, h, w, fd, (int)kh,
                                                                      (int)kw, y, oh, ow);
  else
    conv2d_generic_kernel<T, false><<<(unsigned)blocks, 256, 0, st>>>(x, batch, h, w, fd,
                                                                       (int)kh, (int)kw, y, oh, ow);
  SC_LAUNCH_CHECK("conv2d_generic_kernel");
  SC_CUDA(cudaFreeAsync(fd, st));
  return SC_OK;
}

template <int KH, int KW>
bool tma_ok(const float* x, int64_t h, int64_t w) {
  return (reinterpret_cast<uintptr_t>(x) % 16 == 0) && (w % 4 == 0) && w >= box_cols(KW) &&
         h >= RowsPerStage<KH>::value && h * w < (int64_t)1 << 40;
}

template <int KH, int KW>
int try_tma(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, bool exact,
            float* y, cudaStream_t st, bool* done) {
  *done = false;
  if (!tma_ok<KH, KW>(x, h, w)) return SC_OK;
  *done = true;
  if constexpr ((KH == 7 && KW == 7) || (KH == 5 && KW == 5)) {
    static const bool pairs_kernel = [] {
      const char* e = getenv(KH == 7 ? "SC_CONV7_PAIRS" : "SC_CONV5_PAIRS");
      return e && e[0] == '1';
    }();
    // 512-column CTAs need a grid of at least ~2 waves (config 3 / 5 sizes);
    // small images stay on the 128-column pair kernel
    const int64_t ctas = batch * ((w - KW + 1 + kC4Warps * kC4Cols - 1) / (kC4Warps * kC4Cols)) *
                         ((h - KH + 1 + 255) / 256);
    if (!pairs_kernel && w >= c4_box(KH) && ctas >= 2 * sm_count())
      return exact ? launch_cols4<KH, true>(x, batch, h, w, f, y, st)
                   : launch_cols4<KH, false>(x, batch, h, w, f, y, st);
  }
  return exact ? launch_tma<KH, KW, true>(x, batch, h, w, f, y, st)
               : launch_tma<KH, KW, false>(x, batch, h, w, f, y, st);
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return get_encode(); }
int conv1d_tma(const float* x, int64_t rows, int64_t length, const float* w, int64_t k,
               bool exact, float* y, cudaStream_t st);
int conv2d_big(const float* x, int64_t batch, int64_t h, int64_t w, const float* f_host,
               int64_t kh, int64_t kw, bool exact, float* y, cudaStream_t st);
bool conv2d_mma_applicable(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                           int64_t kh, int64_t kw);
int conv2d_mma(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, int64_t kh,
               int64_t kw, float* y, cudaStream_t st);

bool conv2d_mma_big_applicable(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                               int64_t kh, int64_t kw);
int conv2d_mma_big(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, int64_t kh,
                   int64_t kw, float* y, cudaStream_t st);

int conv2d_f32_dispatch(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                        int64_t kh, int64_t kw, bool exact, float* y, cudaStream_t st) {
  bool done = false;
  int rc = SC_OK;
  // fast mode, large filters (kw >= 10): the large-filter slide-MMA kernel
  // (conv2d_mma_big.cu)
  if (!exact && conv2d_mma_big_applicable(x, batch, h, w, f, kh, kw))
    return conv2d_mma_big(x, batch, h, w, f, kh, kw, y, st);
  // fast mode, filters of >= 36 taps with kw <= 9, kh <= 15 on large images:
  // the slide-MMA tensor-core kernel (conv2d_mma.cu; FMA-bound otherwise)
  if (!exact && kh * kw >= 36 && conv2d_mma_applicable(x, batch, h, w, f, kh, kw))
    return conv2d_mma(x, batch, h, w, f, kh, kw, y, st);
  if (kh == 1) {
    // a 1 x k filter over (batch*h) rows == batched 1-D convolution: the TMA
    // blocked-register kernel shared with pooling (csrc/pool_tma.cu)
    rc = conv1d_tma(x, batch * h, w, f, kw, exact, y, st);
    if (rc != 1) return rc;
    rc = SC_OK;
  }
  if (kh == 3 && kw == 3) rc = try_tma<3, 3>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 5 && kw == 5) rc = try_tma<5, 5>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 7 && kw == 7) rc = try_tma<7, 7>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 1 && kw == 7) rc = try_tma<1, 7>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 1 && kw == 3) rc = try_tma<1, 3>(x, batch, h, w, f, exact, y, st, &done);
  // the paper's mid-size square filters: rotating 4-column kernels
  else if (kh == 9 && kw == 9) rc = try_rot4<9>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 11 && kw == 11) rc = try_rot4<11>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 13 && kw == 13) rc = try_rot4<13>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 15 && kw == 15) rc = try_rot4<15>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 17 && kw == 17) rc = try_rot4<17>(x, batch, h, w, f, exact, y, st, &done);
  else if (kh == 21 && kw == 21) rc = try_rot4<21>(x, batch, h, w, f, exact, y, st, &done);
  if (rc || done) return rc;
  // runtime (kh, kw) up to 64 x 64: the register-blocked kernel (conv2d_big.cu)
  rc = conv2d_big(x, batch, h, w, f, kh, kw, exact, y, st);
  if (rc != 1) return rc;
  return launch_generic<float>(x, batch, h, w, f, kh, kw, exact, y, st);
}

}  // namespace sc

static int check_conv_args(int64_t batch, int64_t h, int64_t w, int64_t kh, int64_t kw,
                           const void* x, const void* f, const void* y) {
  using namespace sc;
  if (batch < 0 || h < 1 || w < 1 || kh < 1 || kw < 1)
    return fail(SC_ERR_SHAPE, "dims must be positive");
  if (kh > h || kw > w)
    return fail(SC_ERR_SHAPE, "filter " + std::to_string(kh) + "x" + std::to_string(kw) +
                                  " exceeds input " + std::to_string(h) + "x" + std::to_string(w));
  if (batch > 0 && (!x || !f || !y)) return fail(SC_ERR_ARG, "conv2d: null pointer");
  return SC_OK;
}

extern "C" int sc_conv2d_f32(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                             int64_t kh, int64_t kw, int mode, float* y, void* stream) {
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return sc::fail(SC_ERR_ARG, "bad mode");
  int rc = check_conv_args(batch, h, w, kh, kw, x, f, y);
  if (rc || batch == 0) return rc;
  return sc::conv2d_f32_dispatch(x, batch, h, w, f, kh, kw, mode == SC_MODE_EXACT, y,
                                 static_cast<cudaStream_t>(stream));
}

extern "C" int64_t sc_conv2d_segment_rows(int64_t batch, int64_t h, int64_t w, int64_t kh,
                                          int64_t kw, int mode) {
  // mirrors try_tma's choice of the 4-column kernel (16-byte aligned input)
  using namespace sc;
  if (batch < 1 || kh < 1 || kw < 1 || kh > h || kw > w) return -1;
  if (kh != kw || (kh != 5 && kh != 7) || w % 4 != 0 || h * w >= (int64_t)1 << 40) return 0;
  const bool pairs = getenv(kh == 7 ? "SC_CONV7_PAIRS" : "SC_CONV5_PAIRS") &&
                     getenv(kh == 7 ? "SC_CONV7_PAIRS" : "SC_CONV5_PAIRS")[0] == '1';
  const int64_t ctas = batch * ((w - kw + 1 + kC4Warps * kC4Cols - 1) / (kC4Warps * kC4Cols)) *
                       ((h - kh + 1 + 255) / 256);
  if (pairs || w < c4_box((int)kh) || ctas < 2 * sm_count() ||
      h < (kh == 7 ? RowsPerStage<7>::value : RowsPerStage<5>::value))
    return 0;
  int64_t rows = 0;
  const bool exact = mode == SC_MODE_EXACT;
  int rc = kh == 7 ? (exact ? cols4_rows<7, true>(batch, h, w, &rows)
                            : cols4_rows<7, false>(batch, h, w, &rows))
                   : (exact ? cols4_rows<5, true>(batch, h, w, &rows)
                            : cols4_rows<5, false>(batch, h, w, &rows));
  return rc ? -1 : rows;
}

extern "C" int sc_conv1d_f32(const float* x, int64_t batch, int64_t length, const float* wt,
                             int64_t k, int mode, float* y, void* stream) {
  // batch signals of `length` samples == a (batch, length) image with a 1 x k
  // filter (bit-identical).
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return sc::fail(SC_ERR_ARG, "bad mode");
  int rc = check_conv_args(1, batch > 0 ? batch : 1, length, 1, k, x, wt, y);
  if (rc || batch == 0) return rc;
  return sc::conv2d_f32_dispatch(x, 1, batch, length, wt, 1, k, mode == SC_MODE_EXACT, y,
                                 static_cast<cudaStream_t>(stream));
}

extern "C" int sc_conv2d_f64(const double* x, int64_t batch, int64_t h, int64_t w,
                             const double* f, int64_t kh, int64_t kw, double* y, void* stream) {
  int rc = check_conv_args(batch, h, w, kh, kw, x, f, y);
  if (rc || batch == 0) return rc;
  return sc::launch_generic<double>(x, batch, h, w, f, kh, kw, true, y,
                                    static_cast<cudaStream_t>(stream));
}
