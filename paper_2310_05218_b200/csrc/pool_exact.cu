// Exact (bit-identical) sliding-window sums and averages for 32 < k <= 512
// on aligned signals: the reference's own arithmetic (pooling.py:28-53), at
// O(log k) adds per output instead of one global pass per stage.
//
// The reference builds doubling partials P_{2w}(j) = P_w(j) + P_w(j + w) up
// to W = the largest power of two <= k, then folds in the other set bits of
// k, largest first: acc = P_W(i); acc = acc + P_b(i + width); width += b.
// Float addition is not associative, so every sum here is formed exactly
// that way.
//
// A warp holds a 1,024-sample window, lane l the 32 CONSECUTIVE samples
// [32 l, 32 l + 32) (one swizzled 128-byte TMA row, as in pool_block.cu).
// A doubling level w is then register adds, with the w (w < 32) or all 32
// (w >= 32) partners that sit in a later lane fetched by __shfl_down_sync.
// The partials of the lower set bits are needed only after P_W, and keeping
// them all would take up to 8 windows of shared memory per warp: the largest
// one is captured on the way up (lane-striped, in registers), the others are
// RECOMPUTED from the tile (still in shared memory) when their turn comes --
// k = 255 costs 22 doubling levels instead of 7.  Each partial passes through a
// 33-float-pitch staging window (conflict-free blocked writes) and is read
// lane-striped at the runtime offset width, which is a per-lane base plus
// immediate row offsets; the running sums stay in registers lane-striped,
// so the final stores are coalesced.  Averages divide by float32(k) with
// the exact reciprocal + FMA correction of common.cuh (div_all_by_k).
//
// The tiles, ring and CTA walk are those of pool_block.cu: 8 warps, windows
// advancing by V = 1024 - B samples (B = the next power of two >= k), a
// 2-deep TMA ring refilled by the last warp done with a slot.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {

constexpr int kWarps = 8;
constexpr int kT = 32;           // consecutive samples per lane
constexpr int kWin = 32 * kT;    // samples per warp window
constexpr int kPitch = 33;       // staging row (floats): conflict-free both ways
constexpr int kNbuf = 2;

template <int B>
struct XGeo {
  static constexpr int V = kWin - B;                            // outputs per warp
  static constexpr int kOutLanes = V / 32;                      // register slots per lane
  static constexpr int kRows = ((kWarps - 1) * V + kWin) / 32;  // TMA box rows
  static constexpr int kBuf = (kRows * 128 + 1023) / 1024 * 1024;
  static constexpr int kStage = 32 * kPitch;                    // floats per warp
  static_assert(kRows <= 256, "TMA box rows");
};

__device__ __forceinline__ void load_lane_row(const unsigned char* rowp, int swz,
                                              float (&c)[kT]) {
#pragma unroll
  for (int q = 0; q < kT / 4; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(rowp + ((q ^ swz) << 4));
    c[4 * q] = v.x;
    c[4 * q + 1] = v.y;
    c[4 * q + 2] = v.z;
    c[4 * q + 3] = v.w;
  }
}

// c = P_from on entry, P_upto on exit (powers of two, upto < 2 * kMaxW):
// level w -> 2w is c(j) = c(j) + c(j + w), pooling.py:37-41
template <int kMaxW>
__device__ __forceinline__ void doubling(float (&c)[kT], int upto, int from = 1) {
#pragma unroll
  for (int w = 1; w < kMaxW; w <<= 1) {
    if (w >= upto) break;  // warp-uniform
    if (w < from) continue;
    if (w < kT) {
      // partners of the last w registers live in lane + 1; fetch them first
      float sh[kT];
#pragma unroll
      for (int r = kT - w; r < kT; ++r) sh[r] = __shfl_down_sync(0xffffffffu, c[r + w - kT], 1);
#pragma unroll
      for (int r = 0; r < kT; ++r) c[r] = __fadd_rn(c[r], r + w < kT ? c[r + w] : sh[r]);
    } else {
#pragma unroll
      for (int r = 0; r < kT; ++r) c[r] = __fadd_rn(c[r], __shfl_down_sync(0xffffffffu, c[r], w / kT));
    }
  }
}

template <int B, int kOp>
__global__ void __launch_bounds__(32 * kWarps, 2)
    pool_exact_sum_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                          int64_t out_len, int64_t tiles_per_row, int64_t n_tiles,
                          int tiles_per_cta, int k, int64_t flat_L, int64_t y_pitch,
                          const float* __restrict__ acc_in, int64_t acc_pitch, int64_t shift,
                          float fk, int k_out) {
  using G = XGeo<B>;
  constexpr int V = G::V;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kNbuf];
  __shared__ int done_cnt[kNbuf];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  float* stage_all = reinterpret_cast<float*>(base + kNbuf * G::kBuf);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned tpr = (unsigned)tiles_per_row;
  const unsigned t_begin = blockIdx.x * (unsigned)tiles_per_cta;
  const unsigned nt = (unsigned)min(n_tiles, (int64_t)t_begin + tiles_per_cta);
  auto issue = [&](unsigned t, int b) {
    const unsigned row = t / tpr;
    const int64_t s0 = (int64_t)(t - row * tpr) * (kWarps * V);  // 64-bit: flat batches exceed 2^32 samples
    mbar_arrive_expect_tx(&full_bar[b], G::kRows * 128);
    tma_load_3d(base + b * G::kBuf, &tmap, &full_bar[b], 0, (int)((s0 + shift) / 32), (int)row);
  };
  if (tid == 0) {
    prefetch_tmap(&tmap);
    for (int i = 0; i < kNbuf; ++i) {
      mbar_init(&full_bar[i], 1);
      done_cnt[i] = 0;
    }
    fence_mbar_init();
    for (int i = 0; i < kNbuf && t_begin + i < nt; ++i) issue(t_begin + i, i);
  }
  __syncthreads();

  const int kw = 1 << (31 - __clz(k));     // W: the largest power of two <= k
  const int low = k & (kw - 1);            // the set bits below W
  const int bit1 = low ? 1 << (31 - __clz(low)) : 0;  // the largest of them
  const float rk = 1.0f / fk;
  const int row0 = (warp * V) / 32 + lane;  // this lane's 128-byte row in the tile
  float* stage = stage_all + warp * G::kStage;
  float* wrow = stage + lane * kPitch;
  int it = 0;
  for (unsigned t = t_begin; t < nt; ++t, ++it) {
    const int b = it % kNbuf;
    mbar_wait(&full_bar[b], (it / kNbuf) & 1);
    const unsigned char* rowp = base + b * G::kBuf + row0 * 128;
    const unsigned row = t / tpr;
    const int64_t o_in_row = (int64_t)(t - row * tpr) * (kWarps * V) + warp * V;
    const int lim = (int)min((int64_t)V, out_len - (int64_t)o_in_row);
    float c[kT];
    float acc[G::kOutLanes];
    if (acc_in) {
      // fold mode (windows > 512, pool1d.cu): acc = the caller's partial sum
      // of the leading bits at i, and the tile starts `shift` samples later;
      // fold every set bit of k (< B) in, largest first, width from 0
      const float* ar = acc_in + (int64_t)row * acc_pitch + o_in_row + lane;
#pragma unroll
      for (int mm = 0; mm < G::kOutLanes; ++mm) acc[mm] = 32 * mm + lane < lim ? ar[32 * mm] : 0.0f;
      int width = 0;
      for (int bit = kw; bit; bit >>= 1) {
        if (!(k & bit)) continue;
        load_lane_row(rowp, row0 & 7, c);
        doubling<B>(c, bit);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < kT; ++r) wrow[r] = c[r];
        __syncwarp();
        const int ld = lane + width;
        const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) acc[mm] = __fadd_rn(acc[mm], sq[kPitch * mm]);
        width += bit;
      }
    } else {
      // The largest lower set bit's partial is captured on the way up to P_W
      // (kept lane-striped in registers, at its fold offset kw): one partial
      // fewer to recompute (k = 255: 22 doubling levels instead of 28).
      float cap[G::kOutLanes];
      load_lane_row(rowp, row0 & 7, c);
      if (bit1) {
        doubling<B>(c, bit1);
#pragma unroll
        for (int r = 0; r < kT; ++r) wrow[r] = c[r];
        __syncwarp();
        const int ld = lane + kw;
        const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) cap[mm] = sq[kPitch * mm];
        __syncwarp();
        doubling<B>(c, kw, bit1);
      } else {
        doubling<B>(c, kw);
      }
      // acc = P_W(i), i = 32 mm + lane (lane-striped)
#pragma unroll
      for (int r = 0; r < kT; ++r) wrow[r] = c[r];
      __syncwarp();
#pragma unroll
      for (int mm = 0; mm < G::kOutLanes; ++mm) acc[mm] = stage[kPitch * mm + lane];
      int width = kw;
      if (bit1) {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) acc[mm] = __fadd_rn(acc[mm], cap[mm]);
        width += bit1;
      }
      // the other set bits, largest first: acc = acc + P_bit(i + width)
      for (int bit = (bit1 ? bit1 : kw) >> 1; bit; bit >>= 1) {
        if (!(k & bit)) continue;
        load_lane_row(rowp, row0 & 7, c);
        doubling<B>(c, bit);
        __syncwarp();  // everyone done reading the previous partial
#pragma unroll
        for (int r = 0; r < kT; ++r) wrow[r] = c[r];
        __syncwarp();
        const int ld = lane + width;
        const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) acc[mm] = __fadd_rn(acc[mm], sq[kPitch * mm]);
        width += bit;
      }
    }
    __syncwarp();
    if (lane == 0) {  // done with slot b: the last warp refills it
      __threadfence_block();
      if (atomicAdd(&done_cnt[b], 1) == kWarps - 1) {
        done_cnt[b] = 0;
        if (t + kNbuf < nt) {
          fence_proxy_async();
          issue(t + kNbuf, b);
        }
      }
    }
    if constexpr (kOp == SC_POOL_AVG) div_all_by_k<G::kOutLanes>(acc, fk, rk);
    float* yr = y + (int64_t)row * y_pitch + o_in_row + lane;
    if (flat_L) {
      // flat-batch mode (signal length not a multiple of 32, as in
      // pool_block.cu): warps inside one signal's kept range store from a
      // shifted base, boundary warps element by element
      const int64_t w0 = (int64_t)o_in_row, wb = w0 / flat_L;
      if (w0 + lim - 1 < wb * flat_L + flat_L - (k_out - 1)) {
        yr = y + (w0 - wb * (k_out - 1)) + lane;
      } else {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) {
          const int64_t p = w0 + 32 * mm + lane, pb = p / flat_L;
          if (32 * mm + lane < lim && p - pb * flat_L < flat_L - (k_out - 1))
            y[p - pb * (k_out - 1)] = acc[mm];
        }
        __syncwarp();
        continue;
      }
    }
    if (lim == V) {
#pragma unroll
      for (int mm = 0; mm < G::kOutLanes; ++mm) yr[32 * mm] = acc[mm];
    } else {
#pragma unroll
      for (int mm = 0; mm < G::kOutLanes; ++mm)
        if (32 * mm + lane < lim) yr[32 * mm] = acc[mm];
    }
    __syncwarp();  // staging reused by the next tile
  }
}

template <int B, int kOp>
int launch(const float* x, int64_t batch, int64_t length, int k, float* y, cudaStream_t st,
           int64_t flat_L, int64_t out_len, int64_t y_pitch, const float* acc_in,
           int64_t acc_pitch, int64_t shift, float fk, int k_out) {
  using G = XGeo<B>;
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[3] = {32, (cuuint64_t)(length / 32), (cuuint64_t)batch};
  cuuint64_t strides[2] = {128, (cuuint64_t)length * sizeof(float)};
  cuuint32_t box[3] = {32, (cuuint32_t)G::kRows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "pool exact tensor map encode failed");
  const int64_t tiles_per_row = (out_len + kWarps * G::V - 1) / (kWarps * G::V);
  const int64_t n_tiles = tiles_per_row * batch;
  if (n_tiles >= 0x7fffffff) return 1;
  const size_t smem = 1024 + kNbuf * (size_t)G::kBuf + (size_t)kWarps * G::kStage * sizeof(float);
  static uint64_t attr = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(pool_exact_sum_kernel<B, kOp>, smem, &attr));
  const int tpc = 8;  // contiguous tiles per CTA
  const int64_t grid = (n_tiles + tpc - 1) / tpc;
  pool_exact_sum_kernel<B, kOp><<<(unsigned)grid, 32 * kWarps, smem, st>>>(
      map, y, out_len, tiles_per_row, n_tiles, tpc, k, flat_L, y_pitch, acc_in, acc_pitch, shift, fk,
      k_out);
  SC_LAUNCH_CHECK("pool_exact_sum_kernel");
  return SC_OK;
}

template <int kOp>
int dispatch(const float* x, int64_t batch, int64_t length, int k, float* y, cudaStream_t st,
             int64_t flat_L, int64_t out_len, int64_t y_pitch, const float* acc_in,
             int64_t acc_pitch, int64_t shift, float fk, int k_out) {
#define SC_EXACT_LAUNCH(B)                                                                   \
  launch<B, kOp>(x, batch, length, k, y, st, flat_L, out_len, y_pitch, acc_in, acc_pitch, shift, \
                 fk, k_out)
  if (k <= 64) return SC_EXACT_LAUNCH(64);
  if (k <= 128) return SC_EXACT_LAUNCH(128);
  if (k <= 256) return SC_EXACT_LAUNCH(256);
  return SC_EXACT_LAUNCH(512);
#undef SC_EXACT_LAUNCH
}

}  // namespace

// Bit-exact SUM / AVG for 32 < k <= 512 on 16-byte aligned signals whose
// length is a multiple of 32 (>= 1,024).  Returns SC_OK / an error if it ran,
// 1 if it does not apply.
int pool1d_exact_sum(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st) {
  static const bool off = getenv("SC_POOL_NO_EXACT_BLOCK") != nullptr;
  if (off || (op != SC_POOL_SUM && op != SC_POOL_AVG) || k <= 32 || k > 512 ||
      reinterpret_cast<uintptr_t>(x) % 16 != 0 || length < kWin || batch > 0x7fffffff)
    return 1;
  // signals not a multiple of 32 samples: the batch as one flat signal
  int64_t flat_L = 0;
  if (length % 32 != 0) {
    if ((batch * length) % 32 != 0) return 1;
    flat_L = length;
    length *= batch;
    batch = 1;
  }
  if (length / 32 > 0x7fffffff) return 1;
  const int64_t out_len = length - k + 1;
  return op == SC_POOL_SUM
             ? dispatch<SC_POOL_SUM>(x, batch, length, (int)k, y, st, flat_L, out_len, out_len,
                                     nullptr, 0, 0, (float)k, (int)k)
             : dispatch<SC_POOL_AVG>(x, batch, length, (int)k, y, st, flat_L, out_len, out_len,
                                     nullptr, 0, 0, (float)k, (int)k);
}

// Building blocks of the exact sums for k > 512 (pool1d.cu:
// launch_exact_big), on signals whose length is a multiple of 32 (>= 1,024),
// 16-byte aligned:
//  * fold == nullptr: P_512 (the reference's doubling partial of width 512,
//    pooling.py:37-41) at every position, rows of pitch `y_pitch`;
//  * fold != nullptr: y(i) = (fold(i) + P_b1(i + shift)) + P_b2(i + shift + b1)
//    + ... over the set bits b1 > b2 > .. of `k_small` (< 512), the tile
//    read `shift` samples on (a multiple of 32) -- the low-bit tail of the
//    reference's left fold (pooling.py:42-51), average divided by `k_total`;
//    flat_L != 0: the batch is one flat signal of signals of flat_L samples,
//    outputs straddling two signals are dropped (y is [B][flat_L - k_total + 1]).
int pool1d_exact_sum_part(int op, const float* x, int64_t batch, int64_t length, int k_small,
                          int64_t k_total, const float* fold, int64_t fold_pitch, int64_t shift,
                          float* y, int64_t y_pitch, int64_t flat_L, cudaStream_t st) {
  if ((op != SC_POOL_SUM && op != SC_POOL_AVG) || reinterpret_cast<uintptr_t>(x) % 16 != 0 ||
      length % 32 != 0 || length < kWin || batch > 0x7fffffff || length / 32 > 0x7fffffff ||
      shift % 32 != 0 || k_small < 1 || k_small > 512 || (fold == nullptr && k_small != 512))
    return 1;
  const float fk = (float)k_total;
  if (fold == nullptr)  // a plain sum: P_512
    return dispatch<SC_POOL_SUM>(x, batch, length, 512, y, st, 0, length - 511, y_pitch, nullptr,
                                 0, 0, fk, 512);
  const int64_t out_len = length - k_total + 1;
  return op == SC_POOL_SUM
             ? dispatch<SC_POOL_SUM>(x, batch, length, k_small, y, st, flat_L, out_len, y_pitch, fold,
                                     fold_pitch, shift, fk, (int)k_total)
             : dispatch<SC_POOL_AVG>(x, batch, length, k_small, y, st, flat_L, out_len, y_pitch, fold,
                                     fold_pitch, shift, fk, (int)k_total);
}

}  // namespace sc
