// Aligned-block sliding-window max for windows of k = B - 1 or B samples,
// B in {64, 128, 256, 512} (BASELINE config 2's k = 255 sweep point; replaces
// pooling.py:60-78 for those windows, bit-exact), and for every other window
// 34 <= k <= 512 as k = A + d (A = 32 / 64 / 128 / 256 the largest power of
// two below k): the window-A kernel stages y_A in shared memory and the
// store loop emits max(y_A(i), y_A(i + d)) -- two overlapping windows that
// cover [i, i + k - 1] (k = 100: 148 -> 94 us, k = 200: 166 -> 99 us, k = 40:
// 109 -> 91 us against the striped doubling they replace).
//
// Van Herk / Gil-Werman with the blocks aligned to the register layout: a
// warp holds a window of 1,024 samples, lane l the 32 CONSECUTIVE samples
// [32 l, 32 l + 32) (read from the swizzled TMA tile with four conflict-free
// LDS.128 ... one 128-byte row per lane), so a block of B samples is B / 32
// whole lanes.  Per lane: a 31-step prefix max P and suffix max S in
// registers, then one segmented shuffle scan of the lane aggregates inside
// each block (log2(B/32) steps, once per lane, not per sample).  Output
// i = 32 l + r is max(S(i), P(i + k - 1)); P(i + k - 1) sits a compile-time
// (lane, register) offset away, one __shfl_down_sync per output.  About 7
// instructions per output against ~40 for the striped log2(k) doubling
// (pool1d.cu), so the kernel is left HBM-bound.
//
// Windows that fall inside one block (i on a block start, or i one past it
// when k = B - 1) take P or S alone.  Every combine is mx(earlier, later);
// with np.maximum's tie rule (common.cuh np_max) that is the rightmost
// maximal element, which is what the reference's doubling order yields.
// The fast pass uses max.NaN; a warp whose outputs include a zero (the only
// case -- a +0/-0 tie -- where the two rules can differ) re-reads its window
// and redoes it with np_max.
//
// Signals whose length is not a multiple of 32 (the 3-D tensor map needs
// 128-byte rows) are processed as ONE flat signal of B L samples: windows
// that straddle two signals are computed and dropped at the store
// (kFlat instantiation).
//
// Tiles of 8 warps x (1024 - B) outputs arrive by one 2-D TMA box each in a
// 2- or 3-deep ring (no producer warp: the last warp done with a slot refills
// it), two 8-warp CTAs per SM, CTAs own contiguous runs of tiles; outputs are
// staged through padded shared memory and written with coalesced stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {

constexpr int kWarps = 8;
constexpr int kT = 32;           // consecutive samples per lane
constexpr int kWin = 32 * kT;    // samples per warp window
constexpr int kPitch = kT + 4;   // staging row (floats), conflict-free STS.128

template <int B>
struct Geo {
  static constexpr int V = kWin - B;                         // outputs per warp
  static constexpr int kOutLanes = V / 32;                   // lanes holding outputs
  static constexpr int kRows = ((kWarps - 1) * V + kWin) / 32;  // TMA box rows
  static constexpr int kBuf = (kRows * 128 + 1023) / 1024 * 1024;
  static constexpr int kStage = kOutLanes * kPitch;          // floats per warp
  // ring depth: 3 where two CTAs per SM still fit in shared memory
  static constexpr int kNbuf = B <= 128 ? 2 : 3;
  static_assert(kRows <= 256, "TMA box rows");
};

// combine ops (a earlier, b later): max.NaN fast pass, np.maximum's rule, or
// '+' (window sums: the same aligned-block structure with a sum combine)
constexpr int kCombMaxFast = 0, kCombMaxExact = 1, kCombAdd = 2;
template <int kComb>
__device__ __forceinline__ float mx(float a, float b) {
  if constexpr (kComb == kCombMaxExact) return np_max(a, b);
  else if constexpr (kComb == kCombAdd) return a + b;
  else return max_nan(a, b);
}
template <bool kExact>
__device__ __forceinline__ float mxb(float a, float b) {  // max only
  return mx<kExact ? kCombMaxExact : kCombMaxFast>(a, b);
}

// Reads the lane's 32 samples (one swizzled 128-byte row of the tile),
// computes y(32 lane + r) and writes the outputs of lanes < V/32 to the
// warp's staging rows; returns whether a valid output was zero.
template <int B, int K, int kEx, bool kAvg = false>
__device__ __forceinline__ bool block_max(const unsigned char* rowp, int swz, int lane,
                                          float* stage_row, int lim, float inv_k = 1.0f) {
  constexpr int LB = B / 32;               // lanes per block
  constexpr int m = (K - 1) / 32, c = (K - 1) % 32;
  constexpr int kOutLanes = (kWin - B) / 32;
  const float kId = kEx == kCombAdd ? 0.0f : -__int_as_float(0x7f800000);  // identity
  float P[kT], S[kT];
#pragma unroll
  for (int q = 0; q < kT / 4; ++q) {
    const float4 v = *reinterpret_cast<const float4*>(rowp + ((q ^ swz) << 4));
    S[4 * q] = v.x;
    S[4 * q + 1] = v.y;
    S[4 * q + 2] = v.z;
    S[4 * q + 3] = v.w;
  }
  P[0] = S[0];
#pragma unroll
  for (int j = 1; j < kT; ++j) P[j] = mx<kEx>(P[j - 1], S[j]);     // lane prefix
#pragma unroll
  for (int j = kT - 2; j >= 0; --j) S[j] = mx<kEx>(S[j], S[j + 1]);  // lane suffix
  // inclusive segmented scans of the lane aggregates inside each block
  // (lane-uniform selects, no divergence)
  const int lb = lane % LB;
  float pv = P[kT - 1], sv = S[0];
#pragma unroll
  for (int d = 1; d < LB; d <<= 1) {
    const float up = __shfl_up_sync(0xffffffffu, pv, d, LB);
    const float dn = __shfl_down_sync(0xffffffffu, sv, d, LB);
    pv = lb >= d ? mx<kEx>(up, pv) : pv;
    sv = lb + d < LB ? mx<kEx>(sv, dn) : sv;
  }
  // exclusive aggregates; identity (-inf) at the block edges
  float pe = __shfl_up_sync(0xffffffffu, pv, 1, LB);
  float se = __shfl_down_sync(0xffffffffu, sv, 1, LB);
  pe = lb > 0 ? pe : kId;
  se = lb < LB - 1 ? se : kId;
#pragma unroll
  for (int j = 0; j < kT; ++j) P[j] = mx<kEx>(pe, P[j]);
#pragma unroll
  for (int j = 0; j < kT; ++j) S[j] = mx<kEx>(S[j], se);
  // y(i) = mx(S(i), P(i + K - 1)); P(i + K - 1) of output register r lives in
  // register (r + c) % 32 of lane + m (+1 when r + c wraps)
  bool zero = false;
#pragma unroll
  for (int q = 0; q < kT / 4; ++q) {
    float o[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = 4 * q + u;
      float pj = (r + c < kT) ? __shfl_down_sync(0xffffffffu, P[(r + c) % kT], m)
                              : __shfl_down_sync(0xffffffffu, P[(r + c) % kT], m + 1);
      float si = S[r];
      if (r == 0) si = lb == 0 ? kId : si;                   // window in one block: P alone
      if (r > 0 && r == B - K) pj = lb == 0 ? kId : pj;      // ends on the block end: S alone
      o[u] = mx<kEx>(si, pj);
      if constexpr (kAvg) o[u] *= inv_k;   // fast-mode average (sums are not bit-exact here)
      if constexpr (kEx == kCombMaxFast) zero |= (o[u] == 0.0f) && (kT * lane + r < lim);
    }
    if (lane < kOutLanes)
      *reinterpret_cast<float4*>(stage_row + 4 * q) = make_float4(o[0], o[1], o[2], o[3]);
  }
  return zero;
}

// kNbuf-deep TMA ring without a producer warp: the first load of each slot
// is issued up front, and the LAST warp to finish with a slot (a shared
// counter) refills it with the CTA's next tile at once.
template <int kOp, int B, int K, bool kFlat>
__global__ void __launch_bounds__(32 * kWarps, 2)
    pool_block_max_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                          int64_t out_len, int64_t tiles_per_row, int64_t n_tiles,
                          int tiles_per_cta, int d, int64_t flat_L) {
  static_assert(kOp == SC_POOL_MAX || true, "");
  // kOp = SUM / AVG (fast mode, K = B - 1 or B only, d == 0): the same
  // structure with '+': every output adds the window's own samples only
  using G = Geo<B>;
  // d > 0: the window is K + d; the warp stages y_K (window K) and stores
  // max(y_K(i), y_K(i + d)) for Vd = floor32(V - d) outputs per warp
  const int V = d ? (G::V - d) & ~31 : G::V;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kNbuf = G::kNbuf;
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
    tma_load_3d(base + b * G::kBuf, &tmap, &full_bar[b], 0, (int)(s0 / 32), (int)row);
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

  const int row0 = (warp * V) / 32 + lane;  // this lane's 128-byte row in the tile
  float* stage = stage_all + warp * G::kStage;
  int it = 0;
  for (unsigned t = t_begin; t < nt; ++t, ++it) {
    const int b = it % kNbuf;
    mbar_wait(&full_bar[b], (it / kNbuf) & 1);
    const unsigned char* rowp = base + b * G::kBuf + row0 * 128;
    const unsigned row = t / tpr;
    const int64_t o_in_row = (int64_t)(t - row * tpr) * (kWarps * V) + warp * V;
    const int lim = (int)min((int64_t)V, out_len - (int64_t)o_in_row);
    float* srow = stage + lane * kPitch;
    const int lim_k = d ? G::V : lim;  // y_K outputs the combine reads
    bool zero = false;
    if constexpr (kOp == SC_POOL_MAX) {
      zero = block_max<B, K, kCombMaxFast>(rowp, row0 & 7, lane, srow, lim_k);
      zero = __any_sync(0xffffffffu, zero);
      if (zero) {  // rare: redo with np.maximum's rule
        __syncwarp();
        block_max<B, K, kCombMaxExact>(rowp, row0 & 7, lane, srow, lim_k);
      }
    } else {
      block_max<B, K, kCombAdd, kOp == SC_POOL_AVG>(rowp, row0 & 7, lane, srow, lim_k,
                                                     1.0f / (float)K);
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
    const float* sp = stage + lane;
    if constexpr (kFlat) {
      // flat-batch mode (signal length not a multiple of 32): the batch is one
      // signal of B L samples; flat output p belongs to signal p / L and is
      // kept iff p % L <= L - k, at y[p - (p / L)(k - 1)]
      const int km1 = K + d - 1;
      // a warp's <= 992 outputs cross at most one signal boundary (L >= 1024):
      // warps entirely inside one signal's kept range (all but ~V / L of
      // them) store exactly as in the aligned mode, from a shifted base
      {
        const int64_t w0 = (int64_t)o_in_row, wb = w0 / flat_L;
        if (w0 + lim - 1 < wb * flat_L + flat_L - km1) {
          float* yr = y + (w0 - wb * km1) + lane;
          if (d == 0) {
#pragma unroll
            for (int mm = 0; mm < G::kOutLanes; ++mm)
              if (32 * mm + lane < lim) yr[32 * mm] = sp[mm * kPitch];
          } else {
            const int ld = lane + d;
            const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
#pragma unroll
            for (int mm = 0; mm < G::kOutLanes; ++mm)
              if (32 * mm + lane < lim)
                yr[32 * mm] = zero ? mxb<true>(sp[mm * kPitch], sq[mm * kPitch])
                                   : mxb<false>(sp[mm * kPitch], sq[mm * kPitch]);
          }
          __syncwarp();
          continue;
        }
      }
      // boundary warps: 32-bit position within the signal, pointer stepped
      const int L32 = (int)flat_L, keep = L32 - km1;
      const int64_t p0 = (int64_t)o_in_row + lane;
      const int64_t bq = p0 / flat_L;
      int rem = (int)(p0 - bq * flat_L);
      float* yp = y + (p0 - bq * km1);
      const int ld = lane + d;
      const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
      const int nv = lim - lane;  // this lane's outputs: 32 mm < nv
#pragma unroll
      for (int mm = 0; mm < G::kOutLanes; ++mm) {
        if (32 * mm < nv && rem < keep) {
          const float v = d == 0 ? sp[mm * kPitch]
                                 : (zero ? mxb<true>(sp[mm * kPitch], sq[mm * kPitch])
                                         : mxb<false>(sp[mm * kPitch], sq[mm * kPitch]));
          *yp = v;
        }
        rem += 32;
        yp += 32;
        if (rem >= L32) rem -= L32, yp -= km1;
      }
      __syncwarp();
      continue;
    }
    float* yr = y + (int64_t)row * out_len + o_in_row + lane;
    if (d == 0) {
      if (lim == V) {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm) yr[32 * mm] = sp[mm * kPitch];
      } else {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm)
          if (32 * mm + lane < lim) yr[32 * mm] = sp[mm * kPitch];
      }
    } else {
      // y(i) = max(y_K(i), y_K(i + d)): i = 32 mm + lane, so i + d sits at
      // row mm + (lane + d) / 32, column (lane + d) % 32 -- a per-lane base
      // and the same immediate row offsets as the plain store
      const int ld = lane + d;
      const float* sq = stage + (ld >> 5) * kPitch + (ld & 31);
      const int lim_d = min(lim, V);
      if (zero) {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm)
          if (32 * mm + lane < lim_d) yr[32 * mm] = mxb<true>(sp[mm * kPitch], sq[mm * kPitch]);
      } else {
#pragma unroll
        for (int mm = 0; mm < G::kOutLanes; ++mm)
          if (32 * mm + lane < lim_d) yr[32 * mm] = mxb<false>(sp[mm * kPitch], sq[mm * kPitch]);
      }
    }
    __syncwarp();  // staging reused by the next tile
  }
}

// k = K + d (d = 0: the plain window K)
// flat_L > 0: x is batch signals of flat_L samples viewed as ONE signal of
// `length` = batch * flat_L samples (batch = 1 here)
template <int B, int K, int kOp = SC_POOL_MAX>
int launch(const float* x, int64_t batch, int64_t length, float* y, cudaStream_t st,
           int d = 0, int64_t flat_L = 0) {
  using G = Geo<B>;
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
  if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "pool block tensor map encode failed");
  const int64_t out_len = length - (K + d) + 1;
  const int vw = d ? (G::V - d) & ~31 : G::V;  // outputs per warp
  const int64_t tiles_per_row = (out_len + kWarps * vw - 1) / (kWarps * vw);
  const int64_t n_tiles = tiles_per_row * batch;
  if (n_tiles >= 0x7fffffff) return 1;
  const size_t smem = 1024 + G::kNbuf * (size_t)G::kBuf + (size_t)kWarps * G::kStage * sizeof(float);
  static uint64_t attr = 0, attr_flat = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(pool_block_max_kernel<kOp, B, K, false>, (int)smem, &attr));
  SC_CUDA(set_smem_limit_once(pool_block_max_kernel<kOp, B, K, true>, (int)smem, &attr_flat));
  // contiguous runs of tiles per CTA (tools/pbcheck.py sweep on config 2:
  // 6 tiles for B = 256, 8 otherwise); env override
  static const int tpc_env = [] {
    const char* e = getenv("SC_POOL_BLOCK_TPC");
    const int n = e ? atoi(e) : 0;
    return (n >= 1 && n <= 4096) ? n : 0;
  }();
  const int tpc = tpc_env ? tpc_env : B == 256 ? 6 : 8;
  const int64_t grid = (n_tiles + tpc - 1) / tpc;
  if (flat_L)
    pool_block_max_kernel<kOp, B, K, true><<<(unsigned)grid, 32 * kWarps, smem, st>>>(
        map, y, out_len, tiles_per_row, n_tiles, tpc, d, flat_L);
  else
    pool_block_max_kernel<kOp, B, K, false><<<(unsigned)grid, 32 * kWarps, smem, st>>>(
        map, y, out_len, tiles_per_row, n_tiles, tpc, d, 0);
  SC_LAUNCH_CHECK("pool_block_max_kernel");
  return SC_OK;
}

// flat view of a batch whose signal length is not a multiple of 32; returns
// false if the batch cannot take the TMA kernels at all
bool block_geometry(const float* x, int64_t& batch, int64_t& length, int64_t& flat_L) {
  flat_L = 0;
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || length < kWin || batch > 0x7fffffff)
    return false;
  if (length % 32 != 0) {
    if ((batch * length) % 32 != 0) return false;
    flat_L = length;
    length *= batch;
    batch = 1;
  }
  return length / 32 <= 0x7fffffff;
}

}  // namespace

// FAST-mode window sums / averages for k = B - 1 or B, B in {128, 256, 512}
// (and k = 63): the aligned-block kernel with a '+' combine -- every output
// is S(i) + P(i + k - 1), sums over its own window only (config 2 k = 255:
// 0.088 ms vs 0.105 for the general lane-granular wide kernel).  Returns
// SC_OK / an error if it ran, 1 if it does not apply.
int pool1d_block_sum(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st) {
  static const bool off = getenv("SC_POOL_NO_BLOCK") != nullptr;
  int64_t flat_L = 0;
  if (off || !block_geometry(x, batch, length, flat_L)) return 1;
  auto go = [&](auto tag) -> int {
    constexpr int kOp = decltype(tag)::value;
    switch (k) {
      case 63: return launch<64, 63, kOp>(x, batch, length, y, st, 0, flat_L);
      case 127: return launch<128, 127, kOp>(x, batch, length, y, st, 0, flat_L);
      case 128: return launch<128, 128, kOp>(x, batch, length, y, st, 0, flat_L);
      case 255: return launch<256, 255, kOp>(x, batch, length, y, st, 0, flat_L);
      case 256: return launch<256, 256, kOp>(x, batch, length, y, st, 0, flat_L);
      case 511: return launch<512, 511, kOp>(x, batch, length, y, st, 0, flat_L);
      case 512: return launch<512, 512, kOp>(x, batch, length, y, st, 0, flat_L);
      default: return 1;
    }
  };
  if (op == SC_POOL_SUM) return go(std::integral_constant<int, SC_POOL_SUM>{});
  if (op == SC_POOL_AVG) return go(std::integral_constant<int, SC_POOL_AVG>{});
  return 1;
}

// Exact sliding max for 34 <= k <= 512 on 16-byte aligned signals whose
// length is a multiple of 32 (>= 1,024); k = B - 1 / B take the one-tiling
// kernels.  Returns
// SC_OK / an error if it ran, 1 if it does not apply.
int pool1d_block_max(const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st) {
  static const bool off = getenv("SC_POOL_NO_BLOCK") != nullptr;
  if (off || reinterpret_cast<uintptr_t>(x) % 16 != 0 || length < kWin || batch > 0x7fffffff)
    return 1;
  // signals not a multiple of 32 samples: the whole batch as one flat signal
  // (needs B L % 32 == 0), outputs that straddle two signals dropped
  int64_t flat_L = 0;
  if (length % 32 != 0) {
    if ((batch * length) % 32 != 0) return 1;
    flat_L = length;
    length *= batch;
    batch = 1;
  }
  if (length / 32 > 0x7fffffff) return 1;
  switch (k) {
    case 63: return launch<64, 63>(x, batch, length, y, st, 0, flat_L);
    case 64: return launch<64, 64>(x, batch, length, y, st, 0, flat_L);
    case 127: return launch<128, 127>(x, batch, length, y, st, 0, flat_L);
    case 128: return launch<128, 128>(x, batch, length, y, st, 0, flat_L);
    case 255: return launch<256, 255>(x, batch, length, y, st, 0, flat_L);
    case 256: return launch<256, 256>(x, batch, length, y, st, 0, flat_L);
    case 511: return launch<512, 511>(x, batch, length, y, st, 0, flat_L);
    case 512: return launch<512, 512>(x, batch, length, y, st, 0, flat_L);
    default: break;
  }
  // any other window 34 .. 512: k = A + d with A = 32 / 64 / 128 / 256 the
  // largest power of two below k: the one-tiling kernel for window A, then
  // max(y_A(i), y_A(i + d)) from the staging rows (the two windows overlap
  // and cover [i, i + k - 1]; taking the later one on ties keeps the
  // rightmost maximal element, as the reference's doubling does)
  if (k > 33 && k <= 512) {  // k <= 33: pool_tma.cu is faster
    if (k <= 64) return launch<32, 32>(x, batch, length, y, st, (int)k - 32, flat_L);
    if (k <= 128) return launch<64, 64>(x, batch, length, y, st, (int)k - 64, flat_L);
    if (k <= 256) return launch<128, 128>(x, batch, length, y, st, (int)k - 128, flat_L);
    return launch<256, 256>(x, batch, length, y, st, (int)k - 256, flat_L);
  }
  return 1;
}

}  // namespace sc
