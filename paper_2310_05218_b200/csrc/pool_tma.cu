// TMA-staged, blocked-register sliding-window pooling (the headline path of
// sc_pool1d_f32; replaces pooling.py:28-78 for aligned signals).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <utility>

#include "common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {

// ------------------------------------------------------------- TMA kernel
// pool_tma_kernel: the headline path for 16-byte aligned signals whose
// length is a multiple of 32.  Persistent CTAs of 8 warps stream tiles of
// 8*V outputs: one elected thread issues a 2-D TMA box (rows of 32 floats,
// 128-byte swizzle) per tile into a double-buffered shared-memory ring.  Each
// warp then owns a window of 32*T samples in a BLOCKED register layout (lane
// l holds samples [T*l, T*l + T) of the window, read with conflict-free
// swizzled LDS.128), so a doubling shift by w < T is a register rename for
// T-w of the values and one __shfl_down_sync for the other w -- no selects.
// Results are staged through a padded shared-memory slab and written with
// coalesced 32-bit stores (output rows are not 16-byte aligned).
// Operation order is the reference's, hence bit-exact sums; max runs the
// cheap max.NaN path and re-runs a window with np.maximum's exact operand
// order whenever one of its outputs is zero (the only case -- a +0/-0 tie --
// where the two can differ), hence bit-exact maxima.
constexpr int kTmaWarps = 8;
// kernel "ops" beyond sc_pool_op: 1-D convolution with K taps (BASELINE config 1)
constexpr int kConvFast = 3;
constexpr int kConvExact = 4;
// fused pair: window sums (or averages) AND window maxima of the same tile in
// one pass -- one read of the input, two output streams (sc_pool1d_pair_f32)
constexpr int kPairSum = 5;
constexpr int kPairAvg = 6;

template <int K>
struct Taps1 {
  float f[K];
};
constexpr int kTmaT = 16;                    // samples per lane
constexpr int kTmaWin = 32 * kTmaT;          // samples per warp window
constexpr int kStageStride = kTmaT + 4;      // padded staging row (floats)

__host__ __device__ constexpr int tma_valid(int k) { return kTmaWin - ((k - 1 + 31) / 32) * 32; }
__host__ __device__ constexpr int tma_rows(int k) {
  return ((kTmaWarps - 1) * tma_valid(k) + kTmaWin + 31) / 32;
}
__host__ __device__ constexpr int tma_buf_bytes(int k) { return (tma_rows(k) * 128 + 1023) / 1024 * 1024; }

template <int kOp, bool kExactMax>
__device__ __forceinline__ float bop(float a, float b) {
  if constexpr (kOp == SC_POOL_MAX) {
    if constexpr (kExactMax) return np_max(a, b);
    else return max_nan(a, b);
  } else {
    return __fadd_rn(a, b);
  }
}

// dst[j] = op(dst[j], src shifted by s)[j] in the blocked layout, s < 64.
template <int T, int kOp, bool kEx, int S>
__device__ __forceinline__ void blocked_step(float (&dst)[T], const float (&src)[T]) {
  constexpr int m = S / T;      // whole-lane part of the shift
  constexpr int r = S % T;      // in-lane part
  float nb[T];
  // values from lane + m (registers r..T-1) and lane + m + 1 (registers 0..r-1)
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const int src_j = j + r;
    if (src_j < T) {
      nb[j] = (m == 0) ? src[src_j] : __shfl_down_sync(0xffffffffu, src[src_j], m);
    } else {
      nb[j] = __shfl_down_sync(0xffffffffu, src[src_j - T], m + 1);
    }
  }
#pragma unroll
  for (int j = 0; j < T; ++j) dst[j] = bop<kOp, kEx>(dst[j], nb[j]);
}

template <int T, int kOp, bool kEx, int K>
__device__ __forceinline__ void blocked_pool(float (&s)[T]) {
  if constexpr (kOp == SC_POOL_MAX) {
    // doubling (pooling.py:67-72) then one overlapping combine (:73-76)
    [&]<int... I>(std::integer_sequence<int, I...>) {
      (([&] {
         constexpr int w = 1 << I;
         if constexpr (2 * w <= K) blocked_step<T, kOp, kEx, w>(s, s);
       }()), ...);
    }(std::make_integer_sequence<int, 7>{});
    constexpr int p = 1 << (31 - __builtin_clz(K));
    if constexpr (p < K) blocked_step<T, kOp, kEx, K - p>(s, s);
  } else {
    // doubling with retained partials (pooling.py:36-41), then the
    // largest-bit-first combine (pooling.py:43-51)
    constexpr int lg = 31 - __builtin_clz(K);
    float part[lg > 0 ? lg : 1][T];
    [&]<int... I>(std::integer_sequence<int, I...>) {
      (([&] {
         if constexpr (I < lg) {
           constexpr int w = 1 << I;
           if constexpr ((K & w) != 0) {
#pragma unroll
             for (int j = 0; j < T; ++j) part[I][j] = s[j];
           }
           blocked_step<T, kOp, kEx, w>(s, s);
         }
       }()), ...);
    }(std::make_integer_sequence<int, 7>{});
    [&]<int... I>(std::integer_sequence<int, I...>) {
      (([&] {
         constexpr int b = lg - 1 - I;  // descending bits
         if constexpr (b >= 0 && (K & (1 << b)) != 0) {
           constexpr int width = (K >> (b + 1)) << (b + 1);
           blocked_step<T, kOp, kEx, width>(s, part[b]);
         }
       }()), ...);
    }(std::make_integer_sequence<int, 7>{});
  }
}

// y[j] = sum_i f[i] x[j + i] on the blocked window: the K-1 samples past the
// lane's 16 come from the next lane(s) by shuffle; exact = reference order
// (reference.py:19-22: multiply then add, taps ascending, from 0).
template <int T, int K, bool kExact>
__device__ __forceinline__ void blocked_conv(float (&s)[T], const Taps1<K>& taps) {
  float e[T + K - 1];
#pragma unroll
  for (int j = 0; j < T; ++j) e[j] = s[j];
#pragma unroll
  for (int i = 0; i < K - 1; ++i) e[T + i] = __shfl_down_sync(0xffffffffu, s[i % T], 1 + i / T);
#pragma unroll
  for (int j = 0; j < T; ++j) {
    float a = 0.0f;
#pragma unroll
    for (int i = 0; i < K; ++i) a = mac<kExact>(a, taps.f[i], e[j + i]);
    s[j] = a;
  }
}

template <int kOp, int K, int NBUF>
__global__ void __launch_bounds__(32 * (kTmaWarps + 1))
    pool_tma_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y,
                    float* __restrict__ y2, int64_t out_len, int64_t tiles_per_row, int64_t n_tiles, int tiles_per_cta,
                    const Taps1<K> taps) {
  constexpr int T = kTmaT;
  constexpr int V = tma_valid(K);
  constexpr int BUF = tma_buf_bytes(K);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[NBUF];
  __shared__ __align__(8) uint64_t empty_bar[NBUF];
  unsigned char* base =
      smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // swizzle-128B: 1 KiB aligned
  float* stage_all = reinterpret_cast<float*>(base + NBUF * BUF);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // programmatic dependent launch: the next kernel in the stream may start
  // its prologue now; this one waits for its predecessor (memory visible)
  // after setting up, so back-to-back launches overlap launch latency and
  // prologue with the predecessor's tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid == 0) {
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], kTmaWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // tile t -> (row, first output); 32-bit math (host guarantees the range)
  // CTA b owns the contiguous tiles [b*tpc, min((b+1)*tpc, n)): the hardware
  // block scheduler then keeps the in-flight window of memory contiguous
  // (measured: grid-stride persistent loops lose ~10% HBM bandwidth on B200)
  const unsigned tpr = (unsigned)tiles_per_row;
  const unsigned t_begin = blockIdx.x * (unsigned)tiles_per_cta;
  const unsigned nt = (unsigned)min(n_tiles, (int64_t)t_begin + tiles_per_cta);

  if (warp == kTmaWarps) {
    // ------------- producer warp: one lane streams this CTA's tiles
    if (lane == 0) {
      prefetch_tmap(&tmap);
      int i = 0;
      for (unsigned t = t_begin; t < nt; ++t, ++i) {
        const int b = i % NBUF;
        if (i >= NBUF) mbar_wait_sleep(&empty_bar[b], ((i / NBUF) - 1) & 1);
        const unsigned row = t / tpr;
        const int64_t s0 = (int64_t)(t - row * tpr) * (kTmaWarps * V);  // 64-bit: flat batches exceed 2^32 samples
        mbar_arrive_expect_tx(&full_bar[b], tma_rows(K) * 128);
        tma_load_3d(base + b * BUF, &tmap, &full_bar[b], 0, (int)(s0 / 32), (int)row);
      }
    }
    return;
  }

  // ------------- consumer warps
  const int p0 = warp * V + T * lane;  // this lane's first sample in the buffer
  float* stage = stage_all + warp * (32 * kStageStride);
  const float fk = (float)K;
  const float inv_k = 1.0f / fk;
  constexpr bool kPow2 = (K & (K - 1)) == 0;

  int it = 0;
  for (unsigned t = t_begin; t < nt; ++t, ++it) {
    const int b = it % NBUF;
    mbar_wait(&full_bar[b], (it / NBUF) & 1);
    const unsigned char* buf = base + b * BUF;
    float s[T];
    auto load = [&]() {
#pragma unroll
      for (int q = 0; q < T / 4; ++q) {
        const int p = p0 + 4 * q;
        const int row = p >> 5, chunk = (p & 31) >> 2;
        const float4 v = *reinterpret_cast<const float4*>(buf + row * 128 +
                                                          ((chunk ^ (row & 7)) << 4));
        s[4 * q] = v.x;
        s[4 * q + 1] = v.y;
        s[4 * q + 2] = v.z;
        s[4 * q + 3] = v.w;
      }
    };
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[b]);
    };
    load();
    release();  // the window is in registers: hand the buffer back at once
    // stage (padded rows, conflict-free STS.128) -> coalesced 32-bit stores
    auto emit = [&](float* __restrict__ dst) {
#pragma unroll
      for (int q = 0; q < T / 4; ++q)
        *reinterpret_cast<float4*>(stage + lane * kStageStride + 4 * q) =
            make_float4(s[4 * q], s[4 * q + 1], s[4 * q + 2], s[4 * q + 3]);
      __syncwarp();
      const unsigned row = t / tpr;
      const int64_t o_in_row = (int64_t)(t - row * tpr) * (kTmaWarps * V) + warp * V;
      const int lim = (int)min((int64_t)V, out_len - (int64_t)o_in_row);
      float* yr = dst + (int64_t)row * out_len + o_in_row + lane;
      const float* sp = stage + (lane / T) * kStageStride + (lane % T);
      if (lim == V) {
#pragma unroll
        for (int m = 0; m < V / 32; ++m) yr[32 * m] = sp[(32 / T) * m * kStageStride];
        if constexpr (V % 32 != 0) {
          if (lane < V % 32) yr[32 * (V / 32)] = sp[(32 / T) * (V / 32) * kStageStride];
        }
      } else {
#pragma unroll
        for (int m = 0; m < (V + 31) / 32; ++m)
          if (32 * m + lane < lim) yr[32 * m] = sp[(32 / T) * m * kStageStride];
      }
      __syncwarp();  // staging slab reused by the next output / tile
    };
    auto pool_max = [&]() {
      float s_in[T];
#pragma unroll
      for (int j = 0; j < T; ++j) s_in[j] = s[j];
      blocked_pool<T, SC_POOL_MAX, false, K>(s);
      bool zero = false;
#pragma unroll
      for (int j = 0; j < T; ++j) zero |= (s[j] == 0.0f) && (T * lane + j < V);
      if (__any_sync(0xffffffffu, zero)) {  // rare: redo with np.maximum's order
#pragma unroll
        for (int j = 0; j < T; ++j) s[j] = s_in[j];
        blocked_pool<T, SC_POOL_MAX, true, K>(s);
      }
    };
    auto pool_sum = [&](bool avg) {
      blocked_pool<T, SC_POOL_SUM, false, K>(s);
      if (avg) {
#pragma unroll
        for (int j = 0; j < T; ++j) s[j] = kPow2 ? s[j] * inv_k : s[j];
        if constexpr (!kPow2) div_all_by_k<T>(s, fk, inv_k);
      }
    };
    if constexpr (kOp == kPairSum || kOp == kPairAvg) {
      float keep[T];
#pragma unroll
      for (int j = 0; j < T; ++j) keep[j] = s[j];
      pool_sum(kOp == kPairAvg);
      emit(y);
#pragma unroll
      for (int j = 0; j < T; ++j) s[j] = keep[j];
      pool_max();
      emit(y2);
    } else {
      if constexpr (kOp == SC_POOL_MAX) pool_max();
      else if constexpr (kOp >= kConvFast) blocked_conv<T, K, kOp == kConvExact>(s, taps);
      else pool_sum(kOp == SC_POOL_AVG);
      emit(y);
    }
  }
}

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = getenv(name);
  const int n = e ? atoi(e) : dflt;
  return (n >= lo && n <= hi) ? n : dflt;
}


template <int kOp, int K, int NBUF>
int launch_nbuf(const float* x, int64_t batch, int64_t length, float* y, cudaStream_t st,
                const float* w, float* y2 = nullptr) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[3] = {32, (cuuint64_t)(length / 32), (cuuint64_t)batch};
  cuuint64_t strides[2] = {128, (cuuint64_t)length * sizeof(float)};
  cuuint32_t box[3] = {32, (cuuint32_t)tma_rows(K), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "pool tensor map encode failed");
  constexpr int V = tma_valid(K);
  const int64_t out_len = length - K + 1;
  const int64_t tiles_per_row = (out_len + kTmaWarps * V - 1) / (kTmaWarps * V);
  const int64_t n_tiles = tiles_per_row * batch;
  if (n_tiles >= 0x7fffffff) return 1;  // not applicable: caller falls back
  const size_t smem = 1024 + NBUF * (size_t)tma_buf_bytes(K) +
                      (size_t)kTmaWarps * 32 * kStageStride * sizeof(float);
  static uint64_t attr = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(pool_tma_kernel<kOp, K, NBUF>, (int)smem, &attr));
  // contiguous tiles per CTA, measured per op / window on config 2 and 1
  // (tools/pool_sweep.py, conv_sweep.py): light kernels (few doubling stages,
  // no division) stream best with 2, heavier ones with 4 -- e.g. k = 16 avg
  // 84.5 -> 82.4 us at 2, k = 16 max 88.2 at 2 vs 82.9 at 4, conv1d k = 7
  // 86.0 -> 84.2 us at 2
  constexpr bool kPow2 = (K & (K - 1)) == 0;
  constexpr int kTpcDefault =
      kOp == SC_POOL_SUM ? (K <= 24 ? 2 : 4)
      : kOp == SC_POOL_AVG ? ((kPow2 && K <= 16) || K == 3 ? 2 : 4)
      : kOp == SC_POOL_MAX ? (K <= 8 ? 2 : 4)
      : (kOp == kPairSum || kOp == kPairAvg) ? 4  // k = 16 under sustained load: 129.5 us at 4, 134.2 at 2
      : 2;  // weighted (conv1d) windows
  const int tpc = env_int("SC_POOL_TPC", kTpcDefault, 1, 64);
  const int64_t grid = (n_tiles + tpc - 1) / tpc;
  Taps1<K> taps{};
  if (w)
    for (int i = 0; i < K; ++i) taps.f[i] = w[i];
  SC_CUDA(launch_pdl(pool_tma_kernel<kOp, K, NBUF>, dim3((unsigned)grid),
                     dim3(32 * (kTmaWarps + 1)), smem, st, map, y, y2, out_len, tiles_per_row,
                     n_tiles, tpc, taps));
  SC_LAUNCH_CHECK("pool_tma_kernel");
  return SC_OK;
}

template <int kOp, int K>
int launch_one(const float* x, int64_t batch, int64_t length, float* y, cudaStream_t st,
               const float* w, float* y2 = nullptr) {
  // ring depth 2 with 4 contiguous tiles per CTA measured best (tools/pool_sweep.py)
  return launch_nbuf<kOp, K, 2>(x, batch, length, y, st, w, y2);
}

template <int kOp, int... Ks>
int launch_switch(int k, const float* x, int64_t batch, int64_t length, float* y,
                  cudaStream_t st, std::integer_sequence<int, Ks...>, const float* w = nullptr,
                  float* y2 = nullptr) {
  int rc = -1000;
  ((k == Ks ? (rc = launch_one<kOp, Ks>(x, batch, length, y, st, w, y2), 0) : 0), ...);
  return rc;
}

using ConvTaps = std::integer_sequence<int, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17>;

using Windows = std::integer_sequence<int, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16, 17,
                                      18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31, 32,
                                      33, 64>;

}  // namespace

// Returns SC_OK / an error if the TMA path ran, or 1 if it does not apply.
int pool1d_tma(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
               cudaStream_t st) {
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || length % 32 != 0 || k < 2 || k > 64 ||
      (k > 33 && k != 64) || length / 32 > 0x7fffffff || batch > 0x7fffffff)
    return 1;
  if (length < kTmaWin) return 1;
  int rc;
  switch (op) {
    case SC_POOL_SUM: rc = launch_switch<SC_POOL_SUM>((int)k, x, batch, length, y, st, Windows{}); break;
    case SC_POOL_AVG: rc = launch_switch<SC_POOL_AVG>((int)k, x, batch, length, y, st, Windows{}); break;
    default: rc = launch_switch<SC_POOL_MAX>((int)k, x, batch, length, y, st, Windows{}); break;
  }
  return rc == -1000 ? 1 : rc;
}

// Fused pair (sc_pool1d_pair_f32): y_a = window sums (op_a = SUM) or averages
// (AVG), y_max = window maxima, both from one read of x; each output is
// bit-identical to its single-op launch (same per-op code on the same
// registers).  Returns 1 when the TMA path does not apply.
int pool1d_pair_tma(int op_a, const float* x, int64_t batch, int64_t length, int64_t k,
                    float* y_a, float* y_max, cudaStream_t st) {
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || length % 32 != 0 || k < 2 || k > 64 ||
      (k > 33 && k != 64) || length / 32 > 0x7fffffff || batch > 0x7fffffff)
    return 1;
  if (length < kTmaWin) return 1;
  const int rc = op_a == SC_POOL_AVG
                     ? launch_switch<kPairAvg>((int)k, x, batch, length, y_a, st, Windows{},
                                               nullptr, y_max)
                     : launch_switch<kPairSum>((int)k, x, batch, length, y_a, st, Windows{},
                                               nullptr, y_max);
  return rc == -1000 ? 1 : rc;
}

// 1-D convolution of `rows` signals of `length` samples with k taps (HOST
// pointer w); returns 1 when the TMA path does not apply.
int conv1d_tma(const float* x, int64_t rows, int64_t length, const float* w, int64_t k,
               bool exact, float* y, cudaStream_t st) {
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || length % 32 != 0 || k < 2 || k > 17 ||
      length < kTmaWin || length / 32 > 0x7fffffff || rows > 0x7fffffff ||
      rows * length > (int64_t)1 << 40)
    return 1;
  const int rc = exact ? launch_switch<kConvExact>((int)k, x, rows, length, y, st, ConvTaps{}, w)
                       : launch_switch<kConvFast>((int)k, x, rows, length, y, st, ConvTaps{}, w);
  return rc == -1000 ? 1 : rc;
}

}  // namespace sc
