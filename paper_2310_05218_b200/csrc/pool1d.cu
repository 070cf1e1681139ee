// 1-D sliding-window sum / average / max pooling (replaces pooling.py:28-78).
//
// Three kernels:
//  * pool_reg_kernel  -- the headline path.  One warp owns a chunk of 32*T
//    consecutive samples of one signal in a lane-striped register layout
//    (register j of lane l holds sample base + 32*j + l, so every load and
//    store instruction is a coalesced 128-byte line).  The reference's doubling
//    schedule S_2w(i) = S_w(i) + S_w(i+w) (pooling.py:37-41) and its
//    largest-bit-first combine (pooling.py:43-51) run entirely in registers:
//    a shift by s = 32*m + r is a register re-index by m plus one __shfl_sync
//    rotation by r, so shifts by multiples of 32 are free.  Operation order is
//    the reference's, hence sums are bit-exact; max uses np.maximum's
//    operand order (pooling.py:70,75), hence bit-exact including NaN and +-0.
//  * pool_prefix_kernel -- FAST-mode window sums for very wide windows: O(1)
//    work per output from two float64 scans (backward / forward) that meet at
//    a split point inside every window of the tile, staged in shared memory.
//  * pool_pass_kernel -- one doubling / combine pass over global memory, the
//    reference's numpy pass verbatim; used for EXACT sums with many set bits
//    and for very wide windows.
#include <algorithm>

#include <cstdlib>

#include "common.cuh"

namespace sc {
int pool1d_tma(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
               cudaStream_t st);
int pool1d_pair_tma(int op_a, const float* x, int64_t batch, int64_t length, int64_t k,
                    float* y_a, float* y_max, cudaStream_t st);
int pool1d_block_sum(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st);
int pool1d_wide(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                cudaStream_t st);
int pool1d_exact_sum(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st);
int pool1d_exact_sum_part(int op, const float* x, int64_t batch, int64_t length, int k_small,
                          int64_t k_total, const float* fold, int64_t fold_pitch, int64_t shift,
                          float* y, int64_t y_pitch, int64_t flat_L, cudaStream_t st);
int pool1d_block_max(const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st);
namespace {

constexpr int kWarpsPerBlock = 8;

constexpr int bit_length(int v) { return v <= 0 ? 0 : 1 + bit_length(v >> 1); }

// ------------------------------------------------------------------ shifts
// out[j] = value at striped position (32*j + lane) + s, for s in [0, 32*M).
// Positions past the chunk end read clamped garbage (never stored).
template <int T, int M, bool kStatic>
__device__ __forceinline__ void shifted(const float (&v)[T], float (&out)[T], int s, int lane) {
  const int m = s >> 5;
  const int r = s & 31;
  float a[T + 1];
#pragma unroll
  for (int j = 0; j < T + 1; ++j) {
    // a[j] = v[min(j + m, T - 1)], m in [0, M)
    float t = v[j < T ? j : T - 1];
    if constexpr (kStatic) {
      t = v[(j + m) < T ? (j + m) : T - 1];
    } else {
#pragma unroll
      for (int mm = 1; mm < M; ++mm) {
        if (m == mm) t = v[(j + mm) < T ? (j + mm) : T - 1];
      }
    }
    a[j] = t;
  }
  if (r == 0) {
#pragma unroll
    for (int j = 0; j < T; ++j) out[j] = a[j];
    return;
  }
  const int src = (lane + r) & 31;
  const bool wrap = (lane + r) >= 32;
  float rot[T + 1];
#pragma unroll
  for (int j = 0; j < T + 1; ++j) {
    if (j < T) rot[j] = __shfl_sync(0xffffffffu, a[j], src);
  }
  rot[T] = rot[T - 1];
  // lanes that wrap need the next register of the source lane, which is a[j+1]
  // rotated; a[T] was clamped, so rot[T] is garbage only for invalid positions.
#pragma unroll
  for (int j = 0; j < T; ++j) out[j] = wrap ? rot[j + 1] : rot[j];
}

template <bool kClean>
__device__ __forceinline__ float max_op(float a, float b) {
  if constexpr (kClean) {
    return fmaxf(a, b);  // exact when the chunk holds no NaN and no zero
  } else {
    return np_max(a, b);
  }
}

// kK > 0: compile-time window; kK == 0: runtime k (< 32*M).
template <int kOp, int T, int M, int kK, bool kClean>
__device__ __forceinline__ void pool_chunk(float (&s)[T], int k, int lane) {
  constexpr bool kStatic = kK > 0;
  const int kk = kStatic ? kK : k;
  float tmp[T];
  if constexpr (kOp == SC_POOL_MAX) {
    int w = 1;
#pragma unroll
    for (int st = 0; st < 12; ++st) {
      if (2 * w > kk) break;
      shifted<T, M, kStatic>(s, tmp, w, lane);
#pragma unroll
      for (int j = 0; j < T; ++j) s[j] = max_op<kClean>(s[j], tmp[j]);
      w *= 2;
    }
    if (w < kk) {
      shifted<T, M, kStatic>(s, tmp, kk - w, lane);
#pragma unroll
      for (int j = 0; j < T; ++j) s[j] = max_op<kClean>(s[j], tmp[j]);
    }
  } else {
    // partials P_b for every bit b of k below its leading bit (pooling.py:36-41)
    constexpr int kBits = bit_length(kK > 0 ? kK : 32 * M);
    float part[kBits][T];
    int w = 1;
    int lg = 0;
#pragma unroll
    for (int st = 0; st < kBits; ++st) {
      if (2 * w > kk) break;
      if (kk & w) {
#pragma unroll
        for (int j = 0; j < T; ++j) part[st][j] = s[j];
      }
      shifted<T, M, kStatic>(s, tmp, w, lane);
#pragma unroll
      for (int j = 0; j < T; ++j) s[j] = __fadd_rn(s[j], tmp[j]);
      w *= 2;
      ++lg;
    }
    // combine remaining bits, largest first (pooling.py:43-51)
    int width = w;
#pragma unroll
    for (int st = kBits - 1; st >= 0; --st) {
      if (st < lg && (kk & (1 << st))) {
        shifted<T, M, kStatic>(part[st], tmp, width, lane);
#pragma unroll
        for (int j = 0; j < T; ++j) s[j] = __fadd_rn(s[j], tmp[j]);
        width += 1 << st;
      }
    }
  }
}

template <int kOp, int T, int M, int kK>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
    pool_reg_kernel(const float* __restrict__ x, int64_t batch, int64_t length, int k,
                    float* __restrict__ y, int64_t chunks_per_row) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (gw >= batch * chunks_per_row) return;
  const int kk = kK > 0 ? kK : k;
  const int valid = 32 * T - (kk - 1);
  // host guarantees batch * chunks_per_row < 2^32: 32-bit division
  const unsigned cpr = (unsigned)chunks_per_row;
  const unsigned row = (unsigned)gw / cpr;
  const int64_t base = (int64_t)((unsigned)gw - row * cpr) * valid;
  const int64_t out_len = length - kk + 1;
  const float* xr = x + (int64_t)row * length + base;
  const int64_t avail = length - base;  // samples of this row from base on

  float s[T];
  bool dirty = false;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const int p = 32 * j + lane;
    float v = (kOp == SC_POOL_MAX) ? -INFINITY : 0.0f;
    if (p < avail) v = __ldg(xr + p);
    s[j] = v;
    if constexpr (kOp == SC_POOL_MAX) dirty |= (v == 0.0f) || (v != v);
  }

  if constexpr (kOp == SC_POOL_MAX) {
    if (__any_sync(0xffffffffu, dirty)) {
      pool_chunk<kOp, T, M, kK, false>(s, kk, lane);
    } else {
      pool_chunk<kOp, T, M, kK, true>(s, kk, lane);
    }
  } else {
    pool_chunk<kOp, T, M, kK, true>(s, kk, lane);
  }

  const int64_t lim = min((int64_t)valid, out_len - base);
  float* yr = y + (int64_t)row * out_len + base;
  const float fk = (float)kk;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    const int p = 32 * j + lane;
    if (p < lim) {
      float v = s[j];
      if constexpr (kOp == SC_POOL_AVG) v = __fdiv_rn(v, fk);
      yr[p] = v;
    }
  }
}

// ------------------------------------------------------------ prefix kernel
// FAST window sums (very wide windows, and wide windows the TMA kernel cannot
// take: unaligned pointers / ragged batches).  Every window i of a chunk of
// at most k - 1 outputs [c0, c) contains the split point c, so
//   y(i) = float(S(i) + P(i + k - 1)),  S(i) = sum x[i .. c),  P(m) = sum x[c .. m]
// with S a backward and P a forward float64 inclusive scan.  Each output only
// ever sums samples of its own window: a non-finite or huge sample outside it
// cannot leak in (a prefix difference Q(i + k) - Q(i) would turn every later
// output of the tile into NaN after one inf).
constexpr int kPrefixThreads = 256;
constexpr int kPrefixTile = 2048;

// inclusive scan of xs[lo_g, hi_g) into q[] at the same indices; backward
// (q[i] = sum_{j >= i} x[j]) when kRev
template <bool kRev>
__device__ __forceinline__ void block_scan_f64(const float* xs, double* q, int lo_g, int hi_g,
                                               double* warp_tot) {
  const int n = hi_g - lo_g;
  const int E = (n + kPrefixThreads - 1) / kPrefixThreads;
  const int lo = threadIdx.x * E;
  const int hi = min(lo + E, n);
  auto at = [&](int j) { return kRev ? hi_g - 1 - j : lo_g + j; };
  double run = 0.0;
  for (int j = lo; j < hi; ++j) run += (double)xs[at(j)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[warp] = inc;
  // exclusive prefix of this thread from the lane to its left (inc - run
  // would turn an inf in this thread's own run into inf - inf = NaN)
  double acc = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) acc = 0.0;
  __syncthreads();
  for (int w = 0; w < warp; ++w) acc += warp_tot[w];
  for (int j = lo; j < hi; ++j) {
    acc += (double)xs[at(j)];
    q[at(j)] = acc;
  }
  __syncthreads();  // q complete; warp_tot free for the next scan
}

template <int kOp>
__global__ void __launch_bounds__(kPrefixThreads)
    pool_prefix_kernel(const float* __restrict__ x, int64_t length, int k, float* __restrict__ y,
                       int64_t tiles_per_row) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t row = blockIdx.x / tiles_per_row;
  const int64_t t0 = (blockIdx.x - row * tiles_per_row) * (int64_t)kPrefixTile;
  const int64_t out_len = length - k + 1;
  const int n_out = (int)min((int64_t)kPrefixTile, out_len - t0);
  const int n_in = n_out + k - 1;
  double* q = reinterpret_cast<double*>(smem_raw);  // [n_in]
  float* xs = reinterpret_cast<float*>(q + (kPrefixTile + k));
  const float* xr = x + row * length + t0;
  for (int i = threadIdx.x; i < n_in; i += kPrefixThreads) xs[i] = __ldg(xr + i);
  __shared__ double warp_tot[kPrefixThreads / 32];
  __syncthreads();
  float* yr = y + row * out_len + t0;
  const float fk = (float)k;
  // chunks of at most k - 1 outputs, so one split point lies in every window
  // of a chunk (one chunk for the k > 2,048 windows this kernel is tuned for)
  const int C = min(n_out, k - 1);
  for (int c0 = 0; c0 < n_out; c0 += C) {
    const int cn = min(C, n_out - c0), c = c0 + cn;
    block_scan_f64<true>(xs, q, c0, c, warp_tot);         // S over [c0, c)
    block_scan_f64<false>(xs, q, c, c + k - 1, warp_tot);  // P over [c, c + k - 1)
    for (int i = c0 + threadIdx.x; i < c; i += kPrefixThreads) {
      float v = (float)(q[i] + q[i + k - 1]);
      if (kOp == SC_POOL_AVG) v = __fdiv_rn(v, fk);
      yr[i] = v;
    }
    __syncthreads();  // q is rewritten by the next chunk
  }
}

// --------------------------------------------------------------- pass kernel
// dst[r, i] = op(a[r, i], b[r, i + shift]) for i < n, per-row pitches.
template <int kOp>
__global__ void pool_pass_kernel(const float* __restrict__ a, int64_t pa,
                                 const float* __restrict__ b, int64_t pb, int64_t shift,
                                 float* __restrict__ dst, int64_t pd, int64_t rows, int64_t n,
                                 float scale_div) {
  const int64_t total = rows * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n;
    const int64_t i = idx - r * n;
    const float u = a[r * pa + i];
    const float v = b[r * pb + i + shift];
    float o;
    if constexpr (kOp == SC_POOL_MAX) {
      o = np_max(u, v);
    } else {
      o = __fadd_rn(u, v);
    }
    if (scale_div != 0.0f) o = __fdiv_rn(o, scale_div);
    dst[r * pd + i] = o;
  }
}

template <int kOp>
__global__ void copy_div_kernel(const float* __restrict__ a, int64_t pa, float* __restrict__ dst,
                                int64_t pd, int64_t rows, int64_t n, float scale_div) {
  const int64_t total = rows * n;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / n;
    const int64_t i = idx - r * n;
    float o = a[r * pa + i];
    if (scale_div != 0.0f) o = __fdiv_rn(o, scale_div);
    dst[r * pd + i] = o;
  }
}

// ------------------------------------------------------------------ launch
template <int kOp, int T, int M, int kK>
int launch_reg(const float* x, int64_t batch, int64_t length, int k, float* y,
               cudaStream_t st) {
  const int valid = 32 * T - (k - 1);
  const int64_t out_len = length - k + 1;
  const int64_t chunks = (out_len + valid - 1) / valid;
  const int64_t warps = batch * chunks;
  const int64_t blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (blocks > 0x7fffffffLL || warps >= 0xffffffffLL)
    return fail(SC_ERR_UNSUPPORTED, "pool1d: grid too large");
  pool_reg_kernel<kOp, T, M, kK><<<(unsigned)blocks, 32 * kWarpsPerBlock, 0, st>>>(
      x, batch, length, k, y, chunks);
  SC_LAUNCH_CHECK("pool_reg_kernel");
  return SC_OK;
}

template <int kOp>
int launch_prefix(const float* x, int64_t batch, int64_t length, int k, float* y,
                  cudaStream_t st) {
  const int64_t out_len = length - k + 1;
  const int64_t tiles = (out_len + kPrefixTile - 1) / kPrefixTile;
  const size_t smem = (size_t)(kPrefixTile + k) * sizeof(double) +
                      (size_t)(kPrefixTile + k) * sizeof(float);
  static uint64_t attr = 0;  // devices whose limit is set (one per kOp instantiation)
  SC_CUDA(set_smem_limit_once(pool_prefix_kernel<kOp>, 200 * 1024, &attr));
  if (batch * tiles > 0x7fffffffLL) return fail(SC_ERR_UNSUPPORTED, "pool1d: grid too large");
  pool_prefix_kernel<kOp><<<(unsigned)(batch * tiles), kPrefixThreads, smem, st>>>(
      x, length, k, y, tiles);
  SC_LAUNCH_CHECK("pool_prefix_kernel");
  return SC_OK;
}

inline unsigned pass_grid(int64_t total) {
  int64_t b = (total + 255) / 256;
  int64_t cap = (int64_t)sm_count() * 16;
  return (unsigned)std::max<int64_t>(1, std::min(b, cap));
}

// The reference's pass structure, verbatim, over global memory.
template <int kOp>
int launch_passes(const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                  cudaStream_t st) {
  const int64_t n = length;
  const int64_t out_len = n - k + 1;
  const float div = (kOp == SC_POOL_AVG) ? (float)k : 0.0f;
  if (k == 1) {
    copy_div_kernel<kOp><<<pass_grid(batch * n), 256, 0, st>>>(x, n, y, out_len, batch, n, div);
    SC_LAUNCH_CHECK("copy_div_kernel");
    return SC_OK;
  }
  const size_t bytes = (size_t)batch * n * sizeof(float);
  int lgk = 63 - __builtin_clzll((unsigned long long)k);
  // buffers: cur (doubling), plus one per set bit below the leading bit (sum)
  int nbuf = 2;
  if (kOp != SC_POOL_MAX) nbuf += __builtin_popcountll((unsigned long long)k) - 1;
  float* scratch = nullptr;
  SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&scratch), bytes * nbuf, st));
  float* bufs[2] = {scratch, scratch + (size_t)batch * n};
  float* parts[64] = {nullptr};
  int next_part = 2;
  const float* cur = x;  // pitch n, valid length cur_len
  int64_t cur_len = n;
  int flip = 0;
  int64_t w = 1;
  for (int st_i = 0; st_i < lgk; ++st_i) {
    if (kOp != SC_POOL_MAX && (k & w) && st_i == 0) {
      parts[0] = const_cast<float*>(x);  // S_1 is the input itself
    } else if (kOp != SC_POOL_MAX && (k & w)) {
      float* p = scratch + (size_t)(next_part++) * batch * n;
      copy_div_kernel<kOp><<<pass_grid(batch * cur_len), 256, 0, st>>>(cur, n, p, n, batch,
                                                                       cur_len, 0.0f);
      SC_LAUNCH_CHECK("copy_div_kernel");
      parts[st_i] = p;
    }
    float* dst = bufs[flip];
    flip ^= 1;
    pool_pass_kernel<kOp><<<pass_grid(batch * (cur_len - w)), 256, 0, st>>>(
        cur, n, cur, n, w, dst, n, batch, cur_len - w, 0.0f);
    SC_LAUNCH_CHECK("pool_pass_kernel");
    cur = dst;
    cur_len -= w;
    w *= 2;
  }
  if (kOp == SC_POOL_MAX) {
    // one overlapping combine (pooling.py:73-76), written straight to y
    if (w < k) {
      pool_pass_kernel<kOp><<<pass_grid(batch * out_len), 256, 0, st>>>(
          cur, n, cur, n, k - w, y, out_len, batch, out_len, 0.0f);
    } else {
      copy_div_kernel<kOp><<<pass_grid(batch * out_len), 256, 0, st>>>(cur, n, y, out_len,
                                                                       batch, out_len, 0.0f);
    }
    SC_LAUNCH_CHECK("pool max combine");
  } else {
    int64_t width = w;
    // find the last set bit below the leading bit to know which pass writes y
    int last = -1;
    for (int b = 0; b < lgk; ++b)
      if (k & (1LL << b)) {
        last = b;
        break;
      }
    if (last < 0) {
      copy_div_kernel<kOp><<<pass_grid(batch * out_len), 256, 0, st>>>(cur, n, y, out_len,
                                                                       batch, out_len, div);
      SC_LAUNCH_CHECK("copy_div_kernel");
    }
    for (int b = lgk - 1; b >= 0; --b) {
      if (!(k & (1LL << b))) continue;
      const int64_t bit = 1LL << b;
      const int64_t m = n - (width + bit) + 1;
      const bool final_pass = (b == last);
      float* dst = final_pass ? y : bufs[flip];
      const int64_t pd = final_pass ? out_len : n;
      pool_pass_kernel<kOp><<<pass_grid(batch * m), 256, 0, st>>>(
          cur, n, parts[b], n, width, dst, pd, batch, m, final_pass ? div : 0.0f);
      SC_LAUNCH_CHECK("pool_pass_kernel");
      if (!final_pass) {
        cur = dst;
        flip ^= 1;
      }
      width += bit;
    }
  }
  SC_CUDA(cudaFreeAsync(scratch, st));
  return SC_OK;
}

// Exact sums / averages for k > 512 on aligned signals (length % 32 == 0):
// the reference's arithmetic (pooling.py:37-51) regrouped by who computes
// which partial, every addition the same.  W = the largest power of two
// <= k.  P_512 at every position comes from the tile kernel (one pass over
// x); P_1024 .. P_W are global doubling passes P_2w(i) = P_w(i) + P_w(i + w)
// (the partials of set bits in [512, W) are kept); the fold
// acc = P_W(i) + P_b(i + width) ... runs over those kept partials, and the
// set bits below 512 are folded in by the tile kernel, which recomputes
// their partials from x and reads acc from global memory.  For k = 1,000
// that is 2 launches instead of 14 global passes.
// flat batches (L % 32 != 0, B L % 32 == 0): one signal of B L samples
// (windows straddling two signals are computed and dropped, as in
// pool_exact.cu); results the passes would write to y go through
// flat_compact_kernel instead.
template <int kOp>
__global__ void flat_compact_kernel(const float* __restrict__ src, int64_t flat_L, int64_t k,
                                    int64_t batch, float* __restrict__ y, float scale_div) {
  const int64_t per = flat_L - k + 1, total = batch * per;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / per, i = e - b * per;
    float o = src[b * flat_L + i];
    if (scale_div != 0.0f) o = __fdiv_rn(o, scale_div);
    y[e] = o;
  }
}

template <int kOp>
int launch_exact_big(const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                     cudaStream_t st) {
  static const bool off = getenv("SC_POOL_NO_EXACT_BLOCK") != nullptr;
  if (off || k <= 512 || reinterpret_cast<uintptr_t>(x) % 16 != 0 || batch > 0x7fffffff)
    return 1;
  int64_t flat_L = 0;
  if (length % 32 != 0) {
    if ((batch * length) % 32 != 0) return 1;
    flat_L = length;
    length *= batch;
    batch = 1;
  }
  if (length < 1024 || length / 32 > 0x7fffffff) return 1;
  const int64_t n = length, out_len = n - k + 1;
  const float div = (kOp == SC_POOL_AVG) ? (float)k : 0.0f;
  const int lgw = 63 - __builtin_clzll((unsigned long long)k);
  const int64_t W = 1LL << lgw;
  const int k_small = (int)(k & 511);
  // buffers: two for the doubling chain + one per kept partial (set bits in
  // [512, W)), all of pitch n
  int kept = 0;
  for (int64_t b = 512; b < W; b <<= 1) kept += (k & b) ? 1 : 0;
  const int nbuf = 2 + kept;
  float* scratch = nullptr;
  SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&scratch), (size_t)batch * n * sizeof(float) * nbuf,
                        st));
  auto buf = [&](int i) { return scratch + (size_t)i * batch * n; };
  int free_next = 2;
  float* parts[64] = {nullptr};
  int rc =
      pool1d_exact_sum_part(SC_POOL_SUM, x, batch, n, 512, 512, nullptr, 0, 0, buf(0), n, 0, st);
  if (rc != SC_OK) {
    cudaFreeAsync(scratch, st);
    return rc;
  }
  float* cur = buf(0);
  int spare = 1;  // index of the free chain buffer
  int64_t cur_len = n - 511;
  for (int64_t w = 512; w < W; w <<= 1) {
    float* dst;
    if (k & w) {  // keep P_w: the chain continues in a fresh buffer
      parts[__builtin_ctzll((unsigned long long)w)] = cur;
      dst = buf(free_next < nbuf ? free_next++ : spare);
    } else {
      dst = buf(spare);
    }
    // P_2w from P_w; the last level writes y directly when nothing follows
    const bool last = (2 * w == W) && k == W && !flat_L;
    pool_pass_kernel<kOp><<<pass_grid(batch * (cur_len - w)), 256, 0, st>>>(
        cur, n, cur, n, w, last ? y : dst, last ? out_len : n, batch, cur_len - w,
        last ? div : 0.0f);
    SC_LAUNCH_CHECK("pool_pass_kernel");
    if (last) {
      SC_CUDA(cudaFreeAsync(scratch, st));
      return SC_OK;
    }
    if (!(k & w)) spare = (int)((cur - scratch) / ((size_t)batch * n));
    cur = dst;
    cur_len -= w;
  }
  // the set bits in [512, W), largest first: acc = acc + P_b(i + width)
  int64_t width = W;
  for (int64_t b = W >> 1; b >= 512; b >>= 1) {
    if (!(k & b)) continue;
    const int64_t m = n - (width + b) + 1;
    const bool last = k_small == 0 && (k & (b - 1)) == 0 && !flat_L;
    float* dst = last ? y : buf(spare);
    pool_pass_kernel<kOp><<<pass_grid(batch * m), 256, 0, st>>>(
        cur, n, parts[__builtin_ctzll((unsigned long long)b)], n, width, dst, last ? out_len : n,
        batch, m, last ? div : 0.0f);
    SC_LAUNCH_CHECK("pool_pass_kernel");
    width += b;
    if (last) {
      SC_CUDA(cudaFreeAsync(scratch, st));
      return SC_OK;
    }
    spare = (int)((cur - scratch) / ((size_t)batch * n));
    cur = dst;
  }
  if (k_small == 0) {  // flat batch, k a multiple of 512: compact into y
    flat_compact_kernel<kOp><<<pass_grid(n), 256, 0, st>>>(cur, flat_L, k, n / flat_L, y, div);
    SC_LAUNCH_CHECK("flat_compact_kernel");
    SC_CUDA(cudaFreeAsync(scratch, st));
    return SC_OK;
  }
  // the set bits below 512, in the tile kernel
  rc = pool1d_exact_sum_part(kOp, x, batch, n, k_small, k, cur, n, width, y, out_len, flat_L, st);
  SC_CUDA(cudaFreeAsync(scratch, st));
  return rc;
}

template <int kOp>
int dispatch(const float* x, int64_t batch, int64_t length, int64_t k, int mode, float* y,
             cudaStream_t st) {
  const bool exact = mode == SC_MODE_EXACT;
  // 33 <= k <= 512 on aligned signals: the aligned-block van Herk /
  // Gil-Werman max (pool_block.cu; one tiling for k = B - 1 / B, two otherwise)
  if constexpr (kOp == SC_POOL_MAX) {
    const int rc = pool1d_block_max(x, batch, length, k, y, st);
    if (rc != 1) return rc;
  }
  // TMA-staged blocked kernel: bit-exact doubling order, so it serves both modes
  {
    const int rc = pool1d_tma(kOp, x, batch, length, k, y, st);
    if (rc != 1) return rc;
  }
  // wide windows: O(1) per output -- prefix sums (fast mode) or the exact
  // van Herk / Gil-Werman max.  For 64 < k <= 256 the striped register
  // doubling is still the faster exact max on B200 (k = 255 before the aligned
  // kernel: 179 us unaligned vHGW vs 130 us doubling), so that kernel serves k > 256
  // (SC_POOL_MAX_WIDE_MIN moves the threshold).
  static const int max_wide_min = [] {
    const char* e = getenv("SC_POOL_MAX_WIDE_MIN");
    return e ? atoi(e) : 257;
  }();
  if (kOp != SC_POOL_MAX && !exact) {  // window sums over aligned blocks (k = B - 1 / B)
    const int rc = pool1d_block_sum(kOp, x, batch, length, k, y, st);
    if (rc != 1) return rc;
  }
  if ((kOp == SC_POOL_MAX && k >= max_wide_min) || (kOp != SC_POOL_MAX && !exact)) {
    const int rc = pool1d_wide(kOp, x, batch, length, k, y, st);
    if (rc != 1) return rc;
  }
  // compile-time specialisations for the BASELINE windows
  if (k == 16) return launch_reg<kOp, 16, 1, 16>(x, batch, length, 16, y, st);
  if (k == 3) return launch_reg<kOp, 16, 1, 3>(x, batch, length, 3, y, st);
  if constexpr (kOp == SC_POOL_MAX) {
    if (k == 64) return launch_reg<kOp, 16, 2, 64>(x, batch, length, 64, y, st);
    if (k == 255) return launch_reg<kOp, 32, 8, 255>(x, batch, length, 255, y, st);
    if (k <= 32) return launch_reg<kOp, 16, 1, 0>(x, batch, length, (int)k, y, st);
    if (k <= 64) return launch_reg<kOp, 16, 2, 0>(x, batch, length, (int)k, y, st);
    if (k <= 256) return launch_reg<kOp, 32, 8, 0>(x, batch, length, (int)k, y, st);
    return launch_passes<kOp>(x, batch, length, k, y, st);
  } else {
  // SUM / AVG
  if (k <= 32) return launch_reg<kOp, 16, 1, 0>(x, batch, length, (int)k, y, st);
  if (exact) {
    // 32 < k <= 512 on aligned signals: the reference's doubling + bit
    // folding per tile in registers (pool_exact.cu)
    {
      const int rc = pool1d_exact_sum(kOp, x, batch, length, k, y, st);
      if (rc != 1) return rc;
    }
    // power-of-two windows need no retained partials: doubling only
    if (k == 64) return launch_reg<kOp, 16, 2, 64>(x, batch, length, 64, y, st);
    if (k == 128) return launch_reg<kOp, 32, 4, 128>(x, batch, length, 128, y, st);
    if (k == 256) return launch_reg<kOp, 32, 8, 256>(x, batch, length, 256, y, st);
    {
      const int rc = launch_exact_big<kOp>(x, batch, length, k, y, st);
      if (rc != 1) return rc;
    }
    return launch_passes<kOp>(x, batch, length, k, y, st);
  }
  if (k <= 8192) return launch_prefix<kOp>(x, batch, length, (int)k, y, st);
  return launch_passes<kOp>(x, batch, length, k, y, st);
  }
}

}  // namespace
}  // namespace sc

extern "C" int64_t sc_pool1d_stages(int op, int64_t k) {
  if (k < 1) return -1;
  const int lg = 63 - __builtin_clzll((unsigned long long)k);
  if (op == SC_POOL_MAX) return lg + (((1LL << lg) != k) ? 1 : 0);
  return lg + __builtin_popcountll((unsigned long long)k) - 1;
}

extern "C" int sc_pool1d_f32(int op, const float* x, int64_t batch, int64_t length, int64_t k,
                             int mode, float* y, void* stream) {
  using namespace sc;
  if (op < SC_POOL_SUM || op > SC_POOL_MAX) return fail(SC_ERR_ARG, "pool1d: bad op");
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return fail(SC_ERR_ARG, "pool1d: bad mode");
  if (batch < 0 || length < 1) return fail(SC_ERR_SHAPE, "pool1d: signal length must be >= 1");
  if (k < 1 || k > length)
    return fail(SC_ERR_SHAPE, "window " + std::to_string(k) + " out of range for length " +
                                  std::to_string(length));
  if (batch == 0) return SC_OK;
  if (!x || !y) return fail(SC_ERR_ARG, "pool1d: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (op) {
    case SC_POOL_SUM: return dispatch<SC_POOL_SUM>(x, batch, length, k, mode, y, st);
    case SC_POOL_AVG: return dispatch<SC_POOL_AVG>(x, batch, length, k, mode, y, st);
    default: return dispatch<SC_POOL_MAX>(x, batch, length, k, mode, y, st);
  }
}

// Fused sum-or-average + max pooling: one read of x for both outputs on the
// TMA kernel's windows (k = 2..33, 64 on aligned signals); any other shape runs
// the two single-op paths back to back.  Either way y_a / y_max are
// bit-identical to what sc_pool1d_f32 writes for op_a / SC_POOL_MAX.
extern "C" int sc_pool1d_pair_f32(int op_a, const float* x, int64_t batch, int64_t length,
                                  int64_t k, int mode, float* y_a, float* y_max, void* stream) {
  using namespace sc;
  if (op_a != SC_POOL_SUM && op_a != SC_POOL_AVG)
    return fail(SC_ERR_ARG, "pool1d_pair: first op must be SUM or AVG");
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return fail(SC_ERR_ARG, "pool1d: bad mode");
  if (batch < 0 || length < 1) return fail(SC_ERR_SHAPE, "pool1d: signal length must be >= 1");
  if (k < 1 || k > length)
    return fail(SC_ERR_SHAPE, "window " + std::to_string(k) + " out of range for length " +
                                  std::to_string(length));
  if (batch == 0) return SC_OK;
  if (!x || !y_a || !y_max) return fail(SC_ERR_ARG, "pool1d: null pointer");
  if (y_a == y_max) return fail(SC_ERR_ARG, "pool1d_pair: outputs alias");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rc = pool1d_pair_tma(op_a, x, batch, length, k, y_a, y_max, st);
  if (rc != 1) return rc;
  const int ra = sc_pool1d_f32(op_a, x, batch, length, k, mode, y_a, stream);
  if (ra != SC_OK) return ra;
  return sc_pool1d_f32(SC_POOL_MAX, x, batch, length, k, mode, y_max, stream);
}
