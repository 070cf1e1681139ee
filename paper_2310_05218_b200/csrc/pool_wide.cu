// Wide-window pooling (33 < k <= 2049): O(1) work per output, independent of k.
//
// Replaces the doubling of pooling.py:28-78 for wide windows (BASELINE config
// 2 sweep, k = 64 / 255), where log2(k) register-doubling stages or a global
// pass per stage would cost far more than the 8 bytes of HBM traffic per
// output.  TMA streams tiles of 4,096 samples (128 swizzled rows of 32
// floats) into a 3-deep ring (thread 0 refills a slot after the CTA barrier
// that shows it consumed), two persistent CTAs per SM own contiguous runs of
// tiles; 8 warps hold the
// tile blocked in registers (16 samples per lane).  Each tile yields
// vt = 4096 - roundup32(k - 1) outputs.
//
//  * SUM / AVG (fast mode): van Herk / Gil-Werman with '+' -- segments of k
//    samples anchored at the tile start, P = running sum from the segment
//    start, S = running sum to the segment end, y(i) = S(i) + P(i + k - 1)
//    (P is stored as 0 at segment ends, which is what the window that starts
//    ON a segment start needs: S(i) alone).  Every output is a sum over its
//    own window's samples only, so an inf / NaN / huge value elsewhere in
//    the tile (or in the neighbouring signal in flat-batch mode) cannot leak
//    into it, and the rounding error scales with the window's own magnitude
//    (measured 2.6e-7 normwise at k = 255 on N(0,1) data; tolerance 1e-5 k).
//    A tile-anchored prefix difference E(i + k) - E(i) was used before: it
//    let one non-finite sample turn every later output of the tile into NaN.
//  * MAX (always bit-exact): van Herk / Gil-Werman -- segments of k samples
//    anchored at the tile start; P = running max from the segment start,
//    S = running max to the segment end (segmented lane / warp / CTA scans),
//    then y(i) = max(S(i), P(i + k - 1)).  Every combine takes (earlier, later)
//    operands, so with np.maximum's tie rule the result is the rightmost
//    maximal element, exactly what the reference's doubling order yields.
//    The fast pass uses max.NaN; if any output of the tile is zero (the only
//    case where the two rules can differ: a +0/-0 tie) the tile is redone
//    with np.maximum semantics.
//  * Persistent CTAs walk grid-strided pairs of contiguous tiles.  Sums on
//    signals whose length is not a multiple of 32 view the batch as one flat
//    signal (kFlat instantiation), dropping the windows that straddle two
//    signals at the store.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

#ifndef SC_WIDE_NBUF
#define SC_WIDE_NBUF 3
#endif

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {

constexpr int kWarps = 8;
constexpr int kT = 16;                 // samples per lane
constexpr int kRows = 128;             // TMA box rows of 32 floats
constexpr int kTile = kRows * 32;      // 4096 samples per tile
constexpr int kBufBytes = kTile * 4;   // 16 KiB
constexpr int kNbuf = SC_WIDE_NBUF;
// X reads at i + k - 1 run up to 2,048 floats past the tile for outputs
// beyond vt (never stored): they land inside arr_s, which follows arr_x
constexpr int kArrBytes = kBufBytes;

// float position -> byte offset in a 128-byte-swizzled array of 32-float rows
__device__ __forceinline__ int swz(int p) {
  const int row = p >> 5, chunk = (p & 31) >> 2;
  return (row << 7) + ((chunk ^ (row & 7)) << 4) + ((p & 3) << 2);
}

__device__ __forceinline__ void bar_consumers() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarps) : "memory");
}

__device__ __forceinline__ bool bar_consumers_or(bool pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred pi, po;\n\t"
      "setp.ne.b32 pi, %1, 0;\n\t"
      "bar.red.or.pred po, 1, %2, pi;\n\t"
      "selp.b32 %0, 1, 0, po;\n\t}"
      : "=r"(r)
      : "r"((int)pred), "n"(32 * kWarps)
      : "memory");
  return r != 0;
}

// combine ops of the segmented scans (a earlier, b later)
constexpr int kCombMaxFast = 0, kCombMaxExact = 1, kCombAdd = 2;
template <int kComb>
__device__ __forceinline__ float mx(float a, float b) {
  if constexpr (kComb == kCombMaxExact) return np_max(a, b);
  else if constexpr (kComb == kCombAdd) return a + b;
  else return max_nan(a, b);
}

// Window op over a tile, every output from its own window's samples only.
// Output i (lane a = i / 16 of the tile, offset r = i % 16) covers
//   [i, end of lane a] + c full lanes + [start of lane b, i + k - 1],
// c = c0 or c0 + 1 with c0 = (k - 1) / 16 - 1 (c = c0 + 1 iff r + (k - 1) % 16
// >= 16).  So with LANE-LOCAL suffix Sf / prefix Pf (no
// segment resets inside a lane: plain register scans) and, per lane L, the op
// of the c0 (G0) or c0 + 1 (G1) lane totals just before L,
//   X(q) = op(G_sel(lane(q)), Pf(q)),   y(i) = op(Sf(i), X(i + k - 1)),
// where the choice sel depends only on q % 16 (j < (k - 1) % 16 -> G1).  G0 / G1
// are sliding windows over the 256 lane totals of the tile: van Herk /
// Gil-Werman at lane granularity (segments of c0 lanes, segmented shuffle
// scans + one cross-warp carry), G0(L) = op(S_T(L - c0), P_T(L - 1)).  Every
// combine is op(earlier, later), so for max ties keep the rightmost maximal
// element (np.maximum's order, pooling.py:70-76) and sums add only window
// samples.  Writes Sf and X to shared memory (swizzled like the tile).
struct WideLane {   // per-lane constants (same for every tile)
  int lg;           // lane index in the tile, 0..255
  int c0;           // full lanes in the shorter window middle
  int km;           // (k - 1) % 16: positions j < km of a lane take G1
  bool seg_start;   // lg % c0 == 0   (lane-total segments of c0 lanes)
  bool seg_end;     // lg % c0 == c0 - 1
  int u;            // lg - c0: first lane of this lane's c0-lane window
  bool u_start;     // u >= 0 and u starts a segment (the window IS a segment)
};

template <int kComb>
__device__ __forceinline__ void wide_tile(const float (&s)[kT], const WideLane& wl, int warp,
                                          int lane, unsigned char* arr_x, unsigned char* arr_s,
                                          float* tot, float* pt, float* st_, float* wagg,
                                          int* wflag) {
  const float kId = kComb == kCombAdd ? 0.0f : -__int_as_float(0x7f800000);  // identity
  // ---- lane-local prefix / suffix (plain scans: no resets inside a lane)
  float pf[kT], sf[kT];
  pf[0] = s[0];
#pragma unroll
  for (int j = 1; j < kT; ++j) pf[j] = mx<kComb>(pf[j - 1], s[j]);
  sf[kT - 1] = s[kT - 1];
#pragma unroll
  for (int j = kT - 2; j >= 0; --j) sf[j] = mx<kComb>(s[j], sf[j + 1]);
  const float T = pf[kT - 1];
  // ---- segmented scans of the lane totals across the warp (segments of c0
  // lanes in tile lane space): P_T from the segment start, S_T to its end
  float pv = T, sv = T;
  int pfl = wl.seg_start, sfl = wl.seg_end;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float upv = __shfl_up_sync(0xffffffffu, pv, d);
    const int upf = __shfl_up_sync(0xffffffffu, pfl, d);
    const float dnv = __shfl_down_sync(0xffffffffu, sv, d);
    const int dnf = __shfl_down_sync(0xffffffffu, sfl, d);
    if (lane >= d && !pfl) {
      pv = mx<kComb>(upv, pv);
      pfl = upf;
    }
    if (lane + d < 32 && !sfl) {
      sv = mx<kComb>(sv, dnv);
      sfl = dnf;
    }
  }
  // ---- across warps: warp aggregates, then a segmented 8-lane scan
  if (lane == 31) {
    wagg[warp] = pv;
    wflag[warp] = pfl;
  }
  if (lane == 0) {
    wagg[kWarps + warp] = sv;
    wflag[kWarps + warp] = sfl;
  }
  bar_consumers();
  {
    // lanes 0..7: P aggregates of warps 0..7 (left to right); lanes 8..15: S
    // aggregates of warps 7..0 (right to left) -- one segmented scan each
    const int w = lane & 7;
    const bool is_s = lane >= 8 && lane < 16;
    float av = kId;
    int af = 0;
    if (lane < 16) {
      av = wagg[is_s ? kWarps + (kWarps - 1 - w) : w];
      af = wflag[is_s ? kWarps + (kWarps - 1 - w) : w];
    }
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      const float uv = __shfl_up_sync(0xffffffffu, av, d);
      const int uf = __shfl_up_sync(0xffffffffu, af, d);
      if (w >= d && !af) {
        av = is_s ? mx<kComb>(av, uv) : mx<kComb>(uv, av);
        af = uf;
      }
    }
    // carry into this warp: inclusive scan at warp - 1 (from the left) and
    // at the mirrored lane of warp + 1 (from the right)
    const float cl = __shfl_sync(0xffffffffu, av, warp > 0 ? warp - 1 : 0);
    const float cr = __shfl_sync(0xffffffffu, av, warp < kWarps - 1 ? 8 + (kWarps - 2 - warp) : 8);
    if (warp > 0 && !pfl) pv = mx<kComb>(cl, pv);
    if (warp < kWarps - 1 && !sfl) sv = mx<kComb>(sv, cr);
  }
  tot[wl.lg] = T;
  pt[wl.lg] = pv;
  st_[wl.lg] = sv;
  bar_consumers();
  // ---- G0 / G1 for this lane: op of the c0 / c0 + 1 lane totals before it
  float g0 = kId, g1 = kId;
  {
    const int u = wl.u;
    if (u >= 0) {
      const float sfx = st_[u];
      g0 = wl.u_start ? sfx : mx<kComb>(sfx, pt[wl.lg - 1]);
      g1 = (u >= 1) ? mx<kComb>(tot[u - 1], g0) : g0;
    }
  }
  // ---- X = op(G_sel, Pf) and Sf to shared memory (swizzled, 16-byte stores)
  const int p0 = wl.lg * kT;
#pragma unroll
  for (int q = 0; q < kT / 4; ++q) {
    float4 x4, s4;
    x4.x = mx<kComb>((4 * q + 0 < wl.km) ? g1 : g0, pf[4 * q + 0]);
    x4.y = mx<kComb>((4 * q + 1 < wl.km) ? g1 : g0, pf[4 * q + 1]);
    x4.z = mx<kComb>((4 * q + 2 < wl.km) ? g1 : g0, pf[4 * q + 2]);
    x4.w = mx<kComb>((4 * q + 3 < wl.km) ? g1 : g0, pf[4 * q + 3]);
    s4 = make_float4(sf[4 * q], sf[4 * q + 1], sf[4 * q + 2], sf[4 * q + 3]);
    *reinterpret_cast<float4*>(arr_x + swz(p0 + 4 * q)) = x4;
    *reinterpret_cast<float4*>(arr_s + swz(p0 + 4 * q)) = s4;
  }
  bar_consumers();
}

template <int kOp, bool kFlat>
__global__ void __launch_bounds__(32 * kWarps, 2)
    pool_wide_kernel(const __grid_constant__ CUtensorMap tmap, float* __restrict__ y, int k,
                     int64_t out_len, int64_t tiles_per_row, int64_t n_tiles, int tiles_per_cta,
                     int vt, int64_t flat_L) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[kNbuf];
  __shared__ float tot[kWarps * 32], pt[kWarps * 32], st_[kWarps * 32];
  __shared__ float wagg[2 * kWarps];
  __shared__ int wflag[2 * kWarps];
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* arr_x = base + kNbuf * kBufBytes;   // X (op of window middle + lane prefix)
  unsigned char* arr_s = arr_x + kArrBytes;         // Sf (lane-local suffix)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const unsigned tpr = (unsigned)tiles_per_row;
  // persistent CTAs: groups of tiles_per_cta contiguous tiles, grid-strided
  // (a CTA per group paid a pipeline fill -- the first tile's full load
  // latency -- every few tiles).  Iteration i of this CTA handles tile
  // tile_of(i) while it < n_tiles (only the last group can be short).
  const unsigned n_t = (unsigned)n_tiles, tpc = (unsigned)tiles_per_cta;
  const unsigned g_stride = gridDim.x * tpc;
  auto tile_of = [&](unsigned i) { return blockIdx.x * tpc + (i / tpc) * g_stride + i % tpc; };
  // No producer warp (a 9th warp would cap the CTA at 96 registers for two
  // CTAs per SM: 5 warps on one SM sub-partition): thread 0 refills a ring
  // slot once a CTA barrier shows every warp has its tile in registers.
  auto issue = [&](unsigned i) {
    const unsigned t = tile_of(i);
    if (t >= n_t) return;
    const int b = i % kNbuf;
    const unsigned row = t / tpr;
    const int64_t s0 = (int64_t)(t - row * tpr) * vt;  // 64-bit: flat batches exceed 2^32 samples
    mbar_arrive_expect_tx(&full_bar[b], kBufBytes);
    tma_load_3d(base + b * kBufBytes, &tmap, &full_bar[b], 0, (int)(s0 / 32), (int)row);
  };
  if (tid == 0) {
    prefetch_tmap(&tmap);
    for (int i = 0; i < kNbuf; ++i) mbar_init(&full_bar[i], 1);
    fence_mbar_init();
    for (int i = 0; i < kNbuf; ++i) issue(i);
  }
  __syncthreads();
  auto refill = [&](unsigned i) {  // after a CTA barrier: slot i % kNbuf is free
    if (tid == 0) {
      fence_proxy_async();
      issue(i + kNbuf);
    }
  };

  WideLane wl;
  wl.lg = warp * 32 + lane;
  wl.c0 = (k - 1) / kT - 1;  // >= 1 for k > 32
  wl.km = (k - 1) % kT;
  wl.seg_start = wl.lg % wl.c0 == 0;
  wl.seg_end = wl.lg % wl.c0 == wl.c0 - 1;
  wl.u = wl.lg - wl.c0;
  wl.u_start = wl.u >= 0 && wl.u % wl.c0 == 0;
  const int p0 = wl.lg * kT;
  const float inv_k = 1.0f / (float)k;
  // output loop addresses: output m of this lane is i = warp*512 + 32 m + lane;
  // swz() repeats every 8 rows, so 8 byte offsets per array (+1024 B per 8 m)
  // serve all 16 reads of Sf(i) and of X(i + k - 1)
  int off_s[8], off_x[8];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int i = warp * (32 * kT) + 32 * m + lane;
    off_s[m] = swz(i);
    off_x[m] = swz(i + k - 1);
  }

  for (unsigned it = 0;; ++it) {
    const unsigned t = tile_of(it);
    if (t >= n_t) break;
    const int b = it % kNbuf;
    mbar_wait(&full_bar[b], (it / kNbuf) & 1);
    const unsigned char* buf = base + b * kBufBytes;
    float s[kT];
    auto load = [&]() {
#pragma unroll
      for (int q = 0; q < kT / 4; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(buf + swz(p0 + 4 * q));
        s[4 * q] = v4.x;
        s[4 * q + 1] = v4.y;
        s[4 * q + 2] = v4.z;
        s[4 * q + 3] = v4.w;
      }
    };
    load();

    const unsigned row = t / tpr;
    const int64_t o0 = (int64_t)(t - row * tpr) * vt;
    float* yr = y + (int64_t)row * out_len + o0;
    const int lim = (int)min((int64_t)vt, out_len - o0);
    auto out_at = [&](int m) {  // y(i) read back from shared memory
      return mx<kOp == SC_POOL_MAX ? kCombMaxFast : kCombAdd>(
          *reinterpret_cast<const float*>(arr_s + off_s[m & 7] + (m >> 3) * 1024),
          *reinterpret_cast<const float*>(arr_x + off_x[m & 7] + (m >> 3) * 1024));
    };

    if constexpr (kOp == SC_POOL_MAX) {
      // fast pass (max.NaN), stored at once; if any output of the tile is zero
      // (a +0/-0 tie may resolve differently) the tile -- still in registers --
      // is redone with np.maximum semantics
      wide_tile<kCombMaxFast>(s, wl, warp, lane, arr_x, arr_s, tot, pt, st_, wagg, wflag);
      refill(it);  // wide_tile's barriers: every warp has its samples in registers
      bool zero = false;
#pragma unroll
      for (int m = 0; m < kT; ++m) {
        const int i = warp * (32 * kT) + 32 * m + lane;
        if (i < lim) {
          const float o = out_at(m);
          zero |= (o == 0.0f);
          yr[i] = o;
        }
      }
      if (bar_consumers_or(zero)) {
        wide_tile<kCombMaxExact>(s, wl, warp, lane, arr_x, arr_s, tot, pt, st_, wagg, wflag);
#pragma unroll
        for (int m = 0; m < kT; ++m) {
          const int i = warp * (32 * kT) + 32 * m + lane;
          if (i < lim)
            yr[i] = np_max(*reinterpret_cast<const float*>(arr_s + off_s[m & 7] + (m >> 3) * 1024),
                           *reinterpret_cast<const float*>(arr_x + off_x[m & 7] + (m >> 3) * 1024));
        }
        bar_consumers();
      }
    } else {
      wide_tile<kCombAdd>(s, wl, warp, lane, arr_x, arr_s, tot, pt, st_, wagg, wflag);
      refill(it);  // wide_tile's barriers: every warp has its samples in registers
      float o[kT];
#pragma unroll
      for (int m = 0; m < kT; ++m) o[m] = out_at(m);  // reads past the tile: unused
      if constexpr (kOp == SC_POOL_AVG) {
        // fast mode only (exact mode never reaches this kernel): multiply by
        // the reciprocal
#pragma unroll
        for (int m = 0; m < kT; ++m) o[m] *= inv_k;
      }
      float* ys = yr;
      if constexpr (kFlat) {
        // flat-batch mode (SUM / AVG only): flat output p of signal p / L is
        // kept iff p % L <= L - k, at y[p - (p / L)(k - 1)].  Tiles (3,840+
        // outputs) inside one signal's kept range store from a shifted base;
        // the few that straddle a boundary go element by element.
        const int64_t tb = o0 / flat_L;
        if (o0 + lim - 1 < tb * flat_L + flat_L - (k - 1)) {
          ys = y + o0 - tb * (k - 1);
        } else {
#pragma unroll
          for (int m = 0; m < kT; ++m) {
            const int i = warp * (32 * kT) + 32 * m + lane;
            const int64_t p = o0 + i, b2 = p / flat_L;
            if (i < lim && p - b2 * flat_L < flat_L - (k - 1)) y[p - b2 * (k - 1)] = o[m];
          }
          continue;
        }
      }
      if (warp * (32 * kT) + 32 * kT <= lim) {  // whole warp in range: no per-output checks
#pragma unroll
        for (int m = 0; m < kT; ++m) ys[warp * (32 * kT) + 32 * m + lane] = o[m];
      } else {
#pragma unroll
        for (int m = 0; m < kT; ++m) {
          const int i = warp * (32 * kT) + 32 * m + lane;
          if (i < lim) ys[i] = o[m];
        }
      }
    }
  }
}

// flat_L > 0: `batch` signals of flat_L samples viewed as one signal (batch = 1)
template <int kOp>
int launch(const float* x, int64_t batch, int64_t length, int64_t k, float* y, cudaStream_t st,
           int64_t flat_L = 0) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  cuuint64_t dims[3] = {32, (cuuint64_t)(length / 32), (cuuint64_t)batch};
  cuuint64_t strides[2] = {128, (cuuint64_t)length * sizeof(float)};
  cuuint32_t box[3] = {32, (cuuint32_t)kRows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "pool wide tensor map encode failed");
  const int vt = kTile - (int)((k - 1 + 31) / 32) * 32;
  const int64_t out_len = length - k + 1;
  const int64_t tiles_per_row = (out_len + vt - 1) / vt;
  const int64_t n_tiles = tiles_per_row * batch;
  if (n_tiles >= 0x7fffffff) return 1;
  const size_t smem = 1024 + (size_t)kNbuf * kBufBytes + (size_t)kArrBytes * 2;
  static uint64_t attr = 0, attr_flat = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(pool_wide_kernel<kOp, false>, (int)smem, &attr, 100));
  if constexpr (kOp != SC_POOL_MAX)
    SC_CUDA(set_smem_limit_once(pool_wide_kernel<kOp, true>, (int)smem, &attr_flat, 100));
  static const int tpc = [] {  // contiguous tiles per CTA (SC_WIDE_TPC)
    const char* e = std::getenv("SC_WIDE_TPC");
    const int n = e ? std::atoi(e) : 0;
    return (n >= 1 && n <= 1024) ? n : 2;
  }();
  const int64_t grid = std::min<int64_t>((n_tiles + tpc - 1) / tpc,
                                         (int64_t)sm_count() * 2);
  if constexpr (kOp != SC_POOL_MAX) {  // flat-batch mode: sums / averages only
    if (flat_L) {
      pool_wide_kernel<kOp, true><<<(unsigned)grid, 32 * kWarps, smem, st>>>(
          map, y, (int)k, out_len, tiles_per_row, n_tiles, tpc, vt, flat_L);
      SC_LAUNCH_CHECK("pool_wide_kernel");
      return SC_OK;
    }
  }
  pool_wide_kernel<kOp, false><<<(unsigned)grid, 32 * kWarps, smem, st>>>(
        map, y, (int)k, out_len, tiles_per_row, n_tiles, tpc, vt, 0);
  SC_LAUNCH_CHECK("pool_wide_kernel");
  return SC_OK;
}

}  // namespace

// Returns SC_OK / an error if the wide path ran, or 1 if it does not apply.
int pool1d_wide(int op, const float* x, int64_t batch, int64_t length, int64_t k, float* y,
                cudaStream_t st) {
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || k <= 32 || k > 2049 ||
      batch > 0x7fffffff || batch * length > (int64_t)1 << 40)
    return 1;
  // signals not a multiple of 32 samples (sums / averages): the batch as one
  // flat signal (B L % 32 == 0), outputs straddling two signals dropped
  int64_t flat_L = 0;
  if (length % 32 != 0) {
    if (op == SC_POOL_MAX || (batch * length) % 32 != 0 || length < 4096) return 1;
    flat_L = length;
    length *= batch;
    batch = 1;
  }
  if (length / 32 > 0x7fffffff) return 1;
  switch (op) {
    case SC_POOL_SUM: return launch<SC_POOL_SUM>(x, batch, length, k, y, st, flat_L);
    case SC_POOL_AVG: return launch<SC_POOL_AVG>(x, batch, length, k, y, st, flat_L);
    default: return launch<SC_POOL_MAX>(x, batch, length, k, y, st);
  }
}

}  // namespace sc
