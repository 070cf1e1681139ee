// 2-D single-channel valid convolution for runtime filter sizes (the paper's
// 11..51 sweep, reference bench.py:20; conv2d_slide_compound / _generic /
// conv2d_reference with any kh x kw up to 64 x 64, kernels.py:235-255).
//
// The filter-size-specialised TMA kernels (conv2d.cu) fully unroll KH x KW
// with the taps as constant operands; that does not scale to 51 x 51 = 2,601
// taps.  Here the taps sit in shared memory and the work is register-blocked
// so each shared-memory load feeds many FMAs:
//   * a CTA owns 64 output rows x 128 output columns of one image and stages
//     the (64 + kh - 1) x (128 + kw - 1 (+pad)) input tile and the taps in
//     shared memory;
//   * a thread owns R = 8 output rows x 4 consecutive columns (32 register
//     accumulators); warp w (of 8) owns rows 8w .. 8w+7, lane l columns 4l .. 4l+3,
//     so a warp's LDS.128 of 4 consecutive inputs per lane is 512 contiguous
//     bytes (conflict-free);
//   * the thread walks the input rows q of its band once (rolling
//     accumulators, the custom kernels' reuse, kernels.py:185-206): input row
//     q feeds output rows r with j = q - r in [0, kh).  Along the row it
//     slides an 8-value register window in steps of 4 taps: one LDS.128 of
//     inputs and, per live output row, one broadcast LDS.128 of 4 taps for
//     16 FMAs -- ~14 FMAs per shared-memory load, so the FP32 pipe, not
//     shared memory, is the limit.  The taps are stored block-major so the
//     8 rows' tap loads are immediate offsets from one pointer, and three
//     input blocks rotate through the window so no register moves are
//     needed (k = 25..63: +8-13 % over row-major taps with a shifted window).
//   * kExact: __fmul_rn + __fadd_rn, and every output still accumulates in
//     the reference's order (j ascending as q ascends, i ascending within a
//     row, from 0): bit-identical to _accumulate_taps (reference.py:15-23).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace sc {
namespace {

constexpr int kR = 8;                 // output rows per thread
constexpr int kC = 4;                 // output columns per thread and column group
constexpr int kMaxK = 64;

// kG column groups: lane l owns columns 4l .. 4l+3 of each 128-column group
// (conflict-free LDS.128 per group); a broadcast tap load feeds 16 kG FMAs.
// kG = 2 (8 x 8 outputs per thread, ~120 registers) measured 10-25 % slower
// than kG = 1 on the 11..63 sweep (fewer resident warps), so only kG = 1 is
// instantiated.  Packed FFMA2 on column pairs (as the 7x7 kernel does) also
// measured slower here (-9 %): the shifted input pairs of every 4-tap block
// must be re-made from registers (~55 moves per 64 FFMA2) or re-loaded with
// volatile scalar loads that sit on the block's critical path.
__host__ __device__ constexpr int tile_cols(int g) { return 128 * g; }
__host__ __device__ constexpr int tile_rows(int warps) { return kR * warps; }
__host__ __device__ constexpr int pad4(int v) { return (v + 3) & ~3; }
// tile row pitch: columns read up to 128 (g - 1) + 124 + 3 + (pad4(kw) - 4) + 4
__host__ __device__ constexpr int tile_pitch(int kw, int g) { return tile_cols(g) + pad4(kw) + 4; }
__host__ __device__ constexpr size_t big_smem(int kh, int kw, int warps, int g) {
  return ((size_t)kh * pad4(kw) + (size_t)(tile_rows(warps) + kh - 1) * tile_pitch(kw, g)) * 4;
}

// one 4-tap block for one output row: 16 FMAs against the 8-value window w
template <bool kExact>
__device__ __forceinline__ void block4(float* acc, const float4 t, const float (&w)[8]) {
#pragma unroll
  for (int c = 0; c < kC; ++c) acc[c] = mac<kExact>(acc[c], t.x, w[c]);
#pragma unroll
  for (int c = 0; c < kC; ++c) acc[c] = mac<kExact>(acc[c], t.y, w[c + 1]);
#pragma unroll
  for (int c = 0; c < kC; ++c) acc[c] = mac<kExact>(acc[c], t.z, w[c + 2]);
#pragma unroll
  for (int c = 0; c < kC; ++c) acc[c] = mac<kExact>(acc[c], t.w, w[c + 3]);
}

// the filter travels in the launch parameters (16 KiB < the 32 KiB limit):
// no per-call allocation or pageable copy
struct BigTaps {
  float f[kMaxK * kMaxK];
};

// kWarps = 8 (64-row tiles, less halo, more warps per SM) for big grids;
// 4 when a single image would leave SMs idle
template <bool kExact, int kWarps, int kG, bool kSplit>
__global__ void __launch_bounds__(32 * kWarps)
    conv2d_big_kernel(const float* __restrict__ x, int h, int w,
                      const __grid_constant__ BigTaps ft, int kh_full, int kw,
                      float* __restrict__ y, int oh, int ow, int nsplit, int jstep) {
  constexpr int kTileRows = tile_rows(kWarps);
  constexpr int kTileCols = tile_cols(kG);
  const float* f = ft.f;
  extern __shared__ __align__(16) float smem[];
  const int kwp = pad4(kw);
  const int pitch = tile_pitch(kw, kG);
  // taps, block-major: 4-tap block b of filter row j at taps[(b * kh + j) * 4],
  // so the blocks of the (up to 8) filter rows one input row meets sit at
  // compile-time offsets -16 r bytes from one pointer (no per-row address
  // arithmetic in the inner loop); zero padded past kw
  // nsplit > 1 (fast mode, small grids): CTA slice s convolves filter rows
  // [s jstep, s jstep + kh) only -- the input shifted down by s jstep rows --
  // into its own partial plane of y; a second kernel adds the planes in order
  const int slice = kSplit ? blockIdx.z % nsplit : 0;
  const int img = kSplit ? blockIdx.z / nsplit : blockIdx.z;
  const int j0 = slice * jstep;
  const int kh = kSplit ? min(kh_full, j0 + jstep) - j0 : kh_full;  // filter rows of this slice
  float* taps = smem;
  float* tile = smem + kh * kwp;             // [kTileRows + kh - 1][pitch]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.y * kTileRows, c0 = blockIdx.x * kTileCols;
  const float* xi = x + ((int64_t)img * h + j0) * w;
  float* yi = y + (int64_t)blockIdx.z * oh * ow;  // [img][slice] planes (= img when unsplit)
  if (kSplit) h -= j0;                       // input rows left below the shift

  for (int e = threadIdx.x; e < kh * kwp; e += blockDim.x) {
    const int j = e / kwp, i = e - j * kwp;
    taps[((i >> 2) * kh + j) * 4 + (i & 3)] = i < kw ? f[(j0 + j) * kw + i] : 0.0f;
  }
  const int rows = kTileRows + kh - 1;
  for (int rr = warp; rr < rows; rr += kWarps) {
    const int gr = r0 + rr;
    float* dst = tile + rr * pitch;
    const float* src = xi + (int64_t)gr * w;
    // cp.async: every load of the fill is in flight at once (an LDG -> STS
    // loop waits out the global latency per element: ~6 % of the kernel)
    for (int cc = lane; cc < pitch; cc += 32) {
      const int gc = c0 + cc;
      const bool ok = gr < h && gc < w;
      cp_async4(dst + cc, ok ? src + gc : xi, ok);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  float acc[kR][kG * kC];
#pragma unroll
  for (int r = 0; r < kR; ++r)
#pragma unroll
    for (int c = 0; c < kG * kC; ++c) acc[r][c] = 0.0f;

  const int nfull = kw >> 2, krem = kw & 3;
  const int bstride = kh * 4;  // floats between consecutive tap blocks of one row
  const float* band = tile + warp * kR * pitch + kC * lane;
  // One input row: ALL = every output row of the band is live (kR-1 <= q <=
  // kh-1), so the r loop has no branches and the 8 tap loads can be hoisted
  // ahead of the FMAs; otherwise rows outside [rlo, rhi] are skipped.
  auto row = [&](auto all_tag, int q) {
    constexpr bool ALL = decltype(all_tag)::value;
    const int rlo = max(0, q - kh + 1), rhi = min(kR - 1, q);
    const float4* xr = reinterpret_cast<const float4*>(band + q * pitch);  // group g at + 32 g
    const float* tq = taps + q * 4;  // block 0 of filter row q; row q - r at tq - 4 r
    // one 4-tap block against the windows (u[g], v[g]) of two 4-input blocks
    auto blk = [&](const float4 (&u)[kG], const float4 (&v)[kG], const float* tb) {
      float wv[kG][8];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        wv[g][0] = u[g].x, wv[g][1] = u[g].y, wv[g][2] = u[g].z, wv[g][3] = u[g].w;
        wv[g][4] = v[g].x, wv[g][5] = v[g].y, wv[g][6] = v[g].z, wv[g][7] = v[g].w;
      }
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        if (!ALL && (r < rlo || r > rhi)) continue;  // warp-uniform
        const float4 t = *reinterpret_cast<const float4*>(tb - 4 * r);
#pragma unroll
        for (int g = 0; g < kG; ++g) block4<kExact>(&acc[r][g * kC], t, wv[g]);
      }
    };
    auto ld = [&](float4 (&d)[kG], int bi) {
#pragma unroll
      for (int g = 0; g < kG; ++g) d[g] = xr[bi + 32 * g];
    };
    // three input blocks rotate through (A, B), (B, C), (C, A): no moves
    float4 A[kG], B[kG], C[kG];
    ld(A, 0);
    int b = 0;
    for (; b + 3 <= nfull; b += 3) {
      ld(B, b + 1);
      blk(A, B, tq);
      tq += bstride;
      ld(C, b + 2);
      blk(B, C, tq);
      tq += bstride;
      ld(A, b + 3);
      blk(C, A, tq);
      tq += bstride;
    }
    for (; b < nfull; ++b) {  // 0..2 blocks
      ld(B, b + 1);
      blk(A, B, tq);
      tq += bstride;
#pragma unroll
      for (int g = 0; g < kG; ++g) A[g] = B[g];
    }
    if (krem) {  // last partial block: only the real taps (a zero tap times
                 // an inf/NaN input would poison the result)
      ld(B, b + 1);
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        if (!ALL && (r < rlo || r > rhi)) continue;
        const float4 t = *reinterpret_cast<const float4*>(tq - 4 * r);
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const float wv[8] = {A[g].x, A[g].y, A[g].z, A[g].w, B[g].x, B[g].y, B[g].z, B[g].w};
          float* a = &acc[r][g * kC];
#pragma unroll
          for (int c = 0; c < kC; ++c) a[c] = mac<kExact>(a[c], t.x, wv[c]);
          if (krem > 1)
#pragma unroll
            for (int c = 0; c < kC; ++c) a[c] = mac<kExact>(a[c], t.y, wv[c + 1]);
          if (krem > 2)
#pragma unroll
            for (int c = 0; c < kC; ++c) a[c] = mac<kExact>(a[c], t.z, wv[c + 2]);
        }
      }
    }
  };
  const int q_end = kR + kh - 1;
  const int s_lo = kR - 1, s_hi = kh - 1;  // steady range (empty when kh < kR)
  for (int q = 0; q < q_end; ++q) {
    if (q >= s_lo && q <= s_hi) row(std::true_type{}, q);
    else row(std::false_type{}, q);
  }

#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int gr = r0 + warp * kR + r;
    if (gr >= oh) break;
    float* yr = yi + (int64_t)gr * ow;
#pragma unroll
    for (int g = 0; g < kG; ++g)
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        const int gc = c0 + 128 * g + kC * lane + c;
        if (gc < ow) yr[gc] = acc[r][g * kC + c];
      }
  }
}

// y[b][i] = ((part[b][0][i] + part[b][1][i]) + ...) -- fixed order, deterministic
__global__ void sum_planes_kernel(const float* __restrict__ part, int nsplit, int64_t plane,
                                  int64_t batch, float* __restrict__ y) {
  const int64_t n = batch * plane;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / plane, i = e - b * plane;
    const float* p = part + b * nsplit * plane + i;
    float acc = p[0];
    for (int s = 1; s < nsplit; ++s) acc += p[s * plane];
    y[e] = acc;
  }
}

template <bool kExact, int kWarps, int kG>
int launch_big(const float* x, int64_t batch, int64_t h, int64_t w, const BigTaps& taps,
               int64_t kh, int64_t kw, float* y, cudaStream_t st) {
  constexpr int kTileRows = tile_rows(kWarps);
  constexpr int kTileCols = tile_cols(kG);
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  const int64_t gx = (ow + kTileCols - 1) / kTileCols, gy = (oh + kTileRows - 1) / kTileRows;
  if (gy > 65535) return 1;
  static uint64_t attr = 0, attr_split = 0;  // devices whose limit is set
  SC_CUDA(set_smem_limit_once(conv2d_big_kernel<kExact, kWarps, kG, false>,
                              big_smem(kMaxK, kMaxK, kWarps, kG), &attr));
  // filter-row split for grids that leave SMs idle (fast mode only: the
  // exact mode must accumulate every output in the reference's order)
  // (only for grids under one wave; slices keep >= 8 filter rows so every
  // warp still has a steady range of all-live rows)
  int nsplit = 1, jstep = (int)kh;
  const int64_t ctas = batch * gx * gy;
  if (!kExact && kh >= 24 && ctas < sm_count()) {
    const int64_t want = (3 * (int64_t)sm_count() / 2 + ctas - 1) / ctas;
    const int n = (int)std::min<int64_t>(want, std::min<int64_t>(8, kh / 8));
    if (n > 1) {
      jstep = (int)((kh + n - 1) / n);
      nsplit = (int)((kh + jstep - 1) / jstep);
    }
  }
  if (batch * nsplit > 65535) nsplit = 1, jstep = (int)kh;
  float* out = y;
  if (nsplit > 1)
    SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&out),
                            (size_t)nsplit * batch * oh * ow * sizeof(float), st));
  const dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)(batch * nsplit));
  const size_t smem = big_smem(jstep, (int)kw, kWarps, kG);
  if (nsplit > 1) {
    SC_CUDA(set_smem_limit_once(conv2d_big_kernel<kExact, kWarps, kG, true>,
                                big_smem(kMaxK, kMaxK, kWarps, kG), &attr_split));
    conv2d_big_kernel<kExact, kWarps, kG, true><<<grid, 32 * kWarps, smem, st>>>(
        x, (int)h, (int)w, taps, (int)kh, (int)kw, out, (int)oh, (int)ow, nsplit, jstep);
  } else {
    conv2d_big_kernel<kExact, kWarps, kG, false><<<grid, 32 * kWarps, smem, st>>>(
        x, (int)h, (int)w, taps, (int)kh, (int)kw, out, (int)oh, (int)ow, 1, (int)kh);
  }
  SC_LAUNCH_CHECK("conv2d_big_kernel");
  if (nsplit > 1) {
    const int64_t n = batch * oh * ow;
    sum_planes_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4 * sm_count()), 256, 0,
                        st>>>(out, nsplit, oh * ow, batch, y);
    SC_LAUNCH_CHECK("sum_planes_kernel");
    SC_CUDA(cudaFreeAsync(out, st));
  }
  return SC_OK;
}

template <bool kExact>
int dispatch_big(const float* x, int64_t batch, int64_t h, int64_t w, const BigTaps& taps,
                 int64_t kh, int64_t kw, float* y, cudaStream_t st) {
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  const int64_t ctas8 = batch * ((ow + 127) / 128) * ((oh + 63) / 64);
  static const int env_warps = [] {
    const char* e = std::getenv("SC_BIG_WARPS");
    return e ? std::atoi(e) : 0;
  }();
  const bool four = env_warps ? env_warps == 4 : ctas8 < 2 * sm_count();
  return four ? launch_big<kExact, 4, 1>(x, batch, h, w, taps, kh, kw, y, st)
              : launch_big<kExact, 8, 1>(x, batch, h, w, taps, kh, kw, y, st);
}

}  // namespace

// Returns SC_OK / an error if it ran, 1 if the shape is outside its range.
int conv2d_big(const float* x, int64_t batch, int64_t h, int64_t w, const float* f_host,
               int64_t kh, int64_t kw, bool exact, float* y, cudaStream_t st) {
  if (kh > kMaxK || kw > kMaxK || batch > 65535 || h * w >= ((int64_t)1 << 31)) return 1;
  static thread_local BigTaps taps;
  std::copy(f_host, f_host + kh * kw, taps.f);
  return exact ? dispatch_big<true>(x, batch, h, w, taps, kh, kw, y, st)
               : dispatch_big<false>(x, batch, h, w, taps, kh, kw, y, st);
}

}  // namespace sc
