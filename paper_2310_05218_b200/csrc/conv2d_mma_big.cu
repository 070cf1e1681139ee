// Large single-channel filters on the 5th-generation tensor cores (fast mode):
// the slide-MMA formulation of _accumulate_taps (reference.py:15-23) for the
// paper's large-filter sweep (kernels.py:248-255, conv2d_slide_compound),
// 2 <= kw <= 57 and 2 <= kh <= 53, chosen by a cost model (roughly
// kh kw >= 13^2 on large grids).  SURVEY 8(f)3 / 8(f)4.
//
// Per input row t and 1,024-column strip:
//   M = 128 lanes m, lane m owning output columns c0 + 8 m + s (s = 0..7),
//   K = 16 kb + k: input samples x[t][c0 + 8 m + 16 kb + k] -- A is the input
//       row itself, read through a no-swizzle K-major descriptor with
//       LBO = 16 B and SBO = 128 B, so A[m][k] = x[8 m + 16 kb + k] (core
//       matrices overlap by one 16-byte row; nothing is expanded in memory,
//       same descriptor as conv2d_mma.cu, tools/micro/hankel_probe.cu),
//   N = (output row o = t - j, shift s): B[(o, s)][k] = f[t - o][16 kb + k - s].
// One MMA adds the taps of ALL filter rows that input row t feeds (a window
// of kh output rows) for 16 input samples per lane:
//   D[m][(o, s)] += sum_k x[t][c0 + 8 m + 16 kb + k] f[t - o][16 kb + k - s].
// D is a TMEM ring of 64 output-row slots of 8 columns (512 columns, one CTA
// per SM); an output row is final after the MMAs of input row o + kh - 1,
// then drained by the epilogue warps and re-zeroed.  The window of row t
// starts on a multiple of 4 rows (D offsets are multiples of 32 columns), the
// remaining 0..3 row phase is a 256-byte offset into a zero-padded B image.
//
// Precision: a scaled fp16 split.  The CTA first scans its input rows for
// the largest magnitude and scales x by a power of two to just under 2^15;
// the filter is scaled the same way on the host.  x' = x1 + x2, f' = f1 + f2
// with fp16 parts (11 significant bits each, so a pair carries ~22 bits of
// the scaled value; samples below 2^-24 of the CTA's maximum lose bits, which
// is an ABSOLUTE error of ~2^-25 of that maximum, i.e. fp32-accumulation
// class); D accumulates x1 f1 + x1 f2 + x2 f1 in fp32 (the x2 f2 term is
// ~2^-24 of a product) and the epilogue undoes the two power-of-two scales
// (exact).  Measured 0.9e-6 (11 x 11) .. 2.8e-6 (25 x 25) .. 1.2e-5 (51 x 51)
// normwise against float64; the large-window figure is the tensor core's fp32
// accumulation over kh x K blocks x 3 MMAs per element.  CTAs whose
// inputs hold inf / NaN or magnitudes outside [2^-87, 2^73] skip the tensor
// cores and compute their outputs with FMAs in the reference tap order.
//
// Narrow images (the paper's 512 x 512): P = floor((1024 - ow) / pitch) + 1
// images sit side by side in one strip, image p at samples p * pitch .. (pitch
// = w rounded up to 8), so its valid outputs only ever read its own samples;
// lanes that straddle two images produce columns >= ow that are not stored.
//
// Warps: 0-5 split (global fp32 row -> x1 / x2 fp16 rows in shared memory,
// 4 rows per batch, two batches of loads in flight), 6-13 epilogue (one TMEM
// lane quarter each, 4 output rows per batch; two groups of four on alternate
// batches, the drained slots published before the global stores), 14 MMA
// issuer (3 products x K blocks x window pieces per input row, one commit per
// batch).  Hand-offs are per batch of 4 rows (~2,000-12,000 cycles of work)
// through per-warp counters read with relaxed loads and one commit barrier.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_common.cuh"

namespace sc {
namespace {
using namespace tc;

constexpr int kStrip = 1024;             // output columns per CTA (128 lanes x 8 shifts)
constexpr int kRB = 4;                   // input rows per batch
constexpr int kXB = 3;                   // batches of split rows in shared memory
constexpr int kRing = 64;                // output-row slots in TMEM (8 columns each)
constexpr int kMaxKH = 53, kMaxKW = 57;
constexpr int kMaxKB = 4;                // K blocks of 16 samples: 16 n_kb >= kw + 7
constexpr int kXRow = 2176;              // bytes per fp16 row (1,080 samples used)
constexpr int kXSlot = 2 * kXRow;        // x1 | x2
constexpr int kND = 32;                  // MMA-completion barriers (one per batch, ring)
constexpr int kSplitWarps = 6;            // warps 0..5; epilogue warps 6..9 (TMEM quarter = warp % 4); issuer 10
constexpr int kEpiGroups = 2;             // epilogue groups of 4 warps, draining alternate batches
constexpr int kWarpEpi0 = kSplitWarps, kWarpIssue = kSplitWarps + 4 * kEpiGroups;
constexpr int kThreads = 32 * (kWarpIssue + 1);
constexpr int kPad = 3;                  // zero slots in front of the B image (row phase)
constexpr int kEStride = 12;             // epilogue staging: floats per TMEM lane (8 + 4 pad: 16-byte
                                         // aligned, conflict-free STS.128, 2-way on 4 banks for the reads)
constexpr int kEStage = 4 * 32 * kEStride * 4;  // bytes per epilogue warp (4 rows x 32 lanes)

__host__ __device__ constexpr int win_rows(int kh) { return (kh + 3 + 1) & ~1; }       // even
__host__ __device__ constexpr int bimg_slots(int kh) { return kPad + win_rows(kh) + 1; }
__host__ __device__ constexpr int bimg_bytes(int kh) { return bimg_slots(kh) * 256; }

struct BigMmaArgs {
  int kh, kw, nkb, nw;
  int oh, ow, h, w;
  int seg_rows;
  int pack, pitch, batch;    // pack > 1: that many images side by side in the strip, `pitch`
                             // samples apart (a multiple of 8, >= w); batch = images in all
  float f_scale, f_unscale;  // 2^sf applied to the taps, and 2^-sf
  long long* trace;          // SC_MMA_BIG_TRACE: clock64 stamps of one CTA, [role][index]
  int trace_cta[3];          // SC_MMA_BIG_TRACE_CTA=x,y,z (default 0,0,0)
};
#define BIG_TRACE(role, idx, v)                                                              \
  do {                                                                                       \
    if (args.trace && (int)blockIdx.x == args.trace_cta[0] &&                                \
        (int)blockIdx.y == args.trace_cta[1] && (int)blockIdx.z == args.trace_cta[2] &&      \
        (idx) < 1024)                                                                        \
      args.trace[(role) * 1024 + (idx)] = (v);                                               \
  } while (0)

struct TapsArg {
  float f[kMaxKH * kMaxKW];
};

// B images in global memory, [part f1 / f2][kb][slot][k half][s][k & 7] fp16:
// element (n = 8 slot + s, k) of the no-swizzle K-major layout (LBO 128 B
// between the k halves, SBO 256 B per 8 rows); slot = kPad + jslot holds
// filter row j = kh - 1 - jslot, zeros elsewhere.  Then the fp32 taps (for
// the FMA fallback).
__global__ void build_b_kernel(const __grid_constant__ TapsArg taps, int kh, int kw, int nkb,
                               float f_scale, __half* __restrict__ bimg,
                               float* __restrict__ taps_out) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the conv kernel's prologue may start
  const int slots = bimg_slots(kh);
  const int per = slots * 128;  // elements per (part, kb) image
  const int total = 2 * nkb * per;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int img = e / per, r = e - img * per;
    const int part = img / nkb, kb = img - part * nkb;
    const int slot = r >> 7, kh2 = (r >> 6) & 1, s = (r >> 3) & 7, k7 = r & 7;
    const int k = 8 * kh2 + k7;
    const int jslot = slot - kPad, j = kh - 1 - jslot, i = 16 * kb + k - s;
    float v = 0.0f;
    if (jslot >= 0 && j >= 0 && i >= 0 && i < kw) v = taps.f[j * kw + i] * f_scale;
    const __half v1 = __float2half_rn(v);
    bimg[e] = part ? __float2half_rn(v - __half2float(v1)) : v1;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kh * kw; e += gridDim.x * blockDim.x)
    taps_out[e] = taps.f[e];
}

// kind::f16 instruction descriptor with fp16 A / B (format 0), D f32,
// both K-major (tc_common.cuh idesc_bf16 sets format 1 = bf16)
__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\tsetp.eq.u32 p, 1, 1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// Progress counters are read with independent relaxed loads (an acquire load
// orders everything after it, so a row of them serialises: ~100 cycles each,
// 700 per batch with six split warps) and one acquire fence once the wait is
// over.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
template <int N>
__device__ __forceinline__ int min_progress(const int (&c)[N]) {
  int m = ld_relaxed(&c[0]);
#pragma unroll
  for (int i = 1; i < N; ++i) m = min(m, ld_relaxed(&c[i]));
  return m;
}
__device__ __forceinline__ void fence_acquire() {
  asm volatile("fence.acq_rel.cta;" ::: "memory");
}

// biased exponents of the largest input magnitude a CTA scales (2^-87 .. 2^73)
constexpr int kExpLo = 40, kExpHi = 200;

template <int NKB>
__global__ void __launch_bounds__(kThreads, 1)
    conv2d_mma_big_kernel(const float* __restrict__ xg, float* __restrict__ y,
                          const uint4* __restrict__ bimg, const float* __restrict__ taps,
                          const __grid_constant__ BigMmaArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ int split_cnt[kSplitWarps], epi_cnt[kEpiGroups][4];       // batches done per warp (release / acquire)
  __shared__ __align__(8) uint64_t done[kND];    // MMA completion, one per batch of input rows
  __shared__ __align__(8) uint64_t ring_ready;
  __shared__ uint32_t tmem_base_sh;
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* xrows = base;                                   // kXB * kRB slots
  unsigned char* estage = xrows + kXB * kRB * kXSlot;            // 4 * kEpiGroups epilogue warps
  unsigned char* bmats = estage + 4 * kEpiGroups * kEStage;                   // 2 * nkb images

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) BIG_TRACE(7, 3, clock64());
  // with a trace buffer: every CTA's entry / exit %globaltimer after the 8 role rows
  const int cta_lin = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (args.trace && threadIdx.x == 0 && cta_lin < 2048) {
    long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    args.trace[8 * 1024 + 4 * cta_lin] = gt;
  }
  constexpr int nkb = NKB;  // K blocks: compile-time so a piece's MMAs issue as one unrolled block
  const int kh = args.kh, kw = args.kw, nw = args.nw;
  const int c0 = blockIdx.x * kStrip;
  const int r0 = blockIdx.y * args.seg_rows;
  const int pack = args.pack, pitch = args.pitch;
  const int img = blockIdx.z * pack;                    // first image of this CTA
  const int nimg = min(pack, args.batch - img);         // images packed in the strip
  const int s_valid = min(args.seg_rows, args.oh - r0);  // output rows of this CTA
  const int t_rows = s_valid + kh - 1;                    // input rows it reads
  const int n_batches = (t_rows + kRB - 1) / kRB;
  const int o_start = -(((kh - 1) + 3) & ~3);            // first ring row, multiple of 4
  const int bimg_b = bimg_bytes(kh);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSplitWarps; ++i) split_cnt[i] = 0;
    for (int i = 0; i < 4 * kEpiGroups; ++i) (&epi_cnt[0][0])[i] = 0;
    for (int s = 0; s < kND; ++s) mbar_init(&done[s], 1);
    mbar_init(&ring_ready, 4);
    fence_mbar_init();
  }
  if (warp == kWarpIssue) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  if (threadIdx.x == 0) BIG_TRACE(7, 0, clock64());

  // ---- range scan of the CTA's input rows (all threads): largest magnitude
  // -> power-of-two scale; inf / NaN or an extreme range -> FMA fallback
  __shared__ uint32_t xmax_sh;
  if (threadIdx.x == 0) xmax_sh = 0;
  __syncthreads();
  {
    const int w = args.w;
    // one image: the samples the K blocks reach from this strip; packed: whole rows
    const int span = pack > 1 ? w : min(kStrip + 16 * nkb + 8, w - c0);
    uint32_t mx = 0;
    auto amax4 = [](uint32_t m, const float4 v) {
      return max(max(m, __float_as_uint(v.x) & 0x7fffffffu),
                 max(__float_as_uint(v.y) & 0x7fffffffu,
                     max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu)));
    };
    for (int p = 0; p < nimg; ++p) {
      const float* xrow0 = xg + (int64_t)(img + p) * args.h * args.w + (int64_t)r0 * args.w;
      if ((w & 3) == 0) {
        // 16 rows per step: 16 independent 16-byte loads in flight per thread
        const int n4 = span >> 2;  // c0 and w are multiples of 4
        const int w4 = w >> 2;
        const float4* rp0 = reinterpret_cast<const float4*>(xrow0 + c0);
        for (int e = threadIdx.x; e < n4; e += kThreads) {
          for (int t = 0; t < t_rows; t += 16) {
            float4 v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = rp0[(int64_t)min(t + j, t_rows - 1) * w4 + e];
#pragma unroll
            for (int j = 0; j < 16; ++j) mx = amax4(mx, v[j]);
          }
        }
      } else {
        for (int t = 0; t < t_rows; ++t) {
          const float* rp = xrow0 + (int64_t)t * w + c0;
          for (int e = threadIdx.x; e < span; e += kThreads)
            mx = max(mx, __float_as_uint(rp[e]) & 0x7fffffffu);
        }
      }
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) atomicMax(&xmax_sh, mx);
  }
  // ---- B images: global -> shared (16-byte copies).  The kernel is launched
  // programmatically dependent on build_b_kernel, so everything above (the
  // range scan reads only x, complete before build_b started) overlaps it;
  // its output is read from here on.
  if (args.trace && threadIdx.x == 0 && cta_lin < 2048) {
    long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    args.trace[8 * 1024 + 4 * cta_lin + 2] = gt;  // range scan done
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    const int n16 = 2 * nkb * bimg_b / 16;
    uint4* dst = reinterpret_cast<uint4*>(bmats);
    for (int e = threadIdx.x; e < n16; e += kThreads) dst[e] = bimg[e];
  }
  fence_proxy_async();  // B images (generic writes) -> tensor core (async proxy)
  __syncthreads();
  if (threadIdx.x == 0) BIG_TRACE(7, 1, clock64());
  const int xexp = (int)(xmax_sh >> 23);  // biased exponent of the largest magnitude
  // all-zero input: any scale works; otherwise 2^(14 - exponent) puts the maximum in [2^14, 2^15)
  const bool bad = xmax_sh != 0 && (xexp < kExpLo || xexp > kExpHi);
  const float x_scale = xmax_sh == 0 ? 1.0f : __uint_as_float((uint32_t)(268 - xexp) << 23);
  const float x_unscale = xmax_sh == 0 ? 1.0f : __uint_as_float((uint32_t)(xexp - 14) << 23);

  if (bad) {
    // no tensor-core pass for this CTA (see the fallback below)
  } else if (warp < kSplitWarps) {
    // ------------------------------------------------------------ split warps
    // A batch is kRB rows x 136 chunks of 8 samples (column c0 + 8 cc -> byte
    // 16 cc of the row's x1 / x2 slots; the K blocks reach 8*127 + 16 nkb + 15
    // <= 1,087).  Thread u of the 192 owns chunks u + 192 j (j = 0, 1, and
    // j = 2 for u < 160) of every batch.  Two batches of loads are kept in flight in
    // registers: with one, the load latency was exposed once per batch
    // (~750 cycles per input row with no MMAs at all).
    constexpr int kChunks = 136, kOwn = 3, kSplitThreads = 32 * kSplitWarps;
    const int u = threadIdx.x;  // 0..191
    const int64_t plane = (int64_t)args.h * args.w;
    const float* xrow0 = xg + (int64_t)img * plane + (int64_t)r0 * args.w;
    const int w = args.w;
    const bool vec = (w & 3) == 0;
    // chunk -> (row of the batch, chunk of the row); the chunk's samples are
    // columns xcol .. xcol + 7 of image img + ximg (packed: pitch is a
    // multiple of 8, so a chunk never straddles two images; ximg < 0: zeros)
    int crow[kOwn], ccol[kOwn], xcol[kOwn], ximg[kOwn];
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
      const int c = u + kSplitThreads * j;
      crow[j] = c / kChunks;
      ccol[j] = c - crow[j] * kChunks;
      if (pack > 1) {
        const int pi = 8 * ccol[j] / pitch;
        ximg[j] = pi < nimg ? pi : -1;
        xcol[j] = 8 * ccol[j] - pi * pitch;
      } else {
        ximg[j] = 0;
        xcol[j] = c0 + 8 * ccol[j];
      }
    }
    const bool own4 = u < kRB * kChunks - (kOwn - 1) * kSplitThreads;  // the last owned chunk exists
    auto load8 = [&](const float* rowp, int col, float (&f)[8]) {
      if (vec && col + 8 <= w) {
        const float4 a = *reinterpret_cast<const float4*>(rowp + col);
        const float4 b = *reinterpret_cast<const float4*>(rowp + col + 4);
        f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w;
        f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = col + j < w ? rowp[col + j] : 0.0f;
      }
    };
    auto split_store = [&](const float (&f)[8], unsigned char* dst) {
      uint32_t w1[4], w2[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a = f[2 * j] * x_scale, b = f[2 * j + 1] * x_scale;
        const uint32_t h = pack_f16x2(a, b);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        w1[j] = h;
        w2[j] = pack_f16x2(a - hf.x, b - hf.y);
      }
      *reinterpret_cast<uint4*>(dst) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
      *reinterpret_cast<uint4*>(dst + kXRow) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
    };
    auto fetch = [&](int b, float (&buf)[kOwn][8]) {
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        if (j == kOwn - 1 && !own4) break;
        const int t = min(b * kRB + crow[j], t_rows - 1);
        if (ximg[j] >= 0) {
          load8(xrow0 + ximg[j] * plane + (int64_t)t * w, xcol[j], buf[j]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) buf[j][i] = 0.0f;
        }
      }
    };
    auto emit = [&](int b, const float (&buf)[kOwn][8]) {
      if (b >= kXB) {
        const int pb = b - kXB;  // the batch that used this slot: its MMAs must be complete
        // back off between probes (the waiters share sub-partitions with the
        // MMA-issuing warp); polling test_wait + nanosleep instead measured
        // 3-5 % slower and did not remove the occasional straggler CTA
        mbar_wait_sleep(&done[pb % kND], (pb / kND) & 1, 32, 256);
      }
      if (threadIdx.x == 0) BIG_TRACE(0, b, clock64());
      unsigned char* slot0 = xrows + (b % kXB) * kRB * kXSlot;
#pragma unroll
      for (int j = 0; j < kOwn; ++j) {
        if (j == kOwn - 1 && !own4) break;
        split_store(buf[j], slot0 + crow[j] * kXSlot + 16 * ccol[j]);
      }
    };
    auto publish = [&](int b) {
      fence_proxy_async();  // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) st_release(&split_cnt[warp], b + 1);
      if (threadIdx.x == 0) BIG_TRACE(1, b, clock64());
    };
    float buf0[kOwn][8], buf1[kOwn][8];
    fetch(0, buf0);
    if (n_batches > 1) fetch(1, buf1);
    for (int b = 0; b < n_batches; b += 2) {
      emit(b, buf0);
      if (b + 2 < n_batches) fetch(b + 2, buf0);
      publish(b);
      if (b + 1 < n_batches) {
        emit(b + 1, buf1);
        if (b + 3 < n_batches) fetch(b + 3, buf1);
        publish(b + 1);
      }
    }
  } else if (warp < kWarpIssue) {
    // ------------------------------------------------------------ epilogue
    // two groups of 4 warps (one per TMEM lane quarter) drain alternating
    // batches of 4 output rows: a batch is a dependent chain (TMEM loads,
    // staging, ~32 global stores, re-zeroing) of ~2,400-4,500 cycles, more
    // than the issuer needs per batch for windows below ~25 rows
    const int q = warp & 3;  // TMEM lane quarter
    const int grp = (warp - kWarpEpi0) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    if (grp == 0) {
      for (int c = 0; c < 512; c += 8) tmem_zero8(lane_base + c);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring_ready);
    }
    const int ow = args.ow;
    const float f_unscale = args.f_unscale;
    // a TMEM lane holds 8 consecutive output columns; the warp's 256 columns
    // go through a padded shared-memory slab so that every global store is a
    // coalesced 128-byte row segment whatever the alignment of the output row
    // (per-lane 32-byte stores cost ~1,000 cycles per output row)
    float* est = reinterpret_cast<float*>(estage + (4 * grp + q) * kEStage);
    const int colw = c0 + 256 * q;  // first column (one image) / strip position (packed) of this warp
    const int64_t oplane = (int64_t)args.oh * ow;
    float* ybase = y + (int64_t)img * oplane;
    // element it * 32 + lane of the warp's 256: its offset inside an output
    // row (packed: image plane + column) and whether it is stored -- fixed
    // for the CTA, so the divisions happen once, not per element and row
    int eoff[8];  // 32-bit: the host packs only while pack * oh * ow < 2^31
    uint32_t emask = 0;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int pos = colw + it * 32 + lane;
      if (pack > 1) {
        const int pi = pos / pitch, c = pos - pi * pitch;
        eoff[it] = pi * (int)oplane + c;
        emask |= (uint32_t)(pi < nimg && c < ow) << it;
      } else {
        eoff[it] = pos;
        emask |= (uint32_t)(pos < ow) << it;
      }
    }
    const bool any_col = __any_sync(0xffffffffu, emask != 0);
    const bool full_cols = pack == 1 && colw + 256 <= ow;  // no per-element bounds
    // two multiplications undo the scales (their product may leave the float range)
    const int n_epi = (s_valid - o_start + 3) / 4;
    int batches_done = 0;  // MMA batches known complete (waited in order)
    int drained = 0;       // batches this warp has drained (published in epi_cnt)
    for (int e = grp; e < n_epi; e += kEpiGroups) {
      const int o0 = o_start + 4 * e;
      const int t_final = min(o0 + 3 + kh - 1, t_rows - 1);
      for (; batches_done <= t_final / kRB; ++batches_done)
        mbar_wait_sleep(&done[batches_done % kND], (batches_done / kND) & 1, 32, 256);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (warp == kWarpEpi0 && lane == 0) BIG_TRACE(5, e, clock64());
      const int slot0 = (o0 - o_start) & (kRing - 1);
      uint32_t v[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i) tmem_ld8(lane_base + (slot0 + i) * 8, v[i]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 4; ++i) tmem_zero8(lane_base + (slot0 + i) * 8);
      // the slots are free as soon as they are re-zeroed: publish before the
      // staging and the global stores, so the issuer never waits on store
      // latency (some CTAs' stores ran slow enough to eat the ring's slack
      // and delay their second half by 12-20 us)
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) st_release(&epi_cnt[grp][q], ++drained);
      if (o0 + 3 >= 0 && any_col) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float o8[8];
#pragma unroll
          for (int s8 = 0; s8 < 8; ++s8)
            o8[s8] = __uint_as_float(v[i][s8]) * x_unscale * f_unscale;
          float4* dst = reinterpret_cast<float4*>(est + (i * 32 + lane) * kEStride);
          dst[0] = make_float4(o8[0], o8[1], o8[2], o8[3]);
          dst[1] = make_float4(o8[4], o8[5], o8[6], o8[7]);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int o = o0 + i;
          if (o >= 0 && o < s_valid) {
            float* yr = ybase + (int64_t)(r0 + o) * ow;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int ee = it * 32 + lane;
              const float val = est[(i * 32 + (ee >> 3)) * kEStride + (ee & 7)];
              if (pack > 1) {
                if ((emask >> it) & 1) yr[eoff[it]] = val;
              } else if (full_cols || colw + ee < ow) {
                yr[colw + ee] = val;  // immediate offsets from one base per row
              }
            }
          }
        }
        __syncwarp();
      }
      if (warp == kWarpEpi0 && lane == 0) BIG_TRACE(6, e, clock64());
    }
  } else {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t bmat_addr = __shfl_sync(0xffffffffu, smem_u32(bmats), 0);
    const uint32_t xrows_addr = __shfl_sync(0xffffffffu, smem_u32(xrows), 0);
    mbar_wait(&ring_ready, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int epi_known = 0;  // epilogue batches known drained
    for (int b = 0; b < n_batches; ++b) {
      if (lane == 0) BIG_TRACE(2, b, clock64());
      while (min_progress(split_cnt) <= b) {
      }
      fence_acquire();
      if (lane == 0) BIG_TRACE(3, b, clock64());
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int rr = 0; rr < kRB; ++rr) {
        const int t = b * kRB + rr;
        if (t >= t_rows) break;
        const int uo = t - kh + 1;   // first output row this input row feeds
        const int a = uo & ~3;       // window start (floor to a multiple of 4)
        const int p = uo - a;        // row phase 0..3
        // ring slots re-entering the window must be drained and zeroed: rows
        // below a + nw - kRing, i.e. epilogue batches [0, need)
        const int need = (a + nw - kRing - o_start + 3) >> 2;
        if (need > epi_known) {
          // group g has drained batches g, g + 2, ..: all batches below
          // min_g(2 c_g + g) are done
          int got;
          for (;;) {
            got = kEpiGroups * min_progress(epi_cnt[0]);
#pragma unroll
            for (int g = 1; g < kEpiGroups; ++g)
              got = min(got, kEpiGroups * min_progress(epi_cnt[g]) + g);
            if (got >= need) break;
          }
          fence_acquire();
          epi_known = got;  // everything the counters show, not just what was needed
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const uint32_t xsrc = xrows_addr + (uint32_t)((b % kXB) * kRB + rr) * kXSlot;
        const int q0 = (a - o_start) & (kRing - 1);  // multiple of 4
        // pieces of the window: split at the ring end and at 32 slots (N <= 256)
        for (int bs = 0; bs < nw;) {
          const int qs = (q0 + bs) & (kRing - 1);
          const int ns = min(min(nw - bs, kRing - qs), 32);
          const uint32_t idesc = idesc_f16(128, ns * 8);
          const uint32_t d = tmem_u + qs * 8;
          const uint32_t boff = (uint32_t)(kPad - p + bs) * 256;
          // descriptors differ only in their 14-bit address fields: one base
          // each, then plain adds (a row's samples stay inside one 16 KiB
          // window of the field, as do the B images)
          const uint64_t da0 = make_desc(xsrc, 16, 128, 0);
          const uint64_t db0 = make_desc(bmat_addr + boff, 128, 256, 0);
          const uint32_t bstep = (uint32_t)bimg_b >> 4;
#pragma unroll
          for (int prod = 0; prod < 3; ++prod) {
            const int xp = prod == 2, fp = prod == 1;  // x1 f1, x1 f2, x2 f1
#pragma unroll
            for (int kb = 0; kb < nkb; ++kb)
              mma_ss(d, da0 + (uint32_t)(xp * (kXRow >> 4) + 2 * kb),
                     db0 + (uint64_t)((fp * nkb + kb) * bstep), idesc);
          }
          bs += ns;
        }
      }
      umma_commit_elect(&done[b % kND]);
      __syncwarp();
      if (lane == 0) BIG_TRACE(4, b, clock64());
      if (args.trace && lane == 0 && cta_lin < 2048 && (b == n_batches - 1 || b == n_batches / 2)) {
        long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        args.trace[8 * 1024 + 4 * cta_lin + 3] = b == n_batches - 1 ? gt : -gt;  // mid-way stamp negated
        if (b != n_batches - 1) args.trace[8 * 1024 + 4 * 2048 + cta_lin] = gt;
      }
    }
  }

  // ---- CTAs whose inputs the scaled split cannot carry: compute with FMAs in
  // the reference tap order (reference.py:19-22), overwriting the MMA results
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) BIG_TRACE(7, 2, clock64());
  if (args.trace && threadIdx.x == 0 && cta_lin < 2048) {
    long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    args.trace[8 * 1024 + 4 * cta_lin + 1] = gt;
  }
  if (bad) {
    const int64_t plane_in = (int64_t)args.h * args.w;
    const int cols = min(kStrip, args.ow - c0);
    for (int p = 0; p < nimg; ++p) {
      const float* ximg = xg + (int64_t)(img + p) * plane_in;
      float* yimg = y + (int64_t)(img + p) * args.oh * args.ow;
      for (int64_t idx = threadIdx.x; idx < (int64_t)s_valid * cols; idx += kThreads) {
        const int r = r0 + (int)(idx / cols), c = c0 + (int)(idx % cols);
        float acc = 0.0f;
        for (int j = 0; j < kh; ++j)
          for (int i = 0; i < kw; ++i)
            acc = fmaf(taps[j * kw + i], ximg[(int64_t)(r + j) * args.w + c + i], acc);
        yimg[(int64_t)r * args.ow + c] = acc;
      }
    }
  }
  if (warp == kWarpIssue) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512)
                 : "memory");
  }
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

size_t smem_bytes(int kh, int nkb) {
  return 1024 + (size_t)kXB * kRB * kXSlot + 4 * kEpiGroups * (size_t)kEStage +
         (size_t)2 * nkb * bimg_bytes(kh);
}


// Row segments: one CTA per SM, every CTA costs ~(rows + kh - 1) input rows
// plus the pipeline fill; pick the segment length minimising waves x rows.
// Returns the output rows per segment and the modelled rows per SM.
// Images packed side by side in one strip (1 = none) and their pitch in samples.
int pack_of(int64_t w, int64_t ow, int* pitch) {
  const int64_t pt = (w + 7) / 8 * 8;
  *pitch = (int)pt;
  if (ow > kStrip - pt) return 1;  // a second image's valid outputs would not fit the lanes
  return (int)std::min<int64_t>((kStrip - ow) / pt + 1, 64);
}
// ... and only while an image group's outputs stay 32-bit addressable
int pack_for(int64_t w, int64_t oh, int64_t ow, int* pitch) {
  int p = pack_of(w, ow, pitch);
  while (p > 1 && (int64_t)p * oh * ow >= ((int64_t)1 << 31)) --p;
  return p;
}

int64_t plan_rows(int64_t batch, int64_t oh, int64_t ow, int64_t kh, int64_t* cost_rows) {
  const int64_t strips = (ow + kStrip - 1) / kStrip;
  const int64_t slots = sm_count();
  int64_t best = -1, rows = oh;
  for (int64_t segs = 1; segs <= std::min<int64_t>(oh, 65535); ++segs) {
    const int64_t r = (oh + segs - 1) / segs;
    const int64_t n = batch * strips * ((oh + r - 1) / r);
    const int64_t cost = (n + slots - 1) / slots * (r + kh - 1 + 12);
    if (best < 0 || cost < best) best = cost, rows = r;
    if (r <= 8 || n > 64 * slots) break;  // shorter segments only add halo rows
  }
  if (cost_rows) *cost_rows = best;
  return rows;
}

}  // namespace

// Whether the large-filter slide-MMA kernel serves this call (fast mode
// only).  SC_CONV_MMA_BIG: 0 off, 1 (default) when the modelled tensor-core
// time beats the FFMA kernels', 2 whenever the shape fits.
bool conv2d_mma_big_applicable(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                               int64_t kh, int64_t kw) {
  const int mode = env_int("SC_CONV_MMA_BIG", 1);  // read per call (A/B in one process)
  if (!mode || kh < 2 || kh > kMaxKH || kw < 2 || kw > kMaxKW) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || h > 0x7fffffff || w > 0x7fffffff || batch > 65535 ||
      batch < 1)
    return false;
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  if (mode == 1) {
    if (kh * kw < 150) return false;
    // cycles per SM: ~115 per MMA (3 products x K blocks x window pieces per
    // input row; issue-bound for short windows, tensor-bound from N ~ 200),
    // ~750 per row at least, ~30,000 for the range scan and fill; the FFMA
    // kernels sustain ~55 % of the FP32 pipe on full grids (measured,
    // tools/mma_big_check.py: the model picks the faster side on the sweep)
    int64_t cost_rows = 0;
    int pitch = 0;
    const int pack = pack_for(w, oh, ow, &pitch);
    plan_rows((batch + pack - 1) / pack, oh, ow, kh, &cost_rows);
    const int nkb = (int)((kw + 7 + 15) / 16), nw = win_rows((int)kh);
    const double n_mma = 3.0 * nkb * ((nw + 31) / 32 + 0.3);
    const double t_mma = (double)cost_rows * std::max(750.0, 115.0 * n_mma) + 30000.0;
    const double t_ffma = (double)batch * oh * ow * kh * kw / (sm_count() * 128.0 * 0.55);
    if (t_mma > 0.75 * t_ffma) return false;
  }
  // a finite filter whose largest tap the power-of-two scale can carry
  float fmax = 0.0f;
  for (int64_t i = 0; i < kh * kw; ++i) {
    const float a = fabsf(f[i]);
    if (!(a <= 0x1p60f)) return false;
    fmax = std::max(fmax, a);
  }
  return fmax >= 0x1p-60f;
}

int conv2d_mma_big(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, int64_t kh,
                   int64_t kw, float* y, cudaStream_t st) {
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  BigMmaArgs a;
  a.kh = (int)kh, a.kw = (int)kw, a.nkb = (int)((kw + 7 + 15) / 16), a.nw = win_rows((int)kh);
  a.oh = (int)oh, a.ow = (int)ow, a.h = (int)h, a.w = (int)w;
  a.trace = nullptr;
  if (const char* e = getenv("SC_MMA_BIG_TRACE")) a.trace = reinterpret_cast<long long*>(strtoull(e, nullptr, 0));
  a.trace_cta[0] = a.trace_cta[1] = a.trace_cta[2] = 0;
  if (const char* e = getenv("SC_MMA_BIG_TRACE_CTA"))
    sscanf(e, "%d,%d,%d", &a.trace_cta[0], &a.trace_cta[1], &a.trace_cta[2]);
  const int64_t strips = (ow + kStrip - 1) / kStrip;
  a.pack = env_int("SC_MMA_BIG_PACK", 1) ? pack_for(w, oh, ow, &a.pitch) : 1;
  if (a.pack == 1) a.pitch = 0;
  a.batch = (int)batch;
  const int64_t groups = (batch + a.pack - 1) / a.pack;
  const int env_rows = env_int("SC_MMA_BIG_ROWS", 0);
  const int64_t rows =
      env_rows > 0 ? std::min<int64_t>(env_rows, oh) : plan_rows(groups, oh, ow, kh, nullptr);
  a.seg_rows = (int)rows;
  const int64_t segs = (oh + rows - 1) / rows;
  if (strips > 0x7fffffff || segs > 65535 || batch > 65535)
    return fail(SC_ERR_UNSUPPORTED, "conv2d mma: grid too large");

  float fmax = 0.0f;
  for (int64_t i = 0; i < kh * kw; ++i) fmax = std::max(fmax, fabsf(f[i]));
  int fe = 0;
  frexpf(fmax, &fe);                       // fmax = m 2^fe, m in [0.5, 1)
  a.f_scale = ldexpf(1.0f, 14 - fe);       // largest tap in [2^13, 2^14)
  a.f_unscale = ldexpf(1.0f, fe - 14);
  static thread_local TapsArg taps;
  std::copy(f, f + kh * kw, taps.f);
  const size_t bbytes = (size_t)2 * a.nkb * bimg_bytes(a.kh);
  unsigned char* scratch = nullptr;
  SC_CUDA(scratch_alloc(reinterpret_cast<void**>(&scratch), bbytes + (size_t)kh * kw * 4, st));
  // stream-ordered free on every exit path (an early error return must not leak it)
  struct ScratchFree {
    void* p;
    cudaStream_t st;
    ~ScratchFree() { cudaFreeAsync(p, st); }
  } scratch_free{scratch, st};
  __half* bimg = reinterpret_cast<__half*>(scratch);
  float* taps_dev = reinterpret_cast<float*>(scratch + bbytes);
  build_b_kernel<<<32, 256, 0, st>>>(taps, a.kh, a.kw, a.nkb, a.f_scale, bimg, taps_dev);
  SC_LAUNCH_CHECK("build_b_kernel");
  const size_t smem = smem_bytes(a.kh, a.nkb);
  dim3 grid((unsigned)strips, (unsigned)segs, (unsigned)groups);
  const uint4* bimg4 = reinterpret_cast<const uint4*>(bimg);
  auto launch = [&](auto kernel, uint64_t* done_attr) -> cudaError_t {
    cudaError_t e = set_smem_limit_once(kernel, smem_bytes(kMaxKH, kMaxKB), done_attr);
    if (e == cudaSuccess)
      e = launch_pdl(kernel, grid, dim3(kThreads), smem, st, x, y, bimg4, (const float*)taps_dev, a);
    return e;
  };
  static uint64_t attrs[kMaxKB] = {};
  switch (a.nkb) {
    case 1: SC_CUDA(launch(conv2d_mma_big_kernel<1>, &attrs[0])); break;
    case 2: SC_CUDA(launch(conv2d_mma_big_kernel<2>, &attrs[1])); break;
    case 3: SC_CUDA(launch(conv2d_mma_big_kernel<3>, &attrs[2])); break;
    default: SC_CUDA(launch(conv2d_mma_big_kernel<4>, &attrs[3])); break;
  }
  SC_LAUNCH_CHECK("conv2d_mma_big_kernel");
  return SC_OK;
}

}  // namespace sc
