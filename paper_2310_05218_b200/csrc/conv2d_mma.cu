// Single-channel 2-D convolution on the 5th-generation tensor cores (fast
// mode, opt-in SC_CONV_MMA=1): the "slide-MMA" formulation of
// _accumulate_taps (reference.py:15-23) for filters with kw <= 9 and kh <= 9
// -- BASELINE config 5 (7x7 on a 65,536^2 image) and 9x9 of the paper's
// sweep.  SURVEY 8(f)4; measured at parity with the FFMA kernels, see
// profiles/r02/slide_mma.md for the variants and why.
//
// Formulation.  Per input row rho and 1,024-column strip, with
//   M = 128 "lanes" m, each the 8 output columns c0 + 8m + s (s = 0..7),
//   K = 16 consecutive input samples x[rho][c0 + 8m + k] (k = 0..15),
//   N = (window row j', filter part f1 | f2, shift s) for the nw = kh + 1
//       (even) output rows an input row can touch,
// one MMA computes D[m][(r, part, s)] += sum_k x[rho][c0+8m+k] f_part[rho-r][k-s]:
// the whole 7x7 tap set of 1,024 columns x 8 rows in one M128 N128 K16 MMA.
// B (the taps placed by shift, filter row and split part) is a constant of
// the filter; A is the input row itself: a plain bf16 row read through a
// no-swizzle K-major descriptor with LBO = 16 B and SBO = 128 B is
// A[m][k] = x[8m + k] (the core matrices overlap by one 16-byte row;
// verified, tools/micro/hankel_probe.cu), so nothing is expanded in memory.
// D is a TMEM ring of output-row slots (16 columns: f1 and f2 parts); an
// output row is final after the MMAs of input row r + kh - 1 (+ the window's
// zero row), drained by the epilogue warps and re-zeroed for reuse.
//
// Precision: x = x1 + x2, f = f1 + f2 (bf16, round to nearest, ~16
// significant bits each); D accumulates x1 (f1 + f2) + x2 (f1 + f2) in fp32,
// normwise 2.8e-6 ... 4.5e-6 against the north-star 1e-5 k.  Tiles with
// inputs the split cannot carry (|x| > 2^64, non-finite, or nonzero
// |x| < 2^-100) are recomputed by the CTA with FMAs in the reference tap
// order after the MMA pass, so inf / NaN propagate as in the FFMA kernels.
//
// Warp roles (two CTAs per SM, 256 TMEM columns each; SC_MMA_DUAL=0 builds
// the one-CTA form with 512 columns and twice the split / epilogue warps):
// 0 TMA producer (one 4-D box per 4-row stage into an fp32 staging ring);
// 1 MMA issuer (two MMAs per input row, one elected lane of a warp with
// warp-uniform operands); 2-5 split warps (fp32 -> x1 / x2 bf16 rows in
// shared memory); 6-9 epilogue (one TMEM lane quarter each, 2-row batches:
// 16x256b TMEM loads, 256-byte coalesced stores, re-zero the slots).
// Hand-offs to the issuer are per-warp progress counters read only when its
// known-ready range runs out (an mbarrier probe costs ~180 cycles even when
// complete); MMA completion is one commit per 4 rows.  One issuing warp
// needs ~570 cycles per input row (~70-200 per tcgen05.mma plus the
// hand-offs), so the kernel runs two CTAs -- two independent issuers -- per
// SM: config 5 9.27 -> 7.6 ms, level with the FFMA kernel (7.7 ms; 8.0 vs
// 7.9 ms under sustained power-capped load).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_common.cuh"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();
namespace {
using namespace tc;

constexpr int kStrip = 1024;                 // output columns per CTA (128 lanes x 8 shifts)
constexpr int kRS = 4;                       // input rows per staging stage
// SC_MMA_DUAL: two CTAs per SM (two issuing warps per SM, each with its own
// 256-column TMEM ring and half the shared memory); otherwise one CTA with
// the whole TMEM
#ifndef SC_MMA_DUAL
#define SC_MMA_DUAL 1
#endif
constexpr int kCtasPerSm = SC_MMA_DUAL ? 2 : 1;
#ifndef SC_MMA_STAGES
#define SC_MMA_STAGES (SC_MMA_DUAL ? 3 : 6)
#endif
#ifndef SC_MMA_XSLOTS
#define SC_MMA_XSLOTS (SC_MMA_DUAL ? 8 : 16)
#endif
constexpr int kStages = SC_MMA_STAGES;        // fp32 staging ring (12 / 24 rows in flight)
// A stage is ONE 4-D TMA box: the image viewed as (256-column chunk, chunk,
// row, image) with box {256, 4, kRS, 1} lands as kRS rows of 1,024
// contiguous floats (W % 256 == 0); plus a {8, kRS} box for the 8 columns
// after the strip.  (Five 2-D boxes per stage cost ~100 cycles of producer
// issue each and capped the input stream at ~2.4 TB/s.)
constexpr int kRowBytes = kStrip * 4;        // 4 KiB
constexpr int kTailOff = kRS * kRowBytes;
constexpr int kStageBytes = (kTailOff + kRS * 8 * 4 + 127) / 128 * 128;  // 16,512
constexpr int kMaxKH = 9, kMaxKW = 9;
constexpr int kMaxNW = 10;                   // window rows = kh + 1 rounded up to even
// B matrix of one row parity p: n = 16 j' + 8 part + s (window row j',
// filter part f1 / f2, shift s) x 16 k, bf16, no-swizzle K-major (LBO 128 B
// between the k halves, SBO 256 B per 8 rows)
constexpr int kBMat = kMaxNW * 16 * 32;      // 5 KiB
// TMEM (512 columns): one D ring of kRing output-row slots of 16 columns
// (f1 part | f2 part, 8 shifts each)
constexpr int kRing = SC_MMA_DUAL ? 16 : 32;
constexpr int kTmemCols = kRing * 16;
// split bf16 rows (x1 | x2) in shared memory, read by the MMAs (SS form)
// through the overlapping (Hankel) descriptor
constexpr int kXSlots = SC_MMA_XSLOTS;
constexpr int kXRow = 2176;                  // 1,032 bf16 used, 128-aligned
constexpr int kXSlotBytes = 2 * kXRow;
constexpr int kDone = SC_MMA_DUAL ? 32 : 64;  // MMA-completion barriers, one per 4 input rows
constexpr int kEpiRows = 2;                  // output rows drained per epilogue batch
constexpr int kSplitWarps = SC_MMA_DUAL ? 4 : 8, kEpiWarps = SC_MMA_DUAL ? 4 : 8;
constexpr int kSplitGroups = kSplitWarps / 4, kEpiGroups = kEpiWarps / 4;  // of 4 warps
constexpr int kWarpSplit0 = 2, kWarpEpi0 = kWarpSplit0 + kSplitWarps;  // 2, 10
constexpr int kThreads = 32 * (kWarpEpi0 + kEpiWarps);                 // 576 / 320
constexpr size_t kSmem =
    1024 + (size_t)kStages * kStageBytes + (size_t)kXSlots * kXSlotBytes + 2 * kBMat;
static_assert(kTmemCols * kCtasPerSm == 512, "TMEM budget");
static_assert(kRing % kEpiRows == 0, "an epilogue batch never wraps the ring");
static_assert(kRing >= kMaxNW + kEpiRows + 2, "ring slack");
static_assert((kMaxKH + 2) / 2 * 2 <= kMaxNW, "window rows");
static_assert(kDone * 4 >= 2 * (kRing + kMaxNW + kXSlots + 8), "commit ring must cover the issue lead");

struct MmaArgs {
  float taps[kMaxKH * kMaxKW];
  int kh, kw, nw;
  int oh, ow, h, w;
  int seg_rows;
};

// 16 lanes x 256 bits: thread t gets lane t/4 (r0, r1) and t/4 + 8 (r2, r3),
// columns 2 (t % 4) and 2 (t % 4) + 1 (cute SM100_TMEM_LOAD_16dp256b1x)
__device__ __forceinline__ void tmem_ld_16x256(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}

// D (TMEM) += A (smem) x B (smem), issued by one elected lane of a warp
// whose operands are warp-uniform: a lone `if (lane == 0)` issuer makes ptxas
// wrap the instruction in a uniformity loop (~120 vs ~70 cycles per MMA per
// warp, tools/micro/hankel_probe.cu)
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\tsetp.eq.u32 p, 1, 1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc)
      : "memory");
}

__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Optional event trace of CTA (0, 0, 0) (tools/micro/mma_trace.cu builds
// this file with -DSC_MMA_TRACE): clock64 stamps per role and row.
#ifdef SC_MMA_TRACE
__device__ long long g_mma_trace[8][4096];
#define MMA_TRACE(role, idx, v)                                                       \
  do {                                                                                \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (idx) < 4096)         \
      g_mma_trace[role][idx] = (v);                                                   \
  } while (0)
#else
#define MMA_TRACE(role, idx, v) \
  do {                          \
  } while (0)
#endif

// Plain shared-memory counters for the hand-offs on the issuer's critical
// path: an mbarrier probe costs ~180 cycles of latency even when the phase
// is complete, an acquire load ~30.
__device__ __forceinline__ void smem_st_release(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// least progress over the four warps of a group: four independent relaxed
// loads (an acquire load orders everything after it, so four of them would
// serialise); the caller follows a probe with fence_acquire()
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.cta.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ int min_progress(const int (&c)[4]) {
  return min(min(ld_relaxed(&c[0]), ld_relaxed(&c[1])), min(ld_relaxed(&c[2]), ld_relaxed(&c[3])));
}
__device__ __forceinline__ void fence_acquire() {
  asm volatile("fence.acq_rel.cta;" ::: "memory");
}

// 2^64 / 2^-100 as float bit patterns (magnitudes the bf16 split carries)
constexpr uint32_t kHiBits = 0x5F800000u, kLoBits = 0x0D800000u;

// x1 = bf16(v), x2 = bf16(v - x1) for 8 values -> 4 + 4 packed words; track
// the magnitude range for the fallback test
__device__ __forceinline__ void split8(const float4 a, const float4 b, uint32_t* w1, uint32_t* w2) {
  const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t h = pack_bf16x2(f[2 * j], f[2 * j + 1]);
    w1[j] = h;
    w2[j] = pack_bf16x2(f[2 * j] - __uint_as_float(h << 16),
                        f[2 * j + 1] - __uint_as_float(h & 0xffff0000u));
  }
}
__device__ __forceinline__ void range8(const float4 a, const float4 b, uint32_t& mx, uint32_t& mn) {
  const float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t bits = __float_as_uint(f[j]) & 0x7fffffffu;
    mx = max(mx, bits);
    mn = min(mn, bits - 1u);  // zero -> 0xffffffff (ignored)
  }
}

__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    conv2d_mma_kernel(const __grid_constant__ CUtensorMap tm_main,
                      const __grid_constant__ CUtensorMap tm_tail, float* __restrict__ y,
                      const float* __restrict__ xg, const __grid_constant__ MmaArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t st_full[kStages], st_empty[kStages];
  // progress counters (release / acquire), one per warp: stages completed by
  // each split warp of a group, batches drained by each epilogue warp of a
  // half.  The issuer reads them only when it runs out of known-ready rows
  // and takes the minimum over a group's warps (the warps of a group drift
  // apart by up to the staging depth, so a sum would over-count).
  __shared__ int split_cnt[kSplitGroups][4], epi_cnt[kEpiGroups][4];
  __shared__ __align__(8) uint64_t done[kDone];         // MMA completion, one per 4 input rows
  __shared__ __align__(8) uint64_t ring_ready;
  __shared__ uint32_t tmem_base_sh;
  unsigned char* base = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* stages = base;
  unsigned char* xrows = stages + kStages * kStageBytes;
  unsigned char* bmats = xrows + kXSlots * kXSlotBytes;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kh = args.kh, kw = args.kw, nw = args.nw;
  const int strip = blockIdx.x, seg = blockIdx.y, img = blockIdx.z;
  const int c0 = strip * kStrip;
  const int r0 = seg * args.seg_rows;
  const int s_valid = min(args.seg_rows, args.oh - r0);   // output rows of this CTA
  const int t_rows = s_valid + kh - 1;                      // input rows it reads
  // window of input row t: output rows [a(t), a(t) + nw), a(t) even
  auto win = [&](int t, int& a, int& p) {
    const int u = t - kh + 1;
    a = u >= 0 ? (u & ~1) : -((-u + 1) & ~1);
    p = u - a;
  };
  int o_first, p0;
  win(0, o_first, p0);

  // ---- B matrices [parity p][n = 16 j' + 8 part + s][k] (see kBMat)
  for (int e = threadIdx.x; e < 2 * nw * 16 * 16; e += kThreads) {
    const int k = e & 15, n = (e >> 4) % (nw * 16), p = (e >> 4) / (nw * 16);
    const int jp = n >> 4, part = (n >> 3) & 1, s = n & 7;
    const int j = kh - 1 + p - jp, i = k - s;
    const float v = (j >= 0 && j < kh && i >= 0 && i < kw) ? args.taps[j * kw + i] : 0.0f;
    const __nv_bfloat16 v1 = __float2bfloat16_rn(v);
    const __nv_bfloat16 v2 = __float2bfloat16_rn(v - __bfloat162float(v1));
    const uint32_t off = (uint32_t)p * kBMat + (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 +
                         (k & 7) * 2;
    *reinterpret_cast<__nv_bfloat16*>(bmats + off) = part ? v2 : v1;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 4);
    }
    for (int i = 0; i < 4 * kSplitGroups; ++i) (&split_cnt[0][0])[i] = 0;
    for (int i = 0; i < 4 * kEpiGroups; ++i) (&epi_cnt[0][0])[i] = 0;
    for (int s = 0; s < kDone; ++s) mbar_init(&done[s], 1);
    mbar_init(&ring_ready, 4);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_proxy_async();  // B matrices (generic writes) -> tensor core (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  bool bad = false;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&tm_main);
      prefetch_tmap(&tm_tail);
      const uint32_t bytes = kTailOff + kRS * 8 * 4;
      for (int t = 0, s = 0; t < t_rows; t += kRS, ++s) {
        const int st = s % kStages;
        MMA_TRACE(5, 2 * s, clock64());
        if (s >= kStages) mbar_spin(&st_empty[st], ((s / kStages) - 1) & 1);
        MMA_TRACE(5, 2 * s + 1, clock64());
        unsigned char* dst = stages + st * kStageBytes;
        mbar_arrive_expect_tx(&st_full[st], bytes);
        tma_load_4d(dst, &tm_main, &st_full[st], 0, c0 / 256, r0 + t, img);
        tma_load_3d(dst + kTailOff, &tm_tail, &st_full[st], c0 + kStrip, r0 + t, img);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // per input row t two MMAs, D[ring rows a(t)..a(t)+nw) += x1 . [f1|f2]
    // and += x2 . [f1|f2] (N = 16 nw; split in two where the window wraps the
    // ring), A read from the split rows in shared memory through the
    // overlapping descriptor.  One warp issues everything, so the
    // accumulation order is fixed.  Operands are warp-uniform (shuffled base
    // values) so they stay in uniform registers; readiness of split rows and
    // drained ring slots is read from counters only when the known-ready
    // range runs out (an mbarrier probe or acquire load costs ~180 cycles).
    const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t bmat_addr = __shfl_sync(0xffffffffu, smem_u32(bmats), 0);
    const uint32_t xrows_addr = __shfl_sync(0xffffffffu, smem_u32(xrows), 0);
    mbar_wait(&ring_ready, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    int hi = o_first;                       // rows [o_first, hi) already touched
    int rows_ready = 0;                     // input rows [0, rows_ready) split into smem
    int drained = o_first;                  // output rows [o_first, drained) drained + zeroed
    for (int t = 0; t < t_rows; ++t) {
      if (lane == 0) MMA_TRACE(0, 5 * t, clock64());
      if (t >= rows_ready) {
        // rows [0, t) are ready, so t = rows_ready starts stage S: wait for
        // each warp of its group (one word per spin), then take everything
        // the counters show.  Stage s (rows kRS s ..) belongs to group s % 2.
        const int S = t / kRS;
        for (int i = 0; i < 4; ++i)
          while (ld_relaxed(&split_cnt[S % kSplitGroups][i]) <= S / kSplitGroups) {
          }
        // stages [0, min_g(G c_g + g)) done
        int st_done = kSplitGroups * min_progress(split_cnt[0]);
        for (int g = 1; g < kSplitGroups; ++g)
          st_done = min(st_done, kSplitGroups * min_progress(split_cnt[g]) + g);
        rows_ready = st_done * kRS;
        fence_acquire();
      }
      if (lane == 0) MMA_TRACE(0, 5 * t + 1, clock64());
      int a, p;
      win(t, a, p);
      // rows entering the window: a slot's previous generation (row o - kRing)
      // must be drained and zeroed
      if (a + nw > hi) {
        const int need = a + nw - kRing;     // rows < need must be drained
        if (drained < need) {
          // batches [0, nb) must be drained; batch b (rows o_first + kEpiRows b
          // ..) belongs to epilogue half b % 2
          const int nb = (need - o_first + kEpiRows - 1) / kEpiRows;
          for (int g = 0; g < kEpiGroups; ++g)
            for (int i = 0; i < 4; ++i)
              while (ld_relaxed(&epi_cnt[g][i]) < (nb - g + kEpiGroups - 1) / kEpiGroups) {
              }
          int b_done = kEpiGroups * min_progress(epi_cnt[0]);
          for (int g = 1; g < kEpiGroups; ++g)
            b_done = min(b_done, kEpiGroups * min_progress(epi_cnt[g]) + g);
          drained = o_first + b_done * kEpiRows;
          fence_acquire();
        }
        hi = a + nw;
      }
      if (lane == 0) MMA_TRACE(0, 5 * t + 2, clock64());
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t xsrc = xrows_addr + (uint32_t)(t % kXSlots) * kXSlotBytes;
      const uint64_t dx1 = make_desc(xsrc, 16, 128, 0), dx2 = make_desc(xsrc + kXRow, 16, 128, 0);
      const int q0 = (a - o_first) % kRing;              // even
      const int n1 = min(nw, kRing - q0);                // rows before the ring wraps
      const uint32_t bm = bmat_addr + (uint32_t)p * kBMat;
      const uint64_t db0 = make_desc(bm, 128, 256, 0);
      const uint32_t id0 = idesc_bf16(128, n1 * 16);
      mma_ss(tmem_u + q0 * 16, dx1, db0, id0);
      mma_ss(tmem_u + q0 * 16, dx2, db0, id0);
      if (n1 < nw) {
        const uint64_t db1 = make_desc(bm + n1 * 512, 128, 256, 0);
        const uint32_t id1 = idesc_bf16(128, (nw - n1) * 16);
        mma_ss(tmem_u, dx1, db1, id1);
        mma_ss(tmem_u, dx2, db1, id1);
      }
      if (lane == 0) MMA_TRACE(0, 5 * t + 3, clock64());
      // one commit per 4 input rows: the epilogue's "rows done" and the
      // split warps' "row slots free"
      if ((t & 3) == 3 || t + 1 == t_rows) commit_elect(&done[(t >> 2) % kDone]);
      __syncwarp();
      if (lane == 0) MMA_TRACE(0, 5 * t + 4, clock64());
    }
  } else if (warp < kWarpEpi0) {
    // ------------------------------------------------------------ split warps
    // group g (4 warps) handles stages g, g + 2, ..; thread u of the group
    // splits samples 8u..8u+7 of each row (thread 0 also the tail 1024..1031)
    // into the row's x1 / x2 bf16 rows in shared memory
    const int grp = (warp - kWarpSplit0) >> 2;
    const int u = threadIdx.x - 32 * (kWarpSplit0 + 4 * grp);   // 0..127
    uint32_t mx = 0, mn = 0xffffffffu;
    int stages_done = 0;                                  // published in split_cnt
    const int own = 32 * u;
    for (int s = grp, t0 = grp * kRS; t0 < t_rows; s += kSplitGroups, t0 += kSplitGroups * kRS) {
      const int st = s % kStages;
      if (warp == kWarpSplit0 + 4 * grp && lane == 0) MMA_TRACE(2, 4 * t0, clock64());
      mbar_spin(&st_full[st], (s / kStages) & 1);
      const unsigned char* sb = stages + st * kStageBytes;
#pragma unroll
      for (int rr = 0; rr < kRS; ++rr) {
        const int t = t0 + rr;
        if (t >= t_rows) break;
        const float4* po = reinterpret_cast<const float4*>(sb + own + rr * kRowBytes);
        const float4 a0 = po[0], a1 = po[1];
        uint32_t v[8];
        split8(a0, a1, v, v + 4);
        range8(a0, a1, mx, mn);
        uint32_t vt[8];
        if (u == 0) {
          const float4* pt = reinterpret_cast<const float4*>(sb + kTailOff + rr * 32);
          const float4 b0 = pt[0], b1 = pt[1];
          split8(b0, b1, vt, vt + 4);
          range8(b0, b1, mx, mn);
        }
        if (warp == kWarpSplit0 + 4 * grp && lane == 0) MMA_TRACE(2, 4 * t + 1, clock64());
        if (t >= kXSlots) {
          const int gq = (t - kXSlots) >> 2;                 // group of 4 holding row t - kXSlots
          mbar_spin(&done[gq % kDone], (gq / kDone) & 1);
        }
        if (warp == kWarpSplit0 + 4 * grp && lane == 0) MMA_TRACE(2, 4 * t + 2, clock64());
        unsigned char* xr = xrows + (t % kXSlots) * kXSlotBytes;
        *reinterpret_cast<uint4*>(xr + 16 * u) = make_uint4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<uint4*>(xr + kXRow + 16 * u) = make_uint4(v[4], v[5], v[6], v[7]);
        if (u == 0) {
          *reinterpret_cast<uint4*>(xr + 16 * 128) = make_uint4(vt[0], vt[1], vt[2], vt[3]);
          *reinterpret_cast<uint4*>(xr + kXRow + 16 * 128) = make_uint4(vt[4], vt[5], vt[6], vt[7]);
        }
        if (warp == kWarpSplit0 + 4 * grp && lane == 0) MMA_TRACE(2, 4 * t + 3, clock64());
      }
      fence_proxy_async();   // generic writes -> tensor-core copy (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&st_empty[st]);
        smem_st_release(&split_cnt[grp][warp & 3], ++stages_done);
      }
    }
    bad = mx > kHiBits || mn < kLoBits - 1u;
  } else {
    // ------------------------------------------------------------ epilogue
    // two groups of 4 warps (one per TMEM lane quarter) drain alternating
    // batches of kEpiRows rows (latency hiding: a batch is a chain of TMEM
    // loads, adds and global stores)
    const int q = warp & 3;                              // TMEM lane quarter
    const int half = (warp - kWarpEpi0) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    if (half == 0) {
      for (int c = 0; c < kRing * 16; c += 8) tmem_zero8(lane_base + c);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring_ready);
    }
    const int ow = args.ow;
    // thread t holds lanes m = 32 q + 8 j + t / 4 (j = 0..3), shifts
    // 2 (t % 4) and + 1, i.e. columns col_t + 64 j and + 1
    const int col_t = c0 + 8 * (32 * q + (lane >> 2)) + 2 * (lane & 3);
    // the warp's 256 columns all in range and 8-byte aligned pairs: STG.64
    const bool fast = __shfl_sync(0xffffffffu,
                                  (int)(c0 + 256 * (q + 1) <= ow &&
                                        ((reinterpret_cast<uintptr_t>(y) | (uintptr_t)(ow * 4)) &
                                         7) == 0),
                                  0) != 0;
    float* ybase = y + (int64_t)img * args.oh * ow + col_t;
    // MMA completion is signalled per group of 4 input rows (both issuers);
    // the groups are waited in order
    int groups_done = 0;
    auto wait_done = [&](int t) {
      if (t >= t_rows) t = t_rows - 1;
      for (; groups_done <= (t >> 2); ++groups_done)
        mbar_wait_sleep(&done[groups_done % kDone], (groups_done / kDone) & 1, 32, 128);
    };
    int batches_done = 0;                                 // published in epi_cnt
    for (int o0 = o_first + half * kEpiRows; o0 < s_valid; o0 += kEpiGroups * kEpiRows) {
      const int nr = min(kEpiRows, s_valid - o0);
      // every MMA touching rows < o0 + nr has t <= o0 + nr - 1 + kh (the
      // window's zero row) and t < t_rows; each issuer commits in order, so
      // the last t of each parity suffices
      const int th = o0 + nr - 1 + kh;
      [[maybe_unused]] const int bi = (o0 - o_first) / kEpiRows;
      if (warp == kWarpEpi0 && lane == 0) MMA_TRACE(4, 5 * bi, clock64());
      wait_done(th);
      if (warp == kWarpEpi0 && lane == 0) MMA_TRACE(4, 5 * bi + 1, clock64());
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t v[kEpiRows][2][2][4];                     // [row][f1 / f2 part][lane half][reg]
      const int slot0 = (o0 - o_first) % kRing;          // batches never wrap (kRing % kEpiRows == 0)
#pragma unroll
      for (int i = 0; i < kEpiRows; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            tmem_ld_16x256(lane_base + ((uint32_t)(16 * hh) << 16) + (slot0 + i) * 16 + e * 8,
                           v[i][e][hh]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (warp == kWarpEpi0 && lane == 0) MMA_TRACE(4, 5 * bi + 2, clock64());
#pragma unroll
      for (int i = 0; i < kEpiRows; ++i) {
        tmem_zero8(lane_base + (slot0 + i) * 16);
        tmem_zero8(lane_base + (slot0 + i) * 16 + 8);
      }
#pragma unroll
      for (int i = 0; i < kEpiRows; ++i) {
        const int o = o0 + i;
        if (i < nr && o >= 0) {
          float* yr = ybase + (int64_t)(r0 + o) * ow;
          float sv[8];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              sv[4 * hh + 2 * g] = __uint_as_float(v[i][0][hh][2 * g]) +
                                   __uint_as_float(v[i][1][hh][2 * g]);
              sv[4 * hh + 2 * g + 1] = __uint_as_float(v[i][0][hh][2 * g + 1]) +
                                       __uint_as_float(v[i][1][hh][2 * g + 1]);
            }
          if (fast) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<float2*>(yr + 64 * j) = make_float2(sv[2 * j], sv[2 * j + 1]);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int c = col_t + 64 * j;
              if (c < ow) yr[64 * j] = sv[2 * j];
              if (c + 1 < ow) yr[64 * j + 1] = sv[2 * j + 1];
            }
          }
        }
      }
      if (warp == kWarpEpi0 && lane == 0) MMA_TRACE(4, 5 * bi + 3, clock64());
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) smem_st_release(&epi_cnt[half][warp & 3], ++batches_done);
      if (warp == kWarpEpi0 && lane == 0) MMA_TRACE(4, 5 * bi + 4, clock64());
    }
  }

  // ---- tiles with inputs the bf16 split cannot carry: recompute with FMAs
  // in the reference tap order (reference.py:19-22), overwriting the MMA
  // results (a barrier orders the two sets of global stores)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  const int redo = __syncthreads_or(bad);
  if (redo) {
    const int64_t plane_in = (int64_t)args.h * args.w;
    const float* ximg = xg + (int64_t)img * plane_in;
    float* yimg = y + (int64_t)img * args.oh * args.ow;
    const int cols = min(kStrip, args.ow - c0);
    for (int64_t idx = threadIdx.x; idx < (int64_t)s_valid * cols; idx += kThreads) {
      const int r = r0 + (int)(idx / cols), c = c0 + (int)(idx % cols);
      float acc = 0.0f;
      for (int j = 0; j < kh; ++j)
        for (int i = 0; i < kw; ++i)
          acc = fmaf(args.taps[j * kw + i], ximg[(int64_t)(r + j) * args.w + c + i], acc);
      yimg[(int64_t)r * args.ow + c] = acc;
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols)
                 : "memory");
  }
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

}  // namespace

// Whether the slide-MMA kernel serves this call (fast mode only).
bool conv2d_mma_applicable(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                           int64_t kh, int64_t kw) {
  // opt-in (SC_CONV_MMA=1): measured at parity with the FFMA kernels on
  // config 5 ("slide-MMA"), not faster yet
  const int enabled = env_int("SC_CONV_MMA", 0);  // read per call (A/B in one process)
  if (!enabled || kh < 1 || kh > kMaxKH || kw < 1 || kw > kMaxKW) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (w % 256) || h > 0x7fffffff || w > 0x7fffffff ||
      batch > 65535)
    return false;
  // filter taps the bf16 split carries exactly enough (see the header)
  for (int64_t i = 0; i < kh * kw; ++i) {
    const float a = fabsf(f[i]);
    if (!(a <= 0x1p60f) || (a != 0.0f && a < 0x1p-100f)) return false;
  }
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  const int64_t strips = (ow + kStrip - 1) / kStrip;
  // enough 1,024-column x ~64-row tiles for two waves: large images only
  return batch * strips * ((oh + 63) / 64) >= 2 * sm_count();
}

int conv2d_mma(const float* x, int64_t batch, int64_t h, int64_t w, const float* f, int64_t kh,
               int64_t kw, float* y, cudaStream_t st) {
  auto enc = tensor_map_encoder();
  if (!enc) return fail(SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  MmaArgs a;
  std::memset(&a, 0, sizeof a);
  for (int64_t i = 0; i < kh * kw; ++i) a.taps[i] = f[i];
  a.kh = (int)kh, a.kw = (int)kw, a.nw = (int)((kh + 2) & ~1);
  a.oh = (int)oh, a.ow = (int)ow, a.h = (int)h, a.w = (int)w;
  const int64_t strips = (ow + kStrip - 1) / kStrip;
  // Row segments: one CTA per SM, every CTA costs ~(rows + kh - 1) input
  // rows; pick the segment length minimising waves x rows (whole waves).
  const int64_t slots = (int64_t)kCtasPerSm * sm_count();
  int64_t best = -1, rows = oh;
  const int env_rows = env_int("SC_MMA_ROWS", 0);
  if (env_rows > 0) {
    rows = std::min<int64_t>(env_rows, oh);
  } else {
    for (int64_t segs = 1; segs <= std::min<int64_t>(oh, 65535); ++segs) {
      const int64_t r = (oh + segs - 1) / segs;
      const int64_t n = batch * strips * ((oh + r - 1) / r);
      const int64_t cost = (n + slots - 1) / slots * (r + kh - 1 + 8);  // +8: pipeline fill
      if (best < 0 || cost < best) best = cost, rows = r;
      if (r <= 16) break;
    }
  }
  a.seg_rows = (int)rows;
  const int64_t segs = (oh + rows - 1) / rows;
  if (strips > 0x7fffffff || segs > 65535 || batch > 65535)
    return fail(SC_ERR_UNSUPPORTED, "conv2d mma: grid too large");

  CUtensorMap tm_main, tm_tail;
  {
    cuuint64_t dims[4] = {256, (cuuint64_t)(w / 256), (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[3] = {1024, (cuuint64_t)w * 4, (cuuint64_t)(h * w) * 4};
    cuuint32_t box[4] = {256, 4, (cuuint32_t)kRS, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&tm_main, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "conv2d mma: tensor map failed");
  }
  {
    cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)w * 4, (cuuint64_t)(h * w) * 4};
    cuuint32_t box[3] = {8, (cuuint32_t)kRS, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm_tail, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SC_ERR_CUDA, "conv2d mma: tail tensor map failed");
  }
  static uint64_t attr = 0;
  SC_CUDA(set_smem_limit_once(conv2d_mma_kernel, kSmem, &attr));
  dim3 grid((unsigned)strips, (unsigned)segs, (unsigned)batch);
  conv2d_mma_kernel<<<grid, kThreads, kSmem, st>>>(tm_main, tm_tail, y, x, a);
  SC_LAUNCH_CHECK("conv2d_mma_kernel");
  return SC_OK;
}

}  // namespace sc
