/*
 * slideconv_b200 -- C ABI of the B200-native (sm_100a) Sliding Window Sum
 * convolution / pooling primitives (arXiv 2310.05218).
 *
 * The reference package (`slideconv`, pure Python + numpy) has no FFI: its
 * boundary is the Python function signatures exported by
 * pkg/src/slideconv/__init__.py:4-49.  Each entry point below replaces the
 * arithmetic behind one of those functions (cited per function); the Python
 * package `paper_2310_05218_b200` binds them with ctypes and keeps the
 * reference's signatures, validation order and exception classes.
 *
 * Conventions
 *   - all sizes are int64_t element counts; tensors are dense, C-contiguous;
 *   - `*_f32/_f64` device entry points take DEVICE pointers (x, y, weights of
 *     the NCHW/im2col paths) and an explicit cudaStream_t passed as void*;
 *     they enqueue work and return without synchronising; they never allocate;
 *   - 2-D single-channel / 1-D filters (`f`, `w`) are HOST pointers: their taps
 *     are copied into the kernel launch parameters (constant bank), so the
 *     filter may be freed as soon as the call returns;
 *   - `*_host` entry points take HOST pointers (pinned or pageable) for x and y
 *     and run a chunked H2D / compute / D2H pipeline on `device`; they return
 *     after the result is in y;
 *   - return 0 (SC_OK) or a negative sc_status; sc_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - mode: SC_MODE_FAST (default; fused multiply-add, O(1)-per-output
 *     window sums for wide windows) or SC_MODE_EXACT (reference operation
 *     order: multiply then add in ascending (j, i) tap order, doubling order
 *     for window sums -> bit-identical to the reference's float32 results).
 *     Max pooling is always bit-exact.
 */
#ifndef SLIDECONV_B200_H
#define SLIDECONV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SC_OK = 0,
  SC_ERR_SHAPE = -1,        /* reference ShapeError (tensor.py:14-15) */
  SC_ERR_ARG = -2,          /* bad enum / null pointer / misaligned pointer */
  SC_ERR_CUDA = -3,         /* CUDA runtime/driver failure */
  SC_ERR_UNSUPPORTED = -4,  /* shape outside what this build serves */
  SC_ERR_CUBLAS = -5        /* cuBLAS missing or failed (contrast path only) */
} sc_status;

typedef enum { SC_POOL_SUM = 0, SC_POOL_AVG = 1, SC_POOL_MAX = 2 } sc_pool_op;
typedef enum { SC_MODE_FAST = 0, SC_MODE_EXACT = 1 } sc_mode;

/* ABI version (major*10000 + minor*100 + patch). */
int sc_version(void);
/* Message for the last non-zero status returned on this thread ("" if none). */
const char* sc_last_error(void);

/* ---- 1-D pooling ---------------------------------------------------------
 * Replaces sliding_window_sum / sliding_window_max (pooling.py:28-78), one
 * call per signal there; here `batch` independent signals of `length`
 * samples each.  x: (batch, length) -> y: (batch, length - k + 1).
 * AVG = float32(sum) / float32(k) (IEEE division), new in this build.
 * Returns SC_ERR_SHAPE unless 1 <= k <= length (pooling.py:32-33). */
int sc_pool1d_f32(int op, const float* x, int64_t batch, int64_t length, int64_t k,
                  int mode, float* y, void* stream);
/* Fused pair (new): y_a = sliding_window_sum (op_a = SC_POOL_SUM) or its
 * average (SC_POOL_AVG) and y_max = sliding_window_max (pooling.py:28-53 and
 * :56-78) of the SAME signals in one pass over x -- one read of the input for
 * both outputs on the TMA kernel's windows (k = 2..33, 64; 16-byte aligned
 * signals of length % 32 == 0); other shapes run the two single-op kernels
 * back to back.  Each output is bit-identical to sc_pool1d_f32's for that op
 * and mode.  y_a and y_max: (batch, length - k + 1) each, not aliased. */
int sc_pool1d_pair_f32(int op_a, const float* x, int64_t batch, int64_t length, int64_t k,
                       int mode, float* y_a, float* y_max, void* stream);
/* Stage count the reference returns alongside y (pooling.py:37-51, :67-76). */
int64_t sc_pool1d_stages(int op, int64_t k);

/* ---- 1-D convolution ------------------------------------------------------
 * Replaces conv1d_slide / conv1d_reference (kernels.py:220-232,
 * reference.py:33-39) -> _accumulate_taps (reference.py:15-23) with kh = 1.
 * x: (batch, length), w: k taps (HOST) -> y: (batch, length - k + 1). */
int sc_conv1d_f32(const float* x, int64_t batch, int64_t length, const float* w, int64_t k,
                  int mode, float* y, void* stream);

/* ---- 2-D single-channel convolution ----------------------------------------
 * Replaces conv2d_reference / conv2d_slide_generic / conv2d_slide_compound /
 * conv2d_custom3 / conv2d_custom5 (reference.py:26-30, kernels.py:235-275),
 * all of which evaluate _accumulate_taps (reference.py:15-23): valid
 * cross-correlation, stride 1.  x: (batch, h, w), f: (kh, kw) HOST ->
 * y: (batch, h - kh + 1, w - kw + 1).  3x3 / 5x5 / 7x7 (and 1x7) run
 * size-specialised TMA-staged kernels; other sizes a runtime-(kh, kw) kernel. */
int sc_conv2d_f32(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                  int64_t kh, int64_t kw, int mode, float* y, void* stream);

/* Introspection (new; no reference counterpart): output rows per CTA row
 * segment of the tiling sc_conv2d_f32 launches for this shape and mode, 0 when
 * the chosen kernel does not tile rows that way (only the 5x5 / 7x7
 * four-column kernels report one), -1 for invalid dims.  Tests use it to
 * oracle-check windows that straddle segment boundaries. */
int64_t sc_conv2d_segment_rows(int64_t batch, int64_t h, int64_t w, int64_t kh, int64_t kw,
                               int mode);

/* Same formula in float64 -- replaces oracle_conv2d (reference.py:42-47). */
int sc_conv2d_f64(const double* x, int64_t batch, int64_t h, int64_t w, const double* f,
                  int64_t kh, int64_t kw, double* y, void* stream);

/* ---- multi-channel NCHW convolution (new) -----------------
 * x: (n, cin, h, w), wt: (cout, cin, kh, kw) DEVICE, zero padding `pad`,
 * stride 1, no bias -> y: (n, cout, h + 2 pad - kh + 1, w + 2 pad - kw + 1).
 * EXACT mode reproduces the composed oracle: per (n, co), sum over ci
 * ascending of the reference's single-channel conv of the padded plane. */
int sc_conv2d_nchw_f32(const float* x, int64_t n, int64_t cin, int64_t h, int64_t w,
                       const float* wt, int64_t cout, int64_t kh, int64_t kw, int64_t pad,
                       int mode, float* y, void* stream);

/* ---- im2col + GEMM contrast (gemm.py:21-69) --------------------------------
 * sc_im2col_f32: x (h, w) -> cols (oh*ow, kh*kw), row r*ow+c = patch
 * x[r:r+kh, c:c+kw] flattened row-major (gemm.py:21-37), for rows
 * [row0, row0 + nrows) of the output only (chunking for huge images). */
int sc_im2col_f32(const float* x, int64_t h, int64_t w, int64_t kh, int64_t kw,
                  int64_t row0, int64_t nrows, float* cols, void* stream);
/* Row-major c (m, n) = a (m, k) @ b (k, n) with cuBLAS SGEMM, TF32 disabled
 * (replaces gemm.py:40-59).  cuBLAS is resolved with dlopen at first use. */
int sc_gemm_f32(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
                void* stream);
/* conv2d_im2col (gemm.py:62-69): im2col chunks of `chunk_rows` output rows
 * into `cols` (>= chunk_rows*ow*kh*kw floats) then cuBLAS GEMV-as-GEMM with
 * the (kh*kw, 1) filter `f_dev` (DEVICE). */
int sc_conv2d_im2col_f32(const float* x, int64_t h, int64_t w, const float* f_dev, int64_t kh,
                         int64_t kw, float* cols, int64_t chunk_rows, float* y, void* stream);

/* ---- row bands across GPUs (new, BASELINE config 5) ----
 * One host thread drives G GPUs; the context owns one NCCL communicator per
 * device (ncclCommInitAll; NCCL is dlopen'ed) plus a comm stream and events.
 * Band g (device devs[g]) is a DEVICE buffer of rows[g] + kh - 1 rows of w
 * floats: its first rows[g] rows hold input rows of band g, the kh - 1 spare
 * rows receive the first kh - 1 rows of band g + 1 (the halo, NCCL send/recv
 * over NVLink).  ys[g] (DEVICE, on devs[g]) receives rows[g] output rows of
 * w - kw + 1 (the last band: rows[g] - kh + 1).  Concatenating ys over g gives
 * the valid conv of the whole image -- bit-identical, since output row r reads
 * input rows r .. r + kh - 1 only (reference.py:15-23, _accumulate_taps).
 * Per device the interior rows are convolved on streams[g] (NULL = legacy
 * default stream) while the halo is in flight; the kh - 1 boundary rows run
 * after it lands.  timeout_ms > 0: wait for completion, polling
 * ncclCommGetAsyncError; on an NCCL error or timeout return SC_ERR_CUDA and
 * mark the context aborted (destroy then aborts the communicators).
 * timeout_ms <= 0: enqueue only. */
typedef struct sc_rowband sc_rowband;
int sc_rowband_create(int ndev, const int* devs, sc_rowband** ctx);
int sc_rowband_destroy(sc_rowband* ctx);
int sc_rowband_conv2d_f32(sc_rowband* ctx, float* const* bands, const int64_t* rows, int64_t w,
                          const float* f, int64_t kh, int64_t kw, int mode, float* const* ys,
                          void* const* streams, int timeout_ms);

/* ---- host-buffer entry points (chunked H2D / compute / D2H pipeline) -------
 * Same semantics as the device entry points; x and y are HOST pointers. */
int sc_pool1d_f32_host(int op, const float* x, int64_t batch, int64_t length, int64_t k,
                       int mode, float* y, int device);
int sc_pool1d_pair_f32_host(int op_a, const float* x, int64_t batch, int64_t length, int64_t k,
                            int mode, float* y_a, float* y_max, int device);
int sc_conv2d_f32_host(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                       int64_t kh, int64_t kw, int mode, float* y, int device);

#ifdef __cplusplus
}
#endif

#endif /* SLIDECONV_B200_H */
