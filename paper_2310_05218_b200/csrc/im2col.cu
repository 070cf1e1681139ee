// The incumbent im2col + GEMM path (gemm.py:21-69), as the contrast column of
// every report: a plain CUDA gather that materialises the (oh*ow, kh*kw)
// column matrix (the memory bloat the paper measures), then cuBLAS SGEMM with
// TF32 disabled.  cuBLAS is dlopen'ed at first use, so the library loads (and
// the sliding-window paths run) without it.
#include <cublas_v2.h>
#include <dlfcn.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace sc {
namespace {

__global__ void im2col_kernel(const float* __restrict__ x, int64_t w, int kh, int kw, int64_t ow,
                              int64_t row0, int64_t nrows, float* __restrict__ cols) {
  const int64_t kk = (int64_t)kh * kw;
  const int64_t total = nrows * ow * kk;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / kk;           // output pixel within the chunk
    const int t = (int)(e - p * kk);    // tap j*kw + i
    const int64_t r = row0 + p / ow;
    const int64_t c = p - (p / ow) * ow;
    const int j = t / kw, i = t - (t / kw) * kw;
    cols[e] = __ldg(x + (r + j) * w + c + i);
  }
}

struct Cublas {
  bool ok = false;
  std::string err;
  decltype(&cublasCreate_v2) create = nullptr;
  decltype(&cublasSetStream_v2) set_stream = nullptr;
  decltype(&cublasSetMathMode) set_math = nullptr;
  decltype(&cublasSgemm_v2) sgemm = nullptr;
  cublasHandle_t handle[64] = {nullptr};
  std::mutex mu;
};

Cublas& cublas() {
  static Cublas cb;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("/usr/local/cuda/lib64/libcublas.so.12", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      cb.err = std::string("dlopen libcublas.so.12 failed: ") + dlerror();
      return;
    }
    cb.create = reinterpret_cast<decltype(cb.create)>(dlsym(lib, "cublasCreate_v2"));
    cb.set_stream = reinterpret_cast<decltype(cb.set_stream)>(dlsym(lib, "cublasSetStream_v2"));
    cb.set_math = reinterpret_cast<decltype(cb.set_math)>(dlsym(lib, "cublasSetMathMode"));
    cb.sgemm = reinterpret_cast<decltype(cb.sgemm)>(dlsym(lib, "cublasSgemm_v2"));
    cb.ok = cb.create && cb.set_stream && cb.set_math && cb.sgemm;
    if (!cb.ok) cb.err = "cuBLAS symbols missing";
  });
  return cb;
}

// row-major c(m,n) = a(m,k) @ b(k,n)  ==  column-major c^T = b^T a^T
int gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k,
         cudaStream_t st) {
  Cublas& cb = cublas();
  if (!cb.ok) return fail(SC_ERR_CUBLAS, cb.err);
  if (m > 0x7fffffff || n > 0x7fffffff || k > 0x7fffffff)
    return fail(SC_ERR_UNSUPPORTED, "gemm: dims exceed int32");
  int dev = 0;
  SC_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(cb.mu);
  cublasHandle_t& hd = cb.handle[dev & 63];
  if (!hd) {
    if (cb.create(&hd) != CUBLAS_STATUS_SUCCESS) return fail(SC_ERR_CUBLAS, "cublasCreate failed");
    // plain IEEE SGEMM: no TF32 tensor-op down-conversion
    cb.set_math(hd, CUBLAS_PEDANTIC_MATH);
  }
  cb.set_stream(hd, st);
  const float one = 1.0f, zero = 0.0f;
  cublasStatus_t s = cb.sgemm(hd, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, (int)k, &one, b,
                              (int)n, a, (int)k, &zero, c, (int)n);
  if (s != CUBLAS_STATUS_SUCCESS)
    return fail(SC_ERR_CUBLAS, "cublasSgemm failed (" + std::to_string((int)s) + ")");
  return SC_OK;
}

int im2col(const float* x, int64_t h, int64_t w, int64_t kh, int64_t kw, int64_t row0,
           int64_t nrows, float* cols, cudaStream_t st) {
  const int64_t ow = w - kw + 1;
  const int64_t total = nrows * ow * kh * kw;
  if (total == 0) return SC_OK;
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32));
  im2col_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, w, (int)kh, (int)kw, ow, row0, nrows, cols);
  SC_LAUNCH_CHECK("im2col_kernel");
  return SC_OK;
}

}  // namespace
}  // namespace sc

extern "C" int sc_im2col_f32(const float* x, int64_t h, int64_t w, int64_t kh, int64_t kw,
                             int64_t row0, int64_t nrows, float* cols, void* stream) {
  using namespace sc;
  if (h < 1 || w < 1 || kh < 1 || kw < 1 || kh > h || kw > w)
    return fail(SC_ERR_SHAPE, "im2col: filter exceeds input or non-positive dims");
  const int64_t oh = h - kh + 1;
  if (row0 < 0 || nrows < 0 || row0 + nrows > oh) return fail(SC_ERR_ARG, "im2col: bad row range");
  if (!x || !cols) return fail(SC_ERR_ARG, "im2col: null pointer");
  return im2col(x, h, w, kh, kw, row0, nrows, cols, static_cast<cudaStream_t>(stream));
}

extern "C" int sc_gemm_f32(const float* a, const float* b, float* c, int64_t m, int64_t n,
                           int64_t k, void* stream) {
  using namespace sc;
  if (m < 0 || n < 0 || k < 0) return fail(SC_ERR_SHAPE, "gemm: negative dims");
  if (m == 0 || n == 0) return SC_OK;
  if (!a || !b || !c) return fail(SC_ERR_ARG, "gemm: null pointer");
  return gemm(a, b, c, m, n, k, static_cast<cudaStream_t>(stream));
}

extern "C" int sc_conv2d_im2col_f32(const float* x, int64_t h, int64_t w, const float* f_dev,
                                    int64_t kh, int64_t kw, float* cols, int64_t chunk_rows,
                                    float* y, void* stream) {
  using namespace sc;
  if (h < 1 || w < 1 || kh < 1 || kw < 1 || kh > h || kw > w)
    return fail(SC_ERR_SHAPE, "conv2d_im2col: filter exceeds input or non-positive dims");
  if (!x || !f_dev || !cols || !y) return fail(SC_ERR_ARG, "conv2d_im2col: null pointer");
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  if (chunk_rows < 1) chunk_rows = oh;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int64_t r = 0; r < oh; r += chunk_rows) {
    const int64_t nr = std::min(chunk_rows, oh - r);
    int rc = im2col(x, h, w, kh, kw, r, nr, cols, st);
    if (rc) return rc;
    rc = gemm(cols, f_dev, y + r * ow, nr * ow, 1, kh * kw, st);
    if (rc) return rc;
  }
  return SC_OK;
}
