// Host-buffer entry points: a chunked H2D -> kernel -> D2H pipeline.
//
// The reference's callers pass host (numpy) arrays and get host arrays back
// (SURVEY 8(b)).  Here x is split into chunks (rows of signals, or row bands
// of images with a kh-1 row halo -- banded evaluation is bit-identical to
// whole-image evaluation); chunk c runs on slot c % 3, each
// slot owning a CUDA stream and device buffers, so the H2D copy of chunk c+1,
// the kernel of chunk c and the D2H copy of chunk c-1 overlap on the two copy
// engines and the SMs.  Pinned host buffers are copied directly; pageable
// ones go through a pinned staging ring filled by parallel host memcpy.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace sc {
int conv2d_f32_dispatch(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                        int64_t kh, int64_t kw, bool exact, float* y, cudaStream_t st);
}

extern "C" int sc_pool1d_f32(int op, const float* x, int64_t batch, int64_t length, int64_t k,
                             int mode, float* y, void* stream);
extern "C" int sc_pool1d_pair_f32(int op_a, const float* x, int64_t batch, int64_t length,
                                  int64_t k, int mode, float* y_a, float* y_max, void* stream);

namespace sc {
namespace {

constexpr int kSlots = 3;
constexpr size_t kMaxChunkBytes = size_t(64) << 20;

// Chunk size: ~1/16 of the transfer (so the unoverlapped first H2D and last
// D2H are short), between 8 and 64 MiB (SC_HOST_CHUNK_MB overrides).
// Chunk sizes (in units: signals, images or output rows) that ramp up
// geometrically from `min_unit` to `full` and back down at the end, so the
// first H2D copy and the last D2H copy -- the parts of the pipeline that
// cannot overlap anything -- are small.
std::vector<int64_t> ramp_sizes(int64_t total, int64_t full, int64_t min_unit) {
  std::vector<int64_t> up, out;
  int64_t s = std::max<int64_t>(1, min_unit), used = 0;
  while (s < full && used + 2 * s <= total) {
    up.push_back(s);
    used += 2 * s;
    s *= 2;
  }
  out = up;
  for (int64_t mid = total - used; mid > 0;) {
    const int64_t c = std::min(full, mid);
    out.push_back(c);
    mid -= c;
  }
  for (auto it = up.rbegin(); it != up.rend(); ++it) out.push_back(*it);
  return out;
}

size_t chunk_bytes(size_t total) {
  if (const char* e = getenv("SC_HOST_CHUNK_MB")) {
    const long mb = atol(e);
    if (mb >= 1 && mb <= 1024) return size_t(mb) << 20;
  }
  return std::min(kMaxChunkBytes, std::max(size_t(8) << 20, total / 16));
}

struct Slot {
  cudaStream_t stream = nullptr;
  float* d_in = nullptr;
  float* d_out = nullptr;
  float* d_out2 = nullptr;  // second output stream (fused pooling pair)
  size_t in_cap = 0, out_cap = 0, out2_cap = 0;
  float* h_in = nullptr;   // pinned staging
  float* h_out = nullptr;
  float* h_out2 = nullptr;
  size_t h_in_cap = 0, h_out_cap = 0, h_out2_cap = 0;
  // pending pageable write-back of the chunk last issued on this slot
  float* wb_dst = nullptr;
  size_t wb_bytes = 0;
  float* wb_dst2 = nullptr;
  size_t wb_bytes2 = 0;
};

struct DeviceCtx {
  std::mutex mu;
  bool init = false;
  Slot slot[kSlots];
};

DeviceCtx& ctx_for(int dev) {
  static DeviceCtx ctx[64];
  return ctx[dev & 63];
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t kMin = size_t(4) << 20;
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t parts = std::min<size_t>(std::min<size_t>(hw, 8), std::max<size_t>(1, bytes / kMin));
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t step = (bytes + parts - 1) / parts;
  for (size_t p = 0; p < parts; ++p) {
    const size_t off = p * step;
    if (off >= bytes) break;
    const size_t n = std::min(step, bytes - off);
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n);
    });
  }
  for (auto& t : th) t.join();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int grow_dev(float** p, size_t* cap, size_t need) {
  if (*cap >= need) return SC_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  SC_CUDA(cudaMalloc(reinterpret_cast<void**>(p), need));
  *cap = need;
  return SC_OK;
}

int grow_host(float** p, size_t* cap, size_t need) {
  if (*cap >= need) return SC_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *cap = 0;
  SC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(p), need, cudaHostAllocDefault));
  *cap = need;
  return SC_OK;
}

struct Chunk {
  const float* in;
  size_t in_bytes;
  float* out;
  size_t out_bytes;
  std::function<int(const float*, float*, float*, cudaStream_t)> run;  // (in, out, out2, stream)
  float* out2 = nullptr;  // second output of the chunk (fused pooling pair), else null
  size_t out2_bytes = 0;
};

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    ok_ = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }
  bool ok() const { return ok_; }

 private:
  int prev_ = 0;
  bool ok_ = false;
};

int finish_slot(Slot& s) {
  SC_CUDA(cudaStreamSynchronize(s.stream));
  if (s.wb_dst) {
    parallel_memcpy(s.wb_dst, s.h_out, s.wb_bytes);
    s.wb_dst = nullptr;
  }
  if (s.wb_dst2) {
    parallel_memcpy(s.wb_dst2, s.h_out2, s.wb_bytes2);
    s.wb_dst2 = nullptr;
  }
  return SC_OK;
}

int run_pipeline(int dev, std::vector<Chunk>& chunks, bool in_pinned, bool out_pinned) {
  DeviceGuard guard(dev);
  if (!guard.ok()) return fail(SC_ERR_CUDA, "cudaSetDevice failed");
  DeviceCtx& ctx = ctx_for(dev);
  std::lock_guard<std::mutex> lock(ctx.mu);
  if (!ctx.init) {
    for (auto& s : ctx.slot) SC_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    ctx.init = true;
  }
  size_t max_in = 0, max_out = 0, max_out2 = 0;
  for (auto& c : chunks) {
    max_in = std::max(max_in, c.in_bytes);
    max_out = std::max(max_out, c.out_bytes);
    max_out2 = std::max(max_out2, c.out2_bytes);
  }
  for (auto& s : ctx.slot) {
    int rc;
    if ((rc = grow_dev(&s.d_in, &s.in_cap, max_in))) return rc;
    if ((rc = grow_dev(&s.d_out, &s.out_cap, max_out))) return rc;
    if (!in_pinned && (rc = grow_host(&s.h_in, &s.h_in_cap, max_in))) return rc;
    if (!out_pinned && (rc = grow_host(&s.h_out, &s.h_out_cap, max_out))) return rc;
    if (max_out2 && (rc = grow_dev(&s.d_out2, &s.out2_cap, max_out2))) return rc;
    if (max_out2 && !out_pinned && (rc = grow_host(&s.h_out2, &s.h_out2_cap, max_out2))) return rc;
  }
  int status = SC_OK;
  for (size_t i = 0; i < chunks.size() && status == SC_OK; ++i) {
    Slot& s = ctx.slot[i % kSlots];
    Chunk& c = chunks[i];
    // A slot's device buffers are reused by chunk i + kSlots on the same
    // stream, so stream order alone protects them.  The host only has to
    // wait when it touches the staging buffers (pageable input / output):
    // with pinned data everything is enqueued up front and the copy engines
    // never wait for a host wake-up.
    if (!(in_pinned && out_pinned) && (status = finish_slot(s))) break;
    const float* src = c.in;
    if (!in_pinned) {
      parallel_memcpy(s.h_in, c.in, c.in_bytes);
      src = s.h_in;
    }
    if (cudaMemcpyAsync(s.d_in, src, c.in_bytes, cudaMemcpyHostToDevice, s.stream) != cudaSuccess) {
      status = cuda_fail(cudaGetLastError(), "H2D copy");
      break;
    }
    if ((status = c.run(s.d_in, s.d_out, s.d_out2, s.stream))) break;
    float* dst = out_pinned ? c.out : s.h_out;
    if (cudaMemcpyAsync(dst, s.d_out, c.out_bytes, cudaMemcpyDeviceToHost, s.stream) !=
        cudaSuccess) {
      status = cuda_fail(cudaGetLastError(), "D2H copy");
      break;
    }
    if (!out_pinned) {
      s.wb_dst = c.out;
      s.wb_bytes = c.out_bytes;
    }
    if (c.out2) {
      float* dst2 = out_pinned ? c.out2 : s.h_out2;
      if (cudaMemcpyAsync(dst2, s.d_out2, c.out2_bytes, cudaMemcpyDeviceToHost, s.stream) !=
          cudaSuccess) {
        status = cuda_fail(cudaGetLastError(), "D2H copy");
        break;
      }
      if (!out_pinned) {
        s.wb_dst2 = c.out2;
        s.wb_bytes2 = c.out2_bytes;
      }
    }
  }
  for (auto& s : ctx.slot) {
    int rc = finish_slot(s);
    if (status == SC_OK) status = rc;
  }
  return status;
}

}  // namespace
}  // namespace sc

namespace sc {
namespace {

// op_a / y: the single op (y_max null), or the fused pair's first op with
// y_max its maxima; chunking is the same, a pair chunk carries two outputs
int pool1d_host(int op, const float* x, int64_t batch, int64_t length, int64_t k, int mode,
                float* y, float* y_max, int device) {
  if (batch < 0 || length < 1) return fail(SC_ERR_SHAPE, "pool1d: signal length must be >= 1");
  if (k < 1 || k > length)
    return fail(SC_ERR_SHAPE, "window " + std::to_string(k) + " out of range for length " +
                                  std::to_string(length));
  if (batch == 0) return SC_OK;
  if (!x || !y) return fail(SC_ERR_ARG, "pool1d: null pointer");
  const bool pair = y_max != nullptr;
  const int64_t out_len = length - k + 1;
  auto run_op = [=](const float* din, int64_t rows, int64_t len, float* dout, float* dout2,
                    cudaStream_t st) {
    return pair ? sc_pool1d_pair_f32(op, din, rows, len, k, mode, dout, dout2, st)
                : sc_pool1d_f32(op, din, rows, len, k, mode, dout, st);
  };
  std::vector<Chunk> chunks;
  const int64_t row_bytes = length * (int64_t)sizeof(float);
  const size_t kChunkBytes = chunk_bytes((size_t)(batch * row_bytes));
  if (row_bytes <= (int64_t)kChunkBytes) {
    const int64_t rows = std::max<int64_t>(1, (int64_t)kChunkBytes / row_bytes);
    int64_t r = 0;
    for (const int64_t nr : ramp_sizes(batch, rows, 1)) {
      const int64_t r0 = r;
      r += nr;
      const size_t ob = (size_t)(nr * out_len) * sizeof(float);
      chunks.push_back({x + r0 * length, (size_t)(nr * length) * sizeof(float), y + r0 * out_len,
                        ob,
                        [=](const float* din, float* dout, float* dout2, cudaStream_t st) {
                          return run_op(din, nr, length, dout, dout2, st);
                        },
                        pair ? y_max + r0 * out_len : nullptr, pair ? ob : 0});
    }
  } else {
    // one signal is larger than a chunk: segments with a k-1 sample overlap.
    // Each segment carries at least 3 (k - 1) outputs (the chunk grows with
    // k), so the re-sent overlap stays under a quarter of the traffic even
    // when k - 1 exceeds the nominal chunk.
    const int64_t seg = std::max<int64_t>(
        {1, (int64_t)(kChunkBytes / sizeof(float)) - (k - 1), 3 * (k - 1)});
    for (int64_t r = 0; r < batch; ++r)
      for (int64_t o = 0; o < out_len; o += seg) {
        const int64_t no = std::min(seg, out_len - o);
        const int64_t ni = no + k - 1;
        const size_t ob = (size_t)no * sizeof(float);
        chunks.push_back({x + r * length + o, (size_t)ni * sizeof(float), y + r * out_len + o, ob,
                          [=](const float* din, float* dout, float* dout2, cudaStream_t st) {
                            return run_op(din, 1, ni, dout, dout2, st);
                          },
                          pair ? y_max + r * out_len + o : nullptr, pair ? ob : 0});
      }
  }
  return run_pipeline(device, chunks, is_pinned(x), is_pinned(y) && (!pair || is_pinned(y_max)));
}

}  // namespace
}  // namespace sc

extern "C" int sc_pool1d_f32_host(int op, const float* x, int64_t batch, int64_t length, int64_t k,
                                  int mode, float* y, int device) {
  using namespace sc;
  if (op < SC_POOL_SUM || op > SC_POOL_MAX) return fail(SC_ERR_ARG, "pool1d: bad op");
  return pool1d_host(op, x, batch, length, k, mode, y, nullptr, device);
}

// Fused pair on host buffers: x goes over the link ONCE for both outputs.
extern "C" int sc_pool1d_pair_f32_host(int op_a, const float* x, int64_t batch, int64_t length,
                                       int64_t k, int mode, float* y_a, float* y_max,
                                       int device) {
  using namespace sc;
  if (op_a != SC_POOL_SUM && op_a != SC_POOL_AVG)
    return fail(SC_ERR_ARG, "pool1d_pair: first op must be SUM or AVG");
  if (!y_max && batch > 0) return fail(SC_ERR_ARG, "pool1d: null pointer");
  if (y_a == y_max && batch > 0) return fail(SC_ERR_ARG, "pool1d_pair: outputs alias");
  return pool1d_host(op_a, x, batch, length, k, mode, y_a, y_max, device);
}

extern "C" int sc_conv2d_f32_host(const float* x, int64_t batch, int64_t h, int64_t w,
                                  const float* f, int64_t kh, int64_t kw, int mode, float* y,
                                  int device) {
  using namespace sc;
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return fail(SC_ERR_ARG, "bad mode");
  if (batch < 0 || h < 1 || w < 1 || kh < 1 || kw < 1)
    return fail(SC_ERR_SHAPE, "dims must be positive");
  if (kh > h || kw > w) return fail(SC_ERR_SHAPE, "filter exceeds input");
  if (batch == 0) return SC_OK;
  if (!x || !f || !y) return fail(SC_ERR_ARG, "conv2d: null pointer");
  const int64_t oh = h - kh + 1, ow = w - kw + 1;
  const bool exact = mode == SC_MODE_EXACT;
  std::vector<float> taps(f, f + kh * kw);  // outlives the lambdas below
  std::vector<Chunk> chunks;
  const int64_t img_bytes = h * w * (int64_t)sizeof(float);
  const size_t kChunkBytes = chunk_bytes((size_t)(batch * img_bytes));
  if (img_bytes <= (int64_t)kChunkBytes) {
    const int64_t imgs = std::max<int64_t>(1, (int64_t)kChunkBytes / img_bytes);
    int64_t b_next = 0;
    for (const int64_t nb : ramp_sizes(batch, imgs, 1)) {
      const int64_t b = b_next;
      b_next += nb;
      chunks.push_back({x + b * h * w, (size_t)(nb * h * w) * sizeof(float), y + b * oh * ow,
                        (size_t)(nb * oh * ow) * sizeof(float),
                        [=, &taps](const float* din, float* dout, float*, cudaStream_t st) {
                          return conv2d_f32_dispatch(din, nb, h, w, taps.data(), kh, kw, exact,
                                                     dout, st);
                        }});
    }
  } else {
    // row bands with a kh-1 row halo (bit-identical to the whole image); at
    // least 3 (kh - 1) output rows per band so the re-sent halo stays under a
    // quarter of the traffic for tall filters on wide images
    const int64_t band = std::max<int64_t>(
        {1, (int64_t)kChunkBytes / (w * (int64_t)sizeof(float)) - (kh - 1), 3 * (kh - 1)});
    for (int64_t b = 0; b < batch; ++b) {
      int64_t o_next = 0;
      for (const int64_t no : ramp_sizes(oh, band, std::max<int64_t>(1, band / 8))) {
        const int64_t o = o_next;
        o_next += no;
        const int64_t ni = no + kh - 1;
        chunks.push_back({x + (b * h + o) * w, (size_t)(ni * w) * sizeof(float),
                          y + (b * oh + o) * ow, (size_t)(no * ow) * sizeof(float),
                          [=, &taps](const float* din, float* dout, float*, cudaStream_t st) {
                            return conv2d_f32_dispatch(din, 1, ni, w, taps.data(), kh, kw, exact,
                                                       dout, st);
                          }});
      }
    }
  }
  return run_pipeline(device, chunks, is_pinned(x), is_pinned(y));
}
