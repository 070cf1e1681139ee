// Row-band 2-D convolution across several GPUs driven by ONE host thread
// (BASELINE config 5: one 65,536^2 image, 7x7, row bands on 1/2/4/8 GPUs).
//
// A valid conv output row r reads input rows r .. r + kh - 1 only
// (reference.py:15-23), so band g is exact once it also holds the first
// kh - 1 rows of band g + 1.  Each band lives in a caller buffer of
// rows_g + kh - 1 rows on its own GPU; the spare rows receive that halo.
// One call, per GPU g, in stream order:
//   comm stream:  wait(caller stream) -> grouped ncclSend(first kh-1 rows ->
//                 g - 1) / ncclRecv(kh-1 rows <- g + 1 into the spare rows)
//   caller stream: interior conv (output rows 0 .. rows_g - kh, which never
//                 read the halo) -- overlaps the exchange over NVLink --
//                 then wait(comm stream) and the 2(kh - 1)-row boundary strip
//                 [rows_g - kh + 1, rows_g + kh - 1) -> its kh - 1 output rows
//                 (a contiguous view of the same buffer: no copy, no concat).
// The last band has no successor and produces rows_g - kh + 1 rows.
// NCCL is dlopen'ed at first use (the library loads without it).  With
// timeout_ms > 0 the call waits for completion, polling
// ncclCommGetAsyncError; a hung or failed exchange aborts the communicators
// and returns SC_ERR_CUDA instead of blocking forever.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace sc {
int conv2d_f32_dispatch(const float* x, int64_t batch, int64_t h, int64_t w, const float* f,
                        int64_t kh, int64_t kw, bool exact, float* y, cudaStream_t st);

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
  ncclResult_t (*async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) { return dlsym(lib, n); };
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.comm_abort = reinterpret_cast<decltype(api.comm_abort)>(sym("ncclCommAbort"));
    api.async_error = reinterpret_cast<decltype(api.async_error)>(sym("ncclCommGetAsyncError"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.ok = api.comm_init_all && api.comm_destroy && api.comm_abort && api.async_error &&
             api.group_start && api.group_end && api.send && api.recv && api.error_string;
    if (!api.ok) api.err = "NCCL symbols missing";
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(SC_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace
}  // namespace sc

struct sc_rowband {
  std::vector<int> devs;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> comm_streams;
  std::vector<cudaEvent_t> ev_ready, ev_halo, ev_done;
  bool aborted = false;
};

namespace {

// Run fn with device `dev` current, restoring the caller's device.
template <class F>
int on_device(int dev, F&& fn) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) return sc::cuda_fail(e, "cudaSetDevice");
  const int rc = fn();
  cudaSetDevice(prev);
  return rc;
}

void release(sc_rowband* ctx) {
  auto& api = sc::nccl();
  for (size_t g = 0; g < ctx->devs.size(); ++g) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(ctx->devs[g]);
    if (g < ctx->comms.size() && ctx->comms[g]) {
      if (ctx->aborted) api.comm_abort(ctx->comms[g]);
      else api.comm_destroy(ctx->comms[g]);
    }
    if (g < ctx->comm_streams.size() && ctx->comm_streams[g])
      cudaStreamDestroy(ctx->comm_streams[g]);
    for (auto* v : {&ctx->ev_ready, &ctx->ev_halo, &ctx->ev_done})
      if (g < v->size() && (*v)[g]) cudaEventDestroy((*v)[g]);
    cudaSetDevice(prev);
  }
  delete ctx;
}

}  // namespace

extern "C" int sc_rowband_create(int ndev, const int* devs, sc_rowband** out) {
  using namespace sc;
  if (!out) return fail(SC_ERR_ARG, "rowband: null context pointer");
  *out = nullptr;
  if (ndev < 1 || ndev > 64 || !devs) return fail(SC_ERR_ARG, "rowband: need 1..64 devices");
  auto& api = nccl();
  if (!api.ok) return fail(SC_ERR_CUDA, api.err);
  auto* ctx = new sc_rowband;
  ctx->devs.assign(devs, devs + ndev);
  ctx->comms.assign(ndev, nullptr);
  ctx->comm_streams.assign(ndev, nullptr);
  ctx->ev_ready.assign(ndev, nullptr);
  ctx->ev_halo.assign(ndev, nullptr);
  ctx->ev_done.assign(ndev, nullptr);
  ncclResult_t r = api.comm_init_all(ctx->comms.data(), ndev, devs);
  if (r != ncclSuccess) {
    ctx->comms.assign(ndev, nullptr);
    release(ctx);
    return nccl_fail(r, "ncclCommInitAll");
  }
  for (int g = 0; g < ndev; ++g) {
    const int rc = on_device(devs[g], [&]() -> int {
      SC_CUDA(cudaStreamCreateWithFlags(&ctx->comm_streams[g], cudaStreamNonBlocking));
      SC_CUDA(cudaEventCreateWithFlags(&ctx->ev_ready[g], cudaEventDisableTiming));
      SC_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo[g], cudaEventDisableTiming));
      SC_CUDA(cudaEventCreateWithFlags(&ctx->ev_done[g], cudaEventDisableTiming));
      return SC_OK;
    });
    if (rc) {
      release(ctx);
      return rc;
    }
  }
  *out = ctx;
  return SC_OK;
}

extern "C" int sc_rowband_destroy(sc_rowband* ctx) {
  if (ctx) release(ctx);
  return SC_OK;
}

extern "C" int sc_rowband_conv2d_f32(sc_rowband* ctx, float* const* bands, const int64_t* rows,
                                     int64_t w, const float* f, int64_t kh, int64_t kw, int mode,
                                     float* const* ys, void* const* streams, int timeout_ms) {
  using namespace sc;
  if (!ctx || !bands || !rows || !f || !ys) return fail(SC_ERR_ARG, "rowband: null pointer");
  if (ctx->aborted) return fail(SC_ERR_CUDA, "rowband: context aborted by an earlier failure");
  if (mode != SC_MODE_FAST && mode != SC_MODE_EXACT) return fail(SC_ERR_ARG, "bad mode");
  const int G = (int)ctx->devs.size();
  if (kh < 1 || kw < 1 || kw > w) return fail(SC_ERR_SHAPE, "rowband: filter exceeds input");
  const int64_t halo = kh - 1;
  for (int g = 0; g < G; ++g) {
    const bool last = g == G - 1;
    if (rows[g] < (last ? kh : std::max<int64_t>(1, halo)))
      return fail(SC_ERR_SHAPE, "rowband: band " + std::to_string(g) + " of " +
                                    std::to_string(rows[g]) + " rows too small for a " +
                                    std::to_string(kh) + "x" + std::to_string(kw) + " filter");
    if (!bands[g] || !ys[g]) return fail(SC_ERR_ARG, "rowband: null band / output pointer");
  }
  auto& api = nccl();
  const bool exact = mode == SC_MODE_EXACT;
  const int64_t ow = w - kw + 1;
  auto user_stream = [&](int g) {
    return streams ? static_cast<cudaStream_t>(streams[g]) : cudaStream_t(nullptr);
  };
  // 1. the comm streams start when each band's data is ready on its stream
  for (int g = 0; g < G && halo > 0 && G > 1; ++g) {
    int rc = on_device(ctx->devs[g], [&]() -> int {
      SC_CUDA(cudaEventRecord(ctx->ev_ready[g], user_stream(g)));
      SC_CUDA(cudaStreamWaitEvent(ctx->comm_streams[g], ctx->ev_ready[g], 0));
      return SC_OK;
    });
    if (rc) return rc;
  }
  // 2. the halo exchange: one NCCL group over all devices (single thread)
  if (halo > 0 && G > 1) {
    ncclResult_t r = api.group_start();
    if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    for (int g = 0; g < G; ++g) {
      const size_t n = (size_t)(halo * w);
      if (g > 0 && (r = api.send(bands[g], n, ncclFloat32, g - 1, ctx->comms[g],
                                  ctx->comm_streams[g])) != ncclSuccess)
        break;
      if (g < G - 1 && (r = api.recv(bands[g] + rows[g] * w, n, ncclFloat32, g + 1, ctx->comms[g],
                                      ctx->comm_streams[g])) != ncclSuccess)
        break;
    }
    const ncclResult_t r2 = api.group_end();
    if (r != ncclSuccess) return nccl_fail(r, "ncclSend/ncclRecv");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
  }
  // 3. interior (overlaps the exchange), then the boundary strip
  for (int g = 0; g < G; ++g) {
    int rc = on_device(ctx->devs[g], [&]() -> int {
      cudaStream_t st = user_stream(g);
      const bool last = g == G - 1 || halo == 0;
      const int64_t n_int = rows[g] - kh + 1;  // output rows needing no halo
      if (n_int > 0) {
        int r = conv2d_f32_dispatch(bands[g], 1, rows[g], w, f, kh, kw, exact, ys[g], st);
        if (r) return r;
      }
      if (!last) {
        SC_CUDA(cudaEventRecord(ctx->ev_halo[g], ctx->comm_streams[g]));
        SC_CUDA(cudaStreamWaitEvent(st, ctx->ev_halo[g], 0));
        const int64_t r0 = std::max<int64_t>(0, n_int);
        int r = conv2d_f32_dispatch(bands[g] + r0 * w, 1, rows[g] + halo - r0, w, f, kh, kw,
                                    exact, ys[g] + r0 * ow, st);
        if (r) return r;
      }
      SC_CUDA(cudaEventRecord(ctx->ev_done[g], st));
      return SC_OK;
    });
    if (rc) return rc;
  }
  if (timeout_ms <= 0) return SC_OK;
  // 4. bounded wait: completion events + NCCL async errors
  const auto t_end = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  std::vector<bool> done(G, false);
  for (int left = G; left > 0;) {
    for (int g = 0; g < G; ++g) {
      if (done[g]) continue;
      ncclResult_t ar = ncclSuccess;
      if (api.async_error(ctx->comms[g], &ar) == ncclSuccess && ar != ncclSuccess &&
          ar != ncclInProgress) {
        ctx->aborted = true;
        return nccl_fail(ar, "rowband: NCCL async error");
      }
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(ctx->devs[g]);
      const cudaError_t q = cudaEventQuery(ctx->ev_done[g]);
      cudaSetDevice(prev);
      if (q == cudaSuccess) {
        done[g] = true;
        --left;
      } else if (q != cudaErrorNotReady) {
        return cuda_fail(q, "rowband: band completion");
      }
    }
    if (left > 0) {
      if (std::chrono::steady_clock::now() > t_end) {
        ctx->aborted = true;  // communicators are aborted at destroy
        return fail(SC_ERR_CUDA, "rowband: halo exchange / band conv timed out after " +
                                     std::to_string(timeout_ms) + " ms");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  return SC_OK;
}
