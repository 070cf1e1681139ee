// Per-CTA timeline of the weights-stationary NCHW kernel on config 4
// (events recorded under -DSC_WS_TRACE, see csrc/nchw_ws.cu):
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
//   -DSC_WS_TRACE -I../../include ws_trace.cu ../../paper_2310_05218_b200/csrc/abi.cu -lcuda -o ws_trace
#include <algorithm>
#include <cstdio>
#include <mutex>
#include <vector>
#include "../../paper_2310_05218_b200/csrc/nchw_ws.cu"

namespace sc {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace sc

int main(int argc, char** argv) {
  const int n = 16, c = 64, h = 112, w = 112;
  float *x, *wt, *y;
  cudaMalloc(&x, (size_t)n * c * h * w * 4);
  cudaMalloc(&y, (size_t)n * c * h * w * 4);
  cudaMalloc(&wt, (size_t)c * c * 9 * 4);
  cudaMemset(x, 0, (size_t)n * c * h * w * 4);
  cudaMemset(wt, 0, (size_t)c * c * 9 * 4);
  for (int it = 0; it < 3; ++it) sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
  cudaDeviceSynchronize();
  // argv[1] == "flush": overwrite a 512 MB buffer first (dirty L2, as the
  // bench's flushed timing of config 4)
  if (argc > 1 && argv[1][0] == 'f') {
    void* fl;
    cudaMalloc(&fl, 512u << 20);
    cudaMemsetAsync(fl, 1, 512u << 20);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  int rc = sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("rc %d %s %.4f ms (pack + conv)\n", rc, cudaGetErrorString(err), ms);
  // the call as a sequence of separately timed launches
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float t_full = 0;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&t_full, a, b);
    }
    printf("full call (pack + conv): %.2f us\n", t_full * 1e3);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&t_full, a, b);
    printf("back to back: %.2f us per call\n", t_full * 1e3 / 20);
  }
  {
    // global timeline of the last call: event-timed call vs kernel spans
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    void* fl;
    cudaMalloc(&fl, 256u << 20);
    for (int it = 0; it < 3; ++it) {
      cudaMemsetAsync(fl, it, 256u << 20);
      cudaEventRecord(a);
      sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ev_ms = 0;
    cudaEventElapsedTime(&ev_ms, a, b);
    static unsigned long long gt[160][2], pk[2];
    cudaMemcpyFromSymbol(gt, sc::g_ws_gt, sizeof gt);
    cudaMemcpyFromSymbol(pk, sc::g_pack_gt, sizeof pk);
    unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
    for (int bb = 0; bb < 144; ++bb) {
      s0 = std::min(s0, gt[bb][0]); s1 = std::max(s1, gt[bb][0]);
      e0 = std::min(e0, gt[bb][1]); e1 = std::max(e1, gt[bb][1]);
    }
    printf("event-timed call %.2f us | globaltimer: pack start -> first conv CTA %.2f, CTA starts spread %.2f, "
           "first CTA end %.2f, last CTA end %.2f us after the first CTA start\n",
           ev_ms * 1e3, ((long long)s0 - (long long)pk[0]) / 1e3, (s1 - s0) / 1e3, (e0 - s0) / 1e3,
           (e1 - s0) / 1e3);
  }
  static unsigned long long tr[160][13];
  printf("trace copy: %s\n", cudaGetErrorString(cudaMemcpyFromSymbol(tr, sc::g_ws_trace, sizeof tr)));
  unsigned long long t0 = ~0ull, tend = 0;
  for (int b = 0; b < 144; ++b) { t0 = std::min(t0, tr[b][0]); tend = std::max(tend, tr[b][5]); }
  printf("kernel span %.2f us\n", (tend - t0) / 1e3);
  const char* names[] = {"start", "A ready", "row0 issued", "last row issued", "last epi", "end", "row0 epi",
                         "1st stage full", "slot r0-1 full", "slot r0+1 full"};
  for (int ev : {0, 7, 8, 9, 1, 2, 6, 3, 4, 5}) {
    std::vector<double> v;
    for (int b = 0; b < 144; ++b) v.push_back((tr[b][ev] - t0) / 1e3);
    std::sort(v.begin(), v.end());
    printf("%-16s min %6.2f  med %6.2f  max %6.2f us (cross-SM clock64, approximate)\n", names[ev], v[0], v[72], v[143]);
  }
  printf("per CTA (us from its start): tma0-before tma0-after 1st-stage pack-done slot0 slot2 A-ready row0-issued row0-epi last-issued last-epi end\n");
  for (int b : {0, 1, 50, 143}) {
    printf("cta %3d:", b);
    for (int ev : {10, 11, 7, 12, 8, 9, 1, 2, 6, 3, 4, 5}) printf(" %8.2f", ((long long)tr[b][ev] - (long long)tr[b][0]) / 1.9e3);
    printf("\n");
  }
  return 0;
}
