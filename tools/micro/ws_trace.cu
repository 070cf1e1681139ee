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

int main() {
  const int n = 16, c = 64, h = 112, w = 112;
  float *x, *wt, *y;
  cudaMalloc(&x, (size_t)n * c * h * w * 4);
  cudaMalloc(&y, (size_t)n * c * h * w * 4);
  cudaMalloc(&wt, (size_t)c * c * 9 * 4);
  cudaMemset(x, 0, (size_t)n * c * h * w * 4);
  cudaMemset(wt, 0, (size_t)c * c * 9 * 4);
  for (int it = 0; it < 3; ++it) sc::nchw3x3_ws(x, n, c, h, w, wt, c, y, 0);
  cudaDeviceSynchronize();
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
  static unsigned long long tr[160][8];
  cudaMemcpyFromSymbol(tr, sc::g_ws_trace, sizeof tr);
  unsigned long long t0 = ~0ull, tend = 0;
  for (int b = 0; b < 144; ++b) { t0 = std::min(t0, tr[b][0]); tend = std::max(tend, tr[b][5]); }
  printf("kernel span %.2f us\n", (tend - t0) / 1e3);
  const char* names[] = {"start", "A ready", "row0 issued", "last row issued", "last epi", "end", "row0 epi"};
  for (int ev : {0, 1, 2, 6, 3, 4, 5}) {
    std::vector<double> v;
    for (int b = 0; b < 144; ++b) v.push_back((tr[b][ev] - t0) / 1e3);
    std::sort(v.begin(), v.end());
    printf("%-16s min %6.2f  med %6.2f  max %6.2f us\n", names[ev], v[0], v[72], v[143]);
  }
  for (int b : {0, 1, 50, 143}) {
    printf("cta %3d:", b);
    for (int ev = 0; ev < 7; ++ev) printf(" %8.2f", ((long long)tr[b][ev] - (long long)tr[b][0]) / 1.9e3);
    printf("\n");
  }
  return 0;
}
