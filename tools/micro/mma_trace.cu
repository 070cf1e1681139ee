// Event trace of the slide-MMA conv kernel, CTA (0,0,0): per role the
// clock64 stamps recorded under -DSC_MMA_TRACE (see csrc/conv2d_mma.cu).
//   ./mma_trace [h] [w] [random 0/1]
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -DSC_MMA_TRACE \
//   -I../../include tools/micro/mma_trace.cu paper_.../csrc/abi.cu -lcuda -o mma_trace
#include <cstdio>
#include <mutex>
#include <vector>
#include "../../paper_2310_05218_b200/csrc/conv2d_mma.cu"

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

__global__ void fill_uniform(float* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (uint32_t)(i >> 32);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    x[i] = (h >> 8) * (2.0f / 16777216.0f) - 1.0f;
  }
}

int main(int argc, char** argv) {
  const int64_t h = argc > 1 ? atoll(argv[1]) : 8192, w = argc > 2 ? atoll(argv[2]) : 65536;
  float *x, *y;
  cudaMalloc(&x, h * w * 4);
  cudaMalloc(&y, h * w * 4);
  cudaMemset(x, 0, h * w * 4);
  if (argc > 3 && atoi(argv[3])) fill_uniform<<<1184, 256>>>(x, h * w);
  float f[49];
  for (int i = 0; i < 49; ++i) f[i] = 0.01f * (i + 1);
  for (int it = 0; it < 3; ++it) {
    int rc = sc::conv2d_mma(x, 1, h, w, f, 7, 7, y, 0);
    if (rc) { printf("rc %d\n", rc); return 1; }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  sc::conv2d_mma(x, 1, h, w, f, 7, 7, y, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("%s  %.3f ms for %lld x %lld\n", cudaGetErrorString(err), ms, (long long)h, (long long)w);
  static long long tr[8][4096];
  cudaMemcpyFromSymbol(tr, sc::g_mma_trace, sizeof tr);
  const char* names[] = {"issuer0", "issuer1", "split0", "split1", "epi", "producer"};
  long long t0 = tr[5][0];
  for (int r = 0; r < 6; ++r) {
    printf("%s:", names[r]);
    const int per = r == 5 ? 2 : 3;
    for (int i = 0; i < 12; ++i) {
      printf(" [");
      for (int j = 0; j < per; ++j) printf("%lld%s", tr[r][per * i + j] - t0, j + 1 < per ? "," : "");
      printf("]");
    }
    printf("\n");
  }
  {
    double a[4] = {0, 0, 0, 0}; int n = 0;
    for (int i = 40; i < 400; i += 2) {
      if (!tr[4][5 * i + 10]) break;
      for (int j = 0; j < 4; ++j) a[j] += tr[4][5 * i + j + 1] - tr[4][5 * i + j];
      ++n;
    }
    printf("epi period per 2 batches %.0f\n", (double)(tr[4][5 * 398] - tr[4][5 * 40]) / 179);
    printf("epi5: wait_done %.0f  ld %.0f  zero+stg issue %.0f  wait_st+arrive %.0f (n=%d)\n", a[0] / n, a[1] / n, a[2] / n, a[3] / n, n);
  }
  for (int r = 0; r < 2; ++r) {
    double a[4] = {0, 0, 0, 0}; int n = 0;
    for (int i = 100; i < 400; ++i) {
      if (!tr[r][5 * i + 5]) break;
      for (int j = 0; j < 4; ++j) a[j] += tr[r][5 * i + j + 1] - tr[r][5 * i + j];
      ++n;
    }
    printf("issuer%d: a_full %.0f  zeroed %.0f  mma issue %.0f  commits %.0f (n=%d)\n", r, a[0] / n, a[1] / n, a[2] / n, a[3] / n, n);
  }
  {
    double a[3] = {0, 0, 0}; int n = 0;
    for (int t = 200; t < 800; t += 2) {
      if (!tr[2][4 * t + 7]) break;
      a[0] += tr[2][4 * t + 1] - tr[2][4 * t];       // st_full wait (+ nothing)
      a[1] += tr[2][4 * t + 2] - tr[2][4 * t + 1];   // split math row t
      a[2] += tr[2][4 * t + 3] - tr[2][4 * t + 2];   // a_free wait + st + arrive row t
      ++n;
    }
    printf("split: st_full %.0f  math %.0f  a_free+st+arrive %.0f (n=%d)\n", a[0] / n, a[1] / n, a[2] / n, n);
    for (int t = 300; t < 306; ++t) printf("  t=%d split a_free-wait-start %lld done %lld | issuer a_full-wait %lld got %lld issued %lld\n", t, tr[2][4*t+2]-t0, tr[2][4*t+3]-t0, tr[0][5*t]-t0, tr[0][5*t+1]-t0, tr[0][5*t+3]-t0);
  }
  // steady-state averages over items 100..400
  for (int r = 0; r < 0; ++r) {
    double a = 0, b = 0, tot = 0; int n = 0;
    for (int i = 100; i < 400; ++i) {
      if (!tr[r][3 * i + 3]) break;
      a += tr[r][3 * i + 1] - tr[r][3 * i];
      b += tr[r][3 * i + 2] - tr[r][3 * i + 1];
      tot += tr[r][3 * i + 3] - tr[r][3 * i];
      ++n;
    }
    if (n) printf("%s steady: wait %.0f  work %.0f  period %.0f cycles (n=%d)\n", names[r], a / n, b / n, tot / n, n);
  }
  return 0;
}
