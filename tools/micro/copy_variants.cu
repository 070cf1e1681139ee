// Which copy-kernel shape reaches cudaMemcpy DtoD bandwidth on B200?
#include <cstdio>
#include <cuda_runtime.h>

constexpr long N = 256L * 262144;  // floats (268 MB)

template <int U, int HINT>
__global__ void copyk(const float4* __restrict__ x, float4* __restrict__ y, long n4) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long i = (blockIdx.x * (long)blockDim.x) * U + threadIdx.x; i < n4; i += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long j = i + (long)u * blockDim.x;
      if (j < n4) v[u] = HINT & 1 ? __ldcs(x + j) : x[j];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long j = i + (long)u * blockDim.x;
      if (j < n4) {
        if (HINT & 2) __stcs(y + j, v[u]); else y[j] = v[u];
      }
    }
  }
}

// one-shot grid (no grid-stride loop), U float4 per thread
template <int U, int HINT>
__global__ void copy_oneshot(const float4* __restrict__ x, float4* __restrict__ y, long n4) {
  const long base = (long)blockIdx.x * blockDim.x * U + threadIdx.x;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long j = base + (long)u * blockDim.x;
    if (j < n4) v[u] = HINT & 1 ? __ldcs(x + j) : x[j];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const long j = base + (long)u * blockDim.x;
    if (j < n4) { if (HINT & 2) __stcs(y + j, v[u]); else y[j] = v[u]; }
  }
}

int main() {
  float *x, *y;
  cudaMalloc(&x, N * 4);
  cudaMalloc(&y, N * 4);
  cudaMemset(x, 0, N * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long n4 = N / 4;
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("%-34s %7.1f us %6.0f GB/s\n", name, ms / 20 * 1e3, 8.0 * N / (ms / 20 * 1e-3) / 1e9);
    }
  };
  run("cudaMemcpyAsync DtoD", [&] { cudaMemcpyAsync(y, x, N * 4, cudaMemcpyDeviceToDevice); });
  run("grid-stride U1", [&] { copyk<1, 0><<<sms * 8, 256>>>((float4*)x, (float4*)y, n4); });
  run("grid-stride U4", [&] { copyk<4, 0><<<sms * 8, 256>>>((float4*)x, (float4*)y, n4); });
  run("grid-stride U4 ldcs", [&] { copyk<4, 1><<<sms * 8, 256>>>((float4*)x, (float4*)y, n4); });
  run("grid-stride U4 stcs", [&] { copyk<4, 2><<<sms * 8, 256>>>((float4*)x, (float4*)y, n4); });
  run("grid-stride U4 ldcs+stcs", [&] { copyk<4, 3><<<sms * 8, 256>>>((float4*)x, (float4*)y, n4); });
  run("grid-stride U8 x4/SM", [&] { copyk<8, 0><<<sms * 4, 256>>>((float4*)x, (float4*)y, n4); });
  run("oneshot U4", [&] { copy_oneshot<4, 0><<<(unsigned)((n4 + 1023) / 1024), 256>>>((float4*)x, (float4*)y, n4); });
  run("oneshot U4 stcs", [&] { copy_oneshot<4, 2><<<(unsigned)((n4 + 1023) / 1024), 256>>>((float4*)x, (float4*)y, n4); });
  run("oneshot U8", [&] { copy_oneshot<8, 0><<<(unsigned)((n4 + 2047) / 2048), 256>>>((float4*)x, (float4*)y, n4); });
  run("oneshot U2", [&] { copy_oneshot<2, 0><<<(unsigned)((n4 + 511) / 512), 256>>>((float4*)x, (float4*)y, n4); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
