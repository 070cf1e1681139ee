// Microbenchmark: what write pattern reaches the copy bandwidth for a
// (256 x 262144) -> (256 x 262129) float32 map (row pitches 16B-aligned in,
// unaligned out), as in sliding-window pooling with k = 16.
#include <cstdio>
#include <cuda_runtime.h>

constexpr long B = 256, L = 262144, K = 16, OL = L - K + 1;

__global__ void copy4(const float4* __restrict__ x, float4* __restrict__ y, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    y[i] = x[i];
}

// read rows with float4, write the first OL of each row with 32-bit coalesced stores
__global__ void rows_st32(const float* __restrict__ x, float* __restrict__ y) {
  const long tiles_per_row = (OL + 1023) / 1024;
  for (long t = blockIdx.x; t < B * tiles_per_row; t += gridDim.x) {
    const long row = t / tiles_per_row, c0 = (t % tiles_per_row) * 1024;
    const float4 v = reinterpret_cast<const float4*>(x + row * L + c0)[threadIdx.x];
    __shared__ float s[1024];
    reinterpret_cast<float4*>(s)[threadIdx.x] = v;
    __syncthreads();
    for (int j = threadIdx.x; j < 1024; j += 256)
      if (c0 + j < OL) y[row * OL + c0 + j] = s[j];
    __syncthreads();
  }
}

// same, but write 16B-aligned float4 chunks in flat output space
__global__ void rows_st128(const float* __restrict__ x, float* __restrict__ y) {
  const long tiles_per_row = (OL + 1023) / 1024;
  __shared__ float s[1024 + 8];
  for (long t = blockIdx.x; t < B * tiles_per_row; t += gridDim.x) {
    const long row = t / tiles_per_row, c0 = (t % tiles_per_row) * 1024;
    const long n = min(1024L, OL - c0);
    const float4 v = reinterpret_cast<const float4*>(x + row * L + c0)[threadIdx.x];
    reinterpret_cast<float4*>(s)[threadIdx.x] = v;
    __syncthreads();
    const long f0 = row * OL + c0;                 // flat output start
    const long a0 = (f0 + 3) & ~3L, a1 = (f0 + n) & ~3L;
    const int head = (int)(a0 - f0);
    if (threadIdx.x < head && threadIdx.x < n) y[f0 + threadIdx.x] = s[threadIdx.x];
    const long n4 = (a1 - a0) / 4;
    for (long q = threadIdx.x; q < n4; q += 256) {
      const int p = head + 4 * q;
      reinterpret_cast<float4*>(y + a0)[q] = make_float4(s[p], s[p + 1], s[p + 2], s[p + 3]);
    }
    const long tail0 = a1 > a0 ? a1 : a0;
    for (long f = tail0 + threadIdx.x; f < f0 + n; f += 256) y[f] = s[f - f0];
    __syncthreads();
  }
}

int main() {
  float *x, *y;
  cudaMalloc(&x, B * L * 4);
  cudaMalloc(&y, B * L * 4);
  cudaMemset(x, 0, B * L * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) {
        if (v == 0) copy4<<<sms * 8, 256>>>((float4*)x, (float4*)y, B * L / 4);
        if (v == 1) rows_st32<<<sms * 8, 256>>>(x, y);
        if (v == 2) rows_st128<<<sms * 8, 256>>>(x, y);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double bytes = 4.0 * (B * L + (v == 0 ? B * L : B * OL));
      if (rep) printf("%s: %.1f us  %.0f GB/s\n", v == 0 ? "copy float4" : v == 1 ? "rows st32" : "rows st128",
                      ms / 20 * 1e3, bytes / (ms / 20 * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
