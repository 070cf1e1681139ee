// Microbenchmark: FP32 FMA issue rates on sm_100a (FFMA reg/reg, FFMA with
// constant-bank operand, packed FFMA2).  Prints achieved TFLOP/s per variant.
#include <cstdio>
#include <cuda_runtime.h>

struct C8 { float f[8]; };

__global__ void k_ffma_reg(float* out, float a, float b, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  float m = a, n = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], m, n);
    m += 1e-7f;  // keep operands live in registers
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma_const(float* out, const C8 c, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], c.f[(r + i) & 7], x[(i + 1) & 7]);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long x[8];
  for (int i = 0; i < 8; ++i) {
    float2 v = make_float2(threadIdx.x * 0.001f + i, i * 0.5f);
    x[i] = *reinterpret_cast<unsigned long long*>(&v);
  }
  float2 mv = make_float2(a, a), nv = make_float2(b, b);
  unsigned long long m = *reinterpret_cast<unsigned long long*>(&mv);
  unsigned long long n = *reinterpret_cast<unsigned long long*>(&nv);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = ffma2(x[i], m, n);
    m += 1;
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&x[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, max clock %d MHz\n", sms, clk / 1000);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = sms * 8, threads = 256;
  C8 c; for (int i = 0; i < 8; ++i) c.f[i] = 0.999f + i * 1e-4f;
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k_ffma_reg<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
      if (v == 1) k_ffma_const<<<blocks, threads>>>(out, c, iters);
      if (v == 2) k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * blocks * threads * (double)iters * 16 * 8 * (v == 2 ? 2 : 1);
      if (rep == 2) printf("%s: %.3f ms  %.1f TFLOP/s\n", v == 0 ? "FFMA reg" : v == 1 ? "FFMA const" : "FFMA2", ms, fl / ms / 1e9);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
