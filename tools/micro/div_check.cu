// Exhaustive check of the reciprocal-plus-FMA-correction division used by the
// pooling average (pool_tma.cu div_by_k) against IEEE division (__fdiv_rn):
// every float32 significand, several exponents, signs, k = 2..300.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float div_by_k(float a, float k, float r) {
  const float q = a * r;
  const float e = fmaf(-k, q, a);
  const float q2 = fmaf(e, r, q);
  return (fabsf(a) < 1e-30f || !(fabsf(a) < 3.0e38f)) ? __fdiv_rn(a, k) : q2;
}

__global__ void check(int k, int exp_lo, int exp_hi, unsigned long long* bad) {
  const float fk = (float)k;
  const float r = 1.0f / fk;
  unsigned long long nbad = 0;
  for (unsigned m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x) {
    for (int e = exp_lo; e <= exp_hi; ++e) {
      for (int sgn = 0; sgn < 2; ++sgn) {
        const unsigned bits = (sgn << 31) | ((unsigned)(e + 127) << 23) | m;
        const float a = __uint_as_float(bits);
        if (__float_as_uint(div_by_k(a, fk, r)) != __float_as_uint(__fdiv_rn(a, fk))) ++nbad;
      }
    }
  }
  atomicAdd(bad, nbad);
}

int main() {
  unsigned long long* bad;
  cudaMallocManaged(&bad, 8);
  unsigned long long total = 0;
  for (int k = 2; k <= 300; ++k) {
    *bad = 0;
    check<<<148 * 8, 256>>>(k, -99, 127, bad);  // every normal exponent with |a| >= 2^-99
    cudaDeviceSynchronize();
    if (*bad) printf("k=%d mismatches=%llu\n", k, *bad);
    total += *bad;
  }
  printf("total mismatches over k=2..300, all significands, exponents -99..127: %llu (%s)\n", total,
         cudaGetErrorString(cudaGetLastError()));
}
