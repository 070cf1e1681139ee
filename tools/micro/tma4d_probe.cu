// Which 4-D TMA configurations are legal on sm_100a? ./tma4d_probe <perm> <swizzle>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  unsigned char* base = sm + ((1024 - (su32(sm) & 1023)) & 1023);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(16384) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(su32(base)), "l"((uint64_t)&m), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(su32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    }
    out[0] = ((float*)base)[1];
  }
}

int main(int argc, char** argv) {
  const int perm = atoi(argv[1]), swz = atoi(argv[2]);
  const int W = 112, H = 112, C = 64, N = 2;
  float* x; cudaMalloc(&x, (size_t)W * H * C * N * 4); cudaMemset(x, 0, (size_t)W * H * C * N * 4);
  float* out; cudaMalloc(&out, 16);
  CUtensorMap m;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  if (perm) {  // (w, c, h, n)
    cuuint64_t d[4] = {W, C, H, N}; cuuint64_t s[3] = {(cuuint64_t)H * W * 4, (cuuint64_t)W * 4, (cuuint64_t)C * H * W * 4};
    cuuint32_t b[4] = {16, 32, 8, 1};
    for (int i = 0; i < 4; ++i) { dims[i] = d[i]; box[i] = b[i]; } for (int i = 0; i < 3; ++i) strides[i] = s[i];
  } else {     // (w, h, c, n)
    cuuint64_t d[4] = {W, H, C, N}; cuuint64_t s[3] = {(cuuint64_t)W * 4, (cuuint64_t)H * W * 4, (cuuint64_t)C * H * W * 4};
    cuuint32_t b[4] = {16, 8, 32, 1};
    for (int i = 0; i < 4; ++i) { dims[i] = d[i]; box[i] = b[i]; } for (int i = 0; i < 3; ++i) strides[i] = s[i];
  }
  CUtensorMapSwizzle sw = swz == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("perm %d swz %d: encode failed %d\n", perm, swz, (int)r); return 0; }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const int neg = argc > 3 ? atoi(argv[3]) : 1;
  const int c0 = argc > 4 ? atoi(argv[4]) : 0;
  k<<<1, 32, 32768>>>(m, (neg & 1) ? -1 : c0, 0, (neg & 2) ? -1 : 0, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("perm %d swz %d neg %d c0 %d: %s\n", perm, swz, neg, c0, cudaGetErrorString(e));
  return 0;
}
