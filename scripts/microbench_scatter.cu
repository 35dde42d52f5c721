// Microbenchmark: the W-block regeneration scatter (scatter32<2>) in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_scatter scripts/microbench_scatter.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t w_off(uint32_t jj, uint32_t i, uint32_t sbo) {
  return (jj >> 3) * sbo + (i >> 3) * 128u + (jj & 7u) * 16u + (i & 7u) * 2u;
}
__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ void scatter32(const uint32_t (&v)[32], uint32_t w_s, uint32_t sbo,
                                          int jj, int i, int q, int cvalid, int jrows) {
  uint32_t addr = w_s + w_off(jj, i, sbo);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t ok = (8 * t < cvalid) & ((uint32_t)jj < (uint32_t)jrows);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"r"(addr),
        "r"(pack_bf16(v[8 * t], v[8 * t + 1])), "r"(pack_bf16(v[8 * t + 2], v[8 * t + 3])),
        "r"(pack_bf16(v[8 * t + 4], v[8 * t + 5])), "r"(pack_bf16(v[8 * t + 6], v[8 * t + 7])),
        "r"(ok));
    i += 8;
    addr += 128u;
    if (i >= q) { i -= q; ++jj; addr = w_s + w_off(jj, i, sbo); }
  }
}

__global__ void bench(int q, int n, int groups, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t w_s = smem_u32(smem);
  const uint32_t sbo = 7 * 8 * 128;
  const int L = threadIdx.x % 128;
  const int part = threadIdx.x / 128;
  const int f0 = L * n + 32 * part;
  int jj = f0 / q, i = f0 % q;
  uint32_t v[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) v[t] = __float_as_uint(0.001f * (t + L));
  __syncthreads();
  long long t0 = clock64();
  for (int g = 0; g < groups; ++g) {
    scatter32(v, w_s, sbo, jj, i, q, 32, 128);
    i += 64;
    while (i >= q) { i -= q; ++jj; }
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] += 1;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long *out;
  cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int threads : {128, 256, 384}) {
    for (int grid : {1, 148}) {
      const int groups = 10;
      bench<<<grid, threads, 120 * 1024>>>(440, 320, groups, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("threads %d grid %d: %s %.1f cycles/group\n", threads, grid, cudaGetErrorString(e),
             (double)c / groups);
    }
  }
  return 0;
}
