// Microbenchmark: completion times of back-to-back regeneration-style MMA steps
// (2 x tcgen05.mma 128x160x16, no-swizzle operands, commit per step to its own mbarrier),
// cold (first use of the tensor pipe in the kernel) and with concurrent TMEM-load traffic.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_06944_b200/csrc -o scripts/mb_regen scripts/microbench_regen.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace dt::ptx;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// loads: 0 = no other activity, 1 = warps 1..3 stream tcgen05.ld of cols [320,512) meanwhile
__global__ void bench(int loads, int warm, int data, int opoff, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[4];
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  uint8_t *base = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  for (int i = threadIdx.x * 16; i < 210 * 1024; i += blockDim.x * 16) {
    uint32_t h = (uint32_t)i * 2654435761u;  // pseudo-random bf16 pairs in [-1, 1)
    uint32_t a = 0x3f80u ^ ((h >> 3) & 0x807fu), b = 0x3f00u ^ ((h >> 13) & 0x807fu);
    uint32_t w = data ? (a | (b << 16)) : 0u;
    *reinterpret_cast<uint4 *>(base + i) = make_uint4(w, w ^ 0x00010001u, w, w);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    done = 0;
  }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t a_s = smem_u32(base + opoff * 1024), b_s = smem_u32(base + (opoff + 16) * 1024);
  const uint32_t idr = idesc_bf16_f32(128, 160);
  auto step = [&](int s, uint64_t *bar) {
    for (int ks = 0; ks < 2; ++ks) {
      uint64_t ad = smem_desc(a_s + ks * 256, 128, 512, SL_NONE);
      uint64_t bd = smem_desc(b_s + ks * 256, 128, 512, SL_NONE);
      mma_bf16_ss(tbase + (uint32_t)(s % 3) * 160u, ad, bd, idr, ks > 0);
    }
    mma_commit(bar);
  };
  uint32_t ph[4] = {0, 0, 0, 0};
  if (threadIdx.x == 0) {
    if (warm) {  // warm the tensor pipe with a few steps first
      for (int r = 0; r < 4; ++r) { step(r, &bars[3]); mbar_wait(&bars[3], ph[3]); ph[3] ^= 1; }
    }
    unsigned long long t0 = gt();
    for (int s = 0; s < 3; ++s) step(s, &bars[s]);
    for (int s = 0; s < 3; ++s) {
      mbar_wait(&bars[s], ph[s]);
      out[blockIdx.x * 4 + s] = gt() - t0;
    }
    done = 1;
  } else if (loads && threadIdx.x >= 32 && threadIdx.x < 128) {  // (other threads idle)
    const int w = threadIdx.x / 32;
    uint32_t acc = 0;
    const uint32_t st_base = smem_u32(base + 40 * 1024);
    while (!done) {
      if (loads & 1) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * w) << 16) + 320u + (acc & 5u) * 32u, v);
        tmem_ld_wait();
        acc += v[0];
      }
      if (loads & 2) {  // shared-memory store stream (like the regeneration scatter)
        for (int k = 0; k < 8; ++k)
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(
                           st_base + ((threadIdx.x * 16 + k * 2048 + acc * 64) & 32767)),
                       "r"(acc));
        ++acc;
      }
    }
    if (acc == 12345) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
  unsigned long long *out;
  cudaMalloc(&out, 8192 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int opoff : {0, 172}) {
    for (int threads : {128, 448}) {
      for (int loads : {0, 3}) {
        const int grid = 148, data = 1;
        bench<<<grid, threads, 216 * 1024>>>(loads, 0, data, opoff, out);
        cudaError_t e = cudaGetLastError(); if (e == cudaSuccess) e = cudaDeviceSynchronize();
        unsigned long long h[4];
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("opoff %3d KB threads %d loads %d: %s  step completions at %.3f %.3f %.3f us\n",
               opoff, threads, loads, cudaGetErrorString(e), h[0] / 1e3, h[1] / 1e3, h[2] / 1e3);
      }
    }
  }
  return 0;
}
