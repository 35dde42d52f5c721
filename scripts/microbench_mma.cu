// Microbenchmark: raw tcgen05.mma kind::f16 issue rate, operands resident in smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_06944_b200/csrc -o /tmp/mbm scripts/microbench_mma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace dt::ptx;

// mode 0: A no-swizzle (LBO 128, SBO 7168), B SW128 (SBO 1024)
// mode 1: A SW128, B SW128
// mode 2: like mode 0 but N = 256
__global__ void bench(int mode, int ksteps, int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *base = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  // zero operands (values irrelevant)
  for (int i = threadIdx.x * 16; i < 200 * 1024; i += blockDim.x * 16)
    *reinterpret_cast<uint4 *>(base + i) = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = slot;
  if (threadIdx.x == 0) {
    const uint32_t N = mode == 2 ? 256 : 128;
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const uint32_t a_s = smem_u32(base), b_s = smem_u32(base + 120 * 1024);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (mode >= 3) {
        // regeneration-style: A (128 x 32) and B (160 x 32) no-swizzle K-major, SBO 512;
        // mode 3: D at column (r % 3) * 160, mode 4: D at column (r & 1) * 256
        const uint32_t idr = idesc_bf16_f32(128, 160);
        const uint32_t dcol = mode == 3 ? (uint32_t)(r % 3) * 160u : (uint32_t)(r & 1) * 256u;
        for (int ks = 0; ks < 2; ++ks) {
          uint64_t ad = smem_desc(a_s + ks * 256, 128, 512, SL_NONE);
          uint64_t bd = smem_desc(b_s + ks * 256, 128, 512, SL_NONE);
          mma_bf16_ss(tbase + dcol, ad, bd, idr, ks > 0);
        }
      } else {
        for (int ks = 0; ks < ksteps; ++ks) {
          uint64_t ad = mode == 1 ? smem_desc(a_s + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024, SL_SW128)
                                  : smem_desc(a_s + ks * 256, 128, 7168, SL_NONE);
          uint64_t bd = smem_desc(b_s + (ks % 4) * 32 + ((ks / 4) % 4) * 16384, 16, 1024, SL_SW128);
          mma_bf16_ss(tbase + (r & 1) * 256, ad, bd, idesc, ks > 0);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
  long long *out;
  cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int mode : {0, 1, 2, 3, 4}) {
    for (int grid : {1, 148}) {
      const int ks = mode >= 3 ? 2 : 28, reps = 200;
      bench<<<grid, 128, 220 * 1024>>>(mode, ks, reps, out);
      cudaError_t e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      double per_mma = (double)c / (ks * reps);
      if (mode >= 3) {
        printf("mode %d grid %3d: %s  %.1f cycles per regen step (2 MMAs 128x160x16 + commit/wait)\n",
               mode, grid, cudaGetErrorString(e), (double)c / reps);
        continue;
      }
      double N = mode == 2 ? 256 : 128;
      printf("mode %d grid %3d: %s  %.1f cycles/MMA (floor %.0f), %.0f MAC/cycle/SM\n", mode, grid,
             cudaGetErrorString(e), per_mma, 128 * N / 256, 128 * N * 16 / per_mma);
    }
  }
  return 0;
}
