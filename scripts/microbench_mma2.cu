// MMA issue-rate microbenchmark: single-CTA (M=128) vs CTA-pair (cta_group::2, M=256) kind::f16
// with N=256, both operands 128B-swizzled K-major (the GEMM's layout), operands resident in smem.
// Times `reps` back-to-back k-blocks of 4 MMAs each with commits to a stage barrier (like the
// GEMM main loop) and reports cycles per MMA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_06944_b200/csrc -o scripts/mb_mma2 scripts/microbench_mma2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace dt::ptx;

template <bool PAIR>
__global__ void __launch_bounds__(128, 1) bench(int reps, int commit_every, int data, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x * 16; i < 200 * 1024; i += blockDim.x * 16) {
    uint32_t h = (uint32_t)i * 2654435761u;
    uint32_t a = 0x3f80u ^ ((h >> 3) & 0x807fu), b = 0x3f00u ^ ((h >> 13) & 0x807fu);
    uint32_t w = data ? (a | (b << 16)) : 0u;
    *reinterpret_cast<uint4 *>(smem + i) = make_uint4(w, w ^ 0x00010001u, w * 3u, w);
  }
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) { if (PAIR) tmem_alloc_pair(&slot, 512); else tmem_alloc(&slot, 512); }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  tc_fence_after();
  const uint32_t tbase = slot;
  const bool issuer = threadIdx.x == 0 && (!PAIR || cluster_ctarank() == 0);
  if (issuer) {
    const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, 256);
    const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 112 * 1024);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      const uint32_t a = a0 + (uint32_t)(r % 7) * 16384u, b = b0 + (uint32_t)(r % 4) * 16384u;
      for (int k = 0; k < 4; ++k) {
        if (PAIR)
          mma_bf16_ss_pair(tbase + (r & 1) * 256, smem_desc(a + k * 32, 16, 1024, SL_SW128),
                           smem_desc(b + k * 32, 16, 1024, SL_SW128), idesc, (r | k) != 0);
        else
          mma_bf16_ss(tbase + (r & 1) * 256, smem_desc(a + k * 32, 16, 1024, SL_SW128),
                      smem_desc(b + k * 32, 16, 1024, SL_SW128), idesc, (r | k) != 0);
      }
      if (PAIR) mma_commit_pair(&bar[r & 7]); else mma_commit(&bar[r & 7]);
      if (commit_every && (r % commit_every) == commit_every - 1) {
        // drain: wait for the last commit
        mbar_wait(&bar[r & 7], (uint32_t)((r >> 3) & 1));
      }
    }
    if (PAIR) mma_commit_pair(&bar[7]); else mma_commit(&bar[7]);
    (void)ph;
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tbase, 512); else tmem_dealloc(tbase, 512);
  }
}

int main() {
  long long *out;
  cudaMalloc(&out, 1024 * 8);
  cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  const int reps = 400;
  for (int data : {0, 1})
  for (int pair : {0, 1}) {
    for (int grid : {148}) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = 210 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaError_t e;
      if (pair) e = cudaLaunchKernelEx(&cfg, bench<true>, reps, 0, data, out);
      else e = cudaLaunchKernelEx(&cfg, bench<false>, reps, 0, data, out);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      // issue time only (no final wait) -> use a second launch that waits at the end
      printf("data %d %s grid %3d: %s  issue %.1f cycles per MMA (per SM: 128x256x16)\n", data, pair ? "pair  " : "single",
             grid, cudaGetErrorString(e), (double)c / (reps * 4));
    }
  }
  return 0;
}
