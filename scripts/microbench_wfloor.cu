// Floor for the bench's output traffic: back-to-back launches that only write y (4096 x 2048
// fp32 = 32 MiB) into R rotating buffers (R * 32 MiB > 2 x L2), timed like bench.py (events
// around K steps). Also: the same with a 3.5 MiB x read per step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_wfloor scripts/microbench_wfloor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) wr(float4 *y, size_t n4, const float4 *x, size_t nx4) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nx4; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = x[i];
    acc.x += v.x;
  }
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_float4(acc.x + i, 1.f, 2.f, 3.f);
}

int main() {
  const size_t ybytes = 4096ull * 2048 * 4, xbytes = 4096ull * 448 * 2;
  const int R = 8;
  float4 *ys[R], *xs[R];
  for (int r = 0; r < R; ++r) { cudaMalloc(&ys[r], ybytes); cudaMalloc(&xs[r], xbytes); }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int withx : {0, 1})
    for (int grid : {148, 296, 592, 1184}) {
      for (int w = 0; w < 20; ++w) wr<<<grid, 512>>>(ys[w % R], ybytes / 16, xs[w % R], withx ? xbytes / 16 : 0);
      cudaEventRecord(e0);
      const int K = 50;
      for (int k = 0; k < K; ++k) wr<<<grid, 512>>>(ys[k % R], ybytes / 16, xs[k % R], withx ? xbytes / 16 : 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("x-read %d grid %4d: %.2f us/step  (%.0f GB/s y-write)\n", withx, grid, ms * 1e3 / K,
             ybytes / (ms * 1e-3 / K) / 1e9);
    }
  // single launch, not rotating, warm
  for (int k = 0; k < 5; ++k) wr<<<592, 512>>>(ys[0], ybytes / 16, xs[0], 0);
  cudaEventRecord(e0);
  for (int k = 0; k < 50; ++k) wr<<<592, 512>>>(ys[0], ybytes / 16, xs[0], 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("same y buffer every step (L2-resident): %.2f us/step\n", ms * 1e3 / 50);
  return 0;
}
