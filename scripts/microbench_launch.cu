// Kernel-to-kernel time of back-to-back launches: empty kernels of various grid / smem sizes,
// with and without griddepcontrol.launch_dependents, in a CUDA graph and as plain launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_launch scripts/microbench_launch.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int *p, int trig) {
  if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p && threadIdx.x == 9999) *p = 1;
}
__global__ void k_smem(int *p) {
  __shared__ float s[5120];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && s[(threadIdx.x + 1) % blockDim.x] == -1.f) *p = 1;
}

int main() {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct Cfg { int grid, block, kind, trig; } cfgs[] = {
      {1, 32, 0, 0}, {148, 256, 0, 0}, {264, 256, 0, 0}, {264, 256, 0, 1}, {264, 256, 1, 0},
      {1184, 256, 0, 0}};
  for (auto c : cfgs) {
    for (int graph : {0, 1}) {
      auto launch = [&]() {
        if (c.kind == 0) k_empty<<<c.grid, c.block, 0, st>>>(nullptr, c.trig);
        else k_smem<<<c.grid, c.block, 0, st>>>(nullptr);
      };
      cudaGraphExec_t ge = nullptr;
      const int N = 100;
      if (graph) {
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < N; ++i) launch();
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
      } else {
        for (int i = 0; i < N; ++i) launch();
      }
      cudaStreamSynchronize(st);
      cudaEventRecord(e0, st);
      if (graph) cudaGraphLaunch(ge, st); else for (int i = 0; i < N; ++i) launch();
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %4d block %3d %s%s %s: %.2f us/launch\n", c.grid, c.block, c.kind ? "smem20K" : "empty",
             c.trig ? "+trigger" : "", graph ? "graph" : "plain", ms * 1e3 / N);
    }
  }
  return 0;
}
