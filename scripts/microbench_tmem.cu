// Microbenchmark: tcgen05.ld throughput/latency on B200 for the epilogue/regen read-back.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld_x32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// mode 0: ld x32 + wait each; mode 1: 2 x ld x32 then wait; mode 2: 4 x ld then wait
__global__ void bench(int mode, int iters, long long *out, uint32_t *sink) {
  __shared__ uint32_t slot;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = slot + ((uint32_t)(32 * (warp & 3)) << 16);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t v[32], w[32], x[32], y[32];
    uint32_t col = (it * 128) & 511;
    if (mode == 0) {
      for (int g = 0; g < 4; ++g) {
        ld_x32(base + col + g * 32, v);
        ld_wait();
        #pragma unroll
        for (int k = 0; k < 32; ++k) acc += v[k];
      }
    } else if (mode == 1) {
      ld_x32(base + col, v); ld_x32(base + col + 32, w); ld_wait();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k] ^ w[k];
      ld_x32(base + col + 64, v); ld_x32(base + col + 96, w); ld_wait();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k] ^ w[k];
    } else {
      ld_x32(base + col, v); ld_x32(base + col + 32, w); ld_x32(base + col + 64, x);
      ld_x32(base + col + 96, y); ld_wait();
      #pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k] ^ w[k] ^ x[k] ^ y[k];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  long long *out;
  uint32_t *sink;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&sink, 1024 * 1024 * 4);
  const int iters = 1000;
  for (int warps : {1, 4, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      bench<<<1, 32 * warps>>>(mode, iters, out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      // bytes read per iteration per CTA: warps * 4 groups * 32 lanes * 32 cols * 4 B
      double bytes = (double)warps * 4 * 32 * 32 * 4 * iters;
      printf("warps %d mode %d: %s %.1f cycles/iter (4 x x32 per warp), %.1f B/cycle/SM\n", warps,
             mode, cudaGetErrorString(e), (double)c / iters, bytes / c);
    }
  }
  return 0;
}
