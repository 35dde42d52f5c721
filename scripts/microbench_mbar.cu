// Microbenchmark: mbarrier ping-pong between an issuer thread and R responder warps through
// rings of depth D (the d_full / d_empty handshake of the row kernels' phase B, nothing else).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbar scripts/microbench_mbar.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_arrive(uint64_t *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t *b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ bool test_wait(uint64_t *b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok;
}
template <int MODE>
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
  if (MODE == 0) while (!try_wait(b, par)) {}
  else while (!test_wait(b, par)) {}
}
__device__ __forceinline__ void tcf_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tcf_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
template <int MODE>
__global__ void k(int D, int R, int iters, int spinners, long long *out, int fences) {
  __shared__ uint64_t full[8], empty[8], never;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], R); }
    mbar_init(&never, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      long long t0 = clock64();
      int s = 0; uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
        wait<MODE>(&empty[s], ph ^ 1);
        if (fences & 1) tcf_after();
        mbar_arrive(&full[s]);
        if (++s == D) { s = 0; ph ^= 1; }
      }
      // drain
      for (int j = 0; j < D; ++j) { wait<MODE>(&empty[s], ph ^ 1); if (++s == D) { s = 0; ph ^= 1; } }
      out[0] = clock64() - t0;
      mbar_arrive(&never);
    }
  } else if (warp <= R) {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait<MODE>(&full[s], ph);
      if (fences & 2) tcf_after();
      if (fences & 4) tcf_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == D) { s = 0; ph ^= 1; }
    }
  } else if (warp <= R + spinners) {
    wait<MODE>(&never, 0);  // idle warps parked on a barrier (like producers with a full ring)
  }
}
int main() {
  long long *out; cudaMallocManaged(&out, 8);
  const int iters = 2000;
  for (int fences : {0, 1, 2, 4, 7})
    for (int R : {1, 16})
        for (int D : {1, 4}) {
          const int sp = 6, threads = 32 * (1 + R + sp);
          k<0><<<1, threads>>>(D, R, iters, sp, out, fences);
          cudaError_t e = cudaDeviceSynchronize();
          printf("fences=%d R=%2d D=%d: %.1f clk/iter (%s)\n", fences, R, D, (double)out[0] / iters, cudaGetErrorString(e));
        }
  return 0;
}
