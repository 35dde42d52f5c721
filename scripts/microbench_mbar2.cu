// Microbenchmark: the row-slab kernel's phase-B handshake alone (issuer / XF2p producer /
// 16 epilogue warps, rings of 3 and 4), with the library's own mbarrier helpers.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_06944_b200/csrc -I include \
//      -o scripts/microbench_mbar2.bin scripts/microbench_mbar2.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"
using namespace dt::ptx;
__device__ __forceinline__ void wait_plain(uint64_t *b, uint32_t par) { while (!mbar_try_wait(b, par)) {} }
__device__ __forceinline__ void wait_trap(uint64_t *b, uint32_t par) {
  uint32_t spins = 0;
  while (!mbar_try_wait(b, par)) if (++spins == (1u << 26)) __trap();
}
__device__ __noinline__ void wait_slow(uint64_t *b, uint32_t par) {
  uint32_t spins = 0;
  while (!mbar_try_wait(b, par))
    if (++spins == (1u << 26)) { printf("timeout %d %d\n", blockIdx.x, threadIdx.x); __trap(); }
}
__device__ __forceinline__ void wait_fastslow(uint64_t *b, uint32_t par) {
  if (mbar_try_wait(b, par)) return;
  wait_slow(b, par);
}
__device__ __noinline__ void wait_fail(uint64_t *b) {
  printf("deepthin: mbarrier wait timeout (block %d thread %d, barrier %p)\n", blockIdx.x, threadIdx.x, b);
  __trap();
}
__device__ __forceinline__ void wait_nested(uint64_t *b, uint32_t par) {
  uint32_t spins = 0;
  while (!mbar_try_wait(b, par)) if (++spins == (1u << 26)) wait_fail(b);
}
__device__ __forceinline__ void wait_unrolled(uint64_t *b, uint32_t par) {
  uint32_t spins = 0;
  for (;;) {
#pragma unroll
    for (int i = 0; i < 8; ++i) if (mbar_try_wait(b, par)) return;
    if (++spins == (1u << 23)) wait_fail(b);
  }
}
__device__ __forceinline__ void wait_clock(uint64_t *b, uint32_t par) {
  if (mbar_try_wait(b, par)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(b, par)) if (clock64() - t0 > (1ll << 34)) wait_fail(b);
}
__device__ __forceinline__ void wait_ptx(uint64_t *b, uint32_t par) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      ".reg .u32 cnt;\n\t"
      "mov.u32 cnt, 0;\n"
      "WAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@p bra WAIT_DONE;\n\t"
      "add.u32 cnt, cnt, 1;\n\t"
      "setp.lt.u32 p, cnt, 0x4000000;\n\t"
      "@p bra WAIT_LOOP;\n\t"
      "trap;\n"
      "WAIT_DONE:\n\t"
      "}" ::"r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ bool try_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(ns) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_hint(uint64_t *b, uint32_t par) {
  uint32_t spins = 0;
  while (!try_wait_hint(b, par, 1000000u)) if (++spins == 4000u) wait_fail(b);
}
template <int V>
__device__ __forceinline__ void W(uint64_t *b, uint32_t par) {
  if ((V >> 3) == 6) wait_ptx(b, par);
  else if ((V >> 3) == 7) wait_hint(b, par);
  else if ((V >> 3) == 4) wait_unrolled(b, par);
  else if ((V >> 3) == 5) wait_clock(b, par);
  else if ((V >> 3) == 1) wait_trap(b, par);
  else if ((V >> 3) == 2) wait_fastslow(b, par);
  else if ((V >> 3) == 3) wait_nested(b, par);
  else if (V & 1) wait_plain(b, par); else mbar_wait(b, par);
}
template <int V>
__device__ __forceinline__ void A(uint64_t *b) { if (V & 2) mbar_arrive_relaxed(b); else mbar_arrive(b); }
// V bit 0: plain wait loop (no spin counter / printf); bit 1: relaxed arrives; bit 2: barriers 128 B apart
template <int V>
__global__ void __launch_bounds__(768, 1) k(int iters, int BS, int ND, long long *out) {
  extern __shared__ uint8_t smem[];
  constexpr int ST = 1;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  uint64_t *b_full = bars, *b_empty = bars + 4 * ST, *d_full = bars + 8 * ST, *d_empty = bars + 12 * ST;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(&b_full[i * ST], 1); mbar_init(&b_empty[i * ST], 1);
      mbar_init(&d_full[i * ST], 1); mbar_init(&d_empty[i * ST], 16);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 1) {
    if (lane == 0) {
      int st = 0; uint32_t ph = 0;
      for (int i = 0; i < iters; ++i) {
        W<V>(&b_empty[st * ST], ph ^ 1);
        A<V>(&b_full[st * ST]);
        if (++st == BS) { st = 0; ph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      long long t0 = clock64();
      int bs = 0, db = 0; uint32_t bph = 0, dph = 0;
      for (int i = 0; i < iters; ++i) {
        W<V>(&b_full[bs * ST], bph);
        W<V>(&d_empty[db * ST], dph ^ 1);
        tc_fence_after();
        A<V>(&b_empty[bs * ST]);
        if (++bs == BS) { bs = 0; bph ^= 1; }
        A<V>(&d_full[db * ST]);
        if (++db == ND) { db = 0; dph ^= 1; }
      }
      out[0] = clock64() - t0;
    }
    __syncwarp();
  } else if (warp >= 8) {
    int db = 0; uint32_t dph = 0;
    for (int i = 0; i < iters; ++i) {
      if (V & 4) { if (lane == 0) W<V>(&d_full[db * ST], dph); __syncwarp(); }
      else W<V>(&d_full[db * ST], dph);
      tc_fence_after();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) A<V>(&d_empty[db * ST]);
      if (++db == ND) { db = 0; dph ^= 1; }
    }
  }
  __syncthreads();
}
template <int V>
void run(long long *out, int G = 1, int ITERS = 2000) {
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int nd : {1, 4}) {
    k<V><<<G, 768, 200 * 1024>>>(ITERS, 3, nd, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("V=%d (wait kind %d: 0 lib/plain 6 ptx-loop+counter 7 suspend-hint; plain %d; lane0-only epilogue polling %d) ND=%d: %.1f clk/iter (%s)\n", V, V >> 3, V & 1, (V >> 2) & 1, nd,
           (double)out[0] / ITERS, cudaGetErrorString(e));
  }
}
int main() {
  long long *out; cudaMallocManaged(&out, 8);
  run<1>(out); run<1>(out, 148); run<1>(out, 1, 16); run<1>(out, 148, 16); run<1>(out, 148, 64);
  return 0;
}
