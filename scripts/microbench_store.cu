// Microbenchmark: output-write rate of epilogue-style stores (y fp32, 4096 x 2048 = 32 MiB).
// Each CTA writes `tiles` tiles of 256 batch rows x 128 columns with 12 epilogue warps:
//   mode 0: lane = column j, 32 x STG.32 per 32-row chunk (the current epilogue pattern)
//   mode 1: per-warp smem staging [32 rows][32 cols] + TMA tensor store (box 32 x 32)
//   mode 2: per-warp-quad staging [32 rows][128 cols] + TMA tensor store (box 128 x 32)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1802_06944_b200/csrc -o scripts/mb_store scripts/microbench_store.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "sm100_ptx.cuh"

using namespace dt::ptx;

constexpr int R = 2048;
int B = 4096;

__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, const void *src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void rd(const float4 *p, size_t n, float *sink) {
  float4 a = make_float4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = p[i];
    a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
  }
  if (a.x == 1234.5f) *sink = a.y + a.z + a.w;
}

__global__ void __launch_bounds__(448, 1)
    bench(const __grid_constant__ CUtensorMap tm32, const __grid_constant__ CUtensorMap tm128,
          float *y, int mode, int tiles_per_cta, int n_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < 2) return;
  const int ew = warp - 2, wq = ew & 3, part = ew / 4;
  for (int t = 0; t < tiles_per_cta; ++t) {
    const int tile = blockIdx.x * tiles_per_cta + t;
    if (tile >= n_tiles) break;
    const int j0 = (tile % (R / 128)) * 128, b0 = (tile / (R / 128)) * 256;
    for (int c32 = part; c32 < 8; c32 += 3) {
      float v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = (float)(r + lane + t);
      const int rb = b0 + 32 * c32;
      if (mode == 0) {
        float *yp = y + (size_t)rb * R + j0 + 32 * wq + lane;
#pragma unroll
        for (int r = 0; r < 32; ++r) yp[(size_t)r * R] = v[r];
      } else if (mode == 1) {
        float *st = reinterpret_cast<float *>(smem + ew * 8192 + (c32 / 3 % 2) * 4096);
        bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) st[r * 32 + lane] = v[r];
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tm32, st, j0 + 32 * wq, rb);
          bulk_commit();
        }
      } else {
        // 4 warps (one per wq) of the same part fill one [32][128] buffer
        float *st = reinterpret_cast<float *>(smem + part * 32768 + (c32 / 3 % 2) * 16384);
        if (wq == 0 && lane == 0) bulk_wait_read<1>();
        named_bar_sync(1 + part, 128);
#pragma unroll
        for (int r = 0; r < 32; ++r) st[r * 128 + 32 * wq + lane] = v[r];
        fence_proxy_async_smem();
        named_bar_sync(1 + part, 128);
        if (wq == 0 && lane == 0) {
          tma_store_2d(&tm128, st, j0, rb);
          bulk_commit();
        }
      }
    }
  }
  if (lane == 0) bulk_wait<0>();
}

typedef CUresult (*PFN_encode)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                               const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                               CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                               CUtensorMapFloatOOBfill);

int main() {
  float *y;
  cudaMalloc(&y, (size_t)32768 * R * 4);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_encode>(fn);
  CUtensorMap tm32, tm128;
  cuuint64_t dims[2] = {R, B}, strides[1] = {R * 4};
  cuuint32_t box32[2] = {32, 32}, box128[2] = {128, 32}, es[2] = {1, 1};
  enc(&tm32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tm128, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box128, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  // L2 flush buffer
  void *flush;
  cudaMalloc(&flush, 256u << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bsz : {4096, 32768})
  for (int fl : {0, 1, 2})
  for (int mode : {0, 2}) {
    B = bsz;
    const int n_tiles = (B / 256) * (R / 128);
    cuuint64_t dims2[2] = {(cuuint64_t)R, (cuuint64_t)B};
    enc(&tm32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims2, strides, box32, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tm128, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims2, strides, box128, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int tpc : {2}) {
      const int grid = (n_tiles + tpc - 1) / tpc;
      float best = 1e9f, tot = 0.f;
      const int reps = 20;
      for (int rep = 0; rep < reps + 3; ++rep) {
        if (fl == 1) cudaMemsetAsync(flush, rep, 256u << 20);
        if (fl == 2) rd<<<1184, 512>>>((const float4 *)flush, (256u << 20) / 16, (float *)flush);
        cudaEventRecord(e0);
        bench<<<grid, 448, 100 * 1024>>>(tm32, tm128, y, mode, tpc, n_tiles);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep >= 3) { best = ms < best ? ms : best; tot += ms; }
      }
      cudaError_t e = cudaGetLastError();
      // check content
      std::vector<float> h(8);
      cudaMemcpy(h.data(), y + (size_t)37 * R + 64, 32, cudaMemcpyDeviceToHost);
      printf("B %d flush %d ", B, fl);
      printf("mode %d tiles/cta %d grid %d: %s best %.2f us avg %.2f us -> %.0f GB/s (y[37][64]=%g)\n", mode,
             tpc, grid, cudaGetErrorString(e), best * 1e3, tot / reps * 1e3,
             (double)B * R * 4 / (best * 1e-3) / 1e9, h[0]);
    }
  }
  return 0;
}
