// In-CTA W-block generation (wgen_block) timed in isolation: 144 CTAs x 256 threads, config-2
// geometry, with and without two extra "spinning" warps polling an mbarrier (like the GEMM's
// producer / MMA warps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -I paper_1802_06944_b200/csrc -o scripts/mb_wgen scripts/microbench_wgen.cu
#include "../paper_1802_06944_b200/csrc/k_tc_gemm.cu"

namespace dt {
void set_error(const std::string &) {}
int check_launch(const char *) { return 0; }
int launch_row_softmax(int64_t, int64_t, void *, int, cudaStream_t) { return 0; }
int launch_pack_x(int64_t, int64_t, int64_t, const void *, int, void *, cudaStream_t) { return 0; }
int encode_tensor_map_2d(CUtensorMap *, int, void *, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t,
                         bool) { return 0; }
void profile_next(cudaEvent_t *b, cudaEvent_t *a) { *b = *a = nullptr; }
namespace {
__global__ void __launch_bounds__(320, 1) k_wgen_only(const GemmParams p, int spin, unsigned long long *t) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int warp = threadIdx.x / 32;
  unsigned long long t0 = clock64();
  if (warp >= 2) {
    if (spin != 2) wgen_block<float>(p, (blockIdx.x % 16) * GM, smem, threadIdx.x - 64);
    named_bar_sync(1, 256);
    if (threadIdx.x == 64) { mbar_arrive(&bar); t[blockIdx.x] = clock64() - t0; }
  } else if (spin && (threadIdx.x % 32) == 0) {
    mbar_wait(&bar, 0);
  }
  __syncthreads();
}
}  // namespace
}  // namespace dt

int main() {
  const int q = 440, r_dim = 2048, rank = 24, n = 320, m = 2816;
  float *xf, *wf;
  cudaMalloc(&xf, m * rank * 4);
  cudaMalloc(&wf, rank * n * 4);
  cudaMemset(xf, 0, m * rank * 4);
  cudaMemset(wf, 0, rank * n * 4);
  unsigned long long *t;
  cudaMalloc(&t, 4096 * 8);
  dt::GemmParams p{};
  p.KB = 7;
  p.rg.q = q; p.rg.r_dim = r_dim; p.rg.ldw = q; p.rg.rank = rank; p.rg.n = n; p.rg.a_rows = 0;
  p.rg.f_dtype = DT_F32; p.rg.xf = xf; p.rg.wf = wf;
  p.off_fs = 144 * 1024;
  cudaFuncSetAttribute(dt::k_wgen_only, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int variant : {0, 1, 2, 0, 1, 2}) {
    const int spin = variant == 2 ? 2 : 0;
    p.rg.r_dim = variant ? 0 : r_dim;  // 1: r_dim 0 -> only the zero-fill phase runs
    cudaEventRecord(e0);
    dt::k_wgen_only<<<144, 320, 220 * 1024>>>(p, spin, t);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[144];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
    printf("variant %d spin %d: %s kernel %.2f us, wgen max %llu cycles\n", variant, spin,
           cudaGetErrorString(cudaGetLastError()), ms * 1e3, mx);
  }
  return 0;
}
