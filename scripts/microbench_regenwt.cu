// Phase-1 (W^T regeneration) kernel timing in isolation: graph-replayed back-to-back launches
// at BASELINE config-2 geometry. Includes the library translation unit to reach the kernel.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include -I paper_1802_06944_b200/csrc -o scripts/mb_regenwt scripts/microbench_regenwt.cu
#include "../paper_1802_06944_b200/csrc/k_tc_gemm.cu"

namespace dt {
void set_error(const std::string &) {}
int check_launch(const char *) { return 0; }
int launch_row_softmax(int64_t, int64_t, void *, int, cudaStream_t) { return 0; }
int launch_pack_x(int64_t, int64_t, int64_t, const void *, int, void *, cudaStream_t) { return 0; }
int encode_tensor_map_2d(CUtensorMap *, int, void *, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t,
                         bool) { return 0; }
}  // namespace dt

namespace dt { namespace {
template <typename FT>
__global__ void __launch_bounds__(256) k_var(int variant, int64_t q, int64_t r_dim, int rank, int n,
                                                  int a_rows, int64_t ldw, const FT *xf,
                                                  const FT *wf, __nv_bfloat16 *wt) {
  __shared__ __align__(16) float xt[RG_K][RG_R + 4];  // +4: the transposing stores are 4-way, not 32-way, conflicted
  __shared__ __align__(16) float ws[RG_K][RG_C];
  const int tid = threadIdx.x, lane = tid % 32, wrp = tid / 32;
  const int a0 = blockIdx.x * RG_R, c0 = blockIdx.y * RG_C;
  float acc[RG_E][4];
#pragma unroll
  for (int e = 0; e < RG_E; ++e)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[e][c] = 0.f;
  if (!(variant & 1)) for (int k0 = 0; k0 < rank; k0 += RG_K) {
    const int kc = min(RG_K, rank - k0);
    // every load of the chunk issued before the first shared-memory store (one latency)
    constexpr int NX = RG_R * RG_K / 256, NW = RG_K * RG_C / 256;
    float xv[NX], wv[NW];
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u, r = e / RG_K, k = e % RG_K;
      xv[u] = (variant & 4) ? (float)e : (a0 + r < a_rows && k < kc) ? ldf(xf + (int64_t)(a0 + r) * rank + k0 + k) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u, k = e / RG_C, c = e % RG_C;
      wv[u] = (variant & 4) ? (float)e : (k < kc && c0 + c < n) ? ldf(wf + (int64_t)(k0 + k) * n + c0 + c) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u;
      xt[e % RG_K][e / RG_K] = xv[u];
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u;
      ws[e / RG_C][e % RG_C] = wv[u];
    }
    __syncthreads();
    // 8 ranks per unrolled group (the staged chunk is zero-padded to a multiple of 8): the
    // shared loads of later ranks issue ahead of the FMAs of earlier ones
    if (!(variant & 16)) for (int k8 = 0; k8 < kc; k8 += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = k8 + kk;
        const float4 w4 = *reinterpret_cast<const float4 *>(&ws[k][4 * lane]);
        const float4 x4 = *reinterpret_cast<const float4 *>(&xt[k][RG_E * wrp]);
        const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
        const float xk[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
        for (int e = 0; e < RG_E; ++e)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[e][c] = fmaf(xk[e], wk[c], acc[e][c]);
      }
    }
    __syncthreads();
  }
  if (variant & 2) { if (acc[0][0] == 1234.f) wt[0] = __float2bfloat16(1.f); return; }
  const int64_t total = q * r_dim;
  const bool flat = ldw == q && (n & 3) == 0;  // W^T == I.ravel(): 8-byte stores
  const int cc = c0 + 4 * lane;
  if (cc >= n) return;
#pragma unroll
  for (int e = 0; e < RG_E; ++e) {
    const int a = a0 + RG_E * wrp + e;
    if (a >= a_rows) continue;
    const int64_t f0 = (int64_t)a * n + cc;
    if (flat && f0 + 4 <= total) {
      __nv_bfloat162 v0 = __floats2bfloat162_rn(acc[e][0], acc[e][1]);
      __nv_bfloat162 v1 = __floats2bfloat162_rn(acc[e][2], acc[e][3]);
      *reinterpret_cast<uint2 *>(wt + f0) =
          make_uint2(*reinterpret_cast<uint32_t *>(&v0), *reinterpret_cast<uint32_t *>(&v1));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t f = f0 + c;
        if (cc + c < n && f < total) {
          const int64_t j = f / q, i = f - j * q;
          wt[j * ldw + i] = __float2bfloat16_rn(acc[e][c]);
        }
      }
    }
  }
}


}}

int main() {
  const int64_t q = 440, r_dim = 2048, rank = 24, n = 320, m = 2816;
  float *xf, *wf;
  __nv_bfloat16 *wt;
  cudaMalloc(&xf, m * rank * 4);
  cudaMalloc(&wf, rank * n * 4);
  cudaMalloc(&wt, r_dim * q * 2);
  cudaMemset(xf, 0, m * rank * 4);
  cudaMemset(wf, 0, rank * n * 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int64_t a_rows = (q * r_dim + n - 1) / n;
  const dim3 grid((unsigned)((a_rows + dt::RG_R - 1) / dt::RG_R), (unsigned)((n + dt::RG_C - 1) / dt::RG_C));
  const int N = 100;
  for (int variant : {0, 6, 22, 3}) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i)
    dt::k_var<float><<<grid, 256, 0, st>>>(variant, q, r_dim, (int)rank, (int)n, (int)a_rows, q, xf, wf, wt);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEventRecord(e0, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("variant %d (1 no-loop, 2 no-store, 4 no-load, 16 no-fma) grid %ux%u: %s %.2f us/launch\n", variant, grid.x, grid.y, cudaGetErrorString(cudaGetLastError()),
         ms * 1e3 / N);
  }
  return 0;
}
