// LSTM cell of BASELINE config 4 (speech-RNN-shaped model): the elementwise step that follows
// the eight DeepThin-compressed gate contractions. Not in the reference (SURVEY.md §8(a) a8:
// LSTM gates are "not in the reference"); its math is the standard cell, gate order i, f, g, o:
//   i = sigmoid(gx_i + gh_i), f = sigmoid(gx_f + gh_f), g = tanh(gx_g + gh_g),
//   o = sigmoid(gx_o + gh_o), c' = f c + i g, h' = o tanh(c').
// gx: input projections (bf16, batched over all time steps by the tensor-core path, biases
// included); gh: recurrent projections (fp32, this step). c is updated in place (fp32); h' is
// written in fp32 (next step's recurrent input) and bf16 (the sequence output).
#include <cuda_bf16.h>

#include "dt_internal.h"

namespace dt {
namespace {

__device__ __forceinline__ float sigm(float z) { return 1.f / (1.f + expf(-z)); }

struct CellArgs {
  const __nv_bfloat16 *gx[4];
  const float *gh[4];
  int64_t ld_gx;  // row stride of gx (elements)
};

__global__ void __launch_bounds__(256) k_lstm_cell(int64_t batch, int64_t hidden, CellArgs a,
                                                    float *c, float *h32, __nv_bfloat16 *h16) {
  const int64_t tot = batch * hidden;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / hidden, j = e - b * hidden, gxo = b * a.ld_gx + j;
    const float zi = __bfloat162float(a.gx[0][gxo]) + a.gh[0][e];
    const float zf = __bfloat162float(a.gx[1][gxo]) + a.gh[1][e];
    const float zg = __bfloat162float(a.gx[2][gxo]) + a.gh[2][e];
    const float zo = __bfloat162float(a.gx[3][gxo]) + a.gh[3][e];
    const float cn = sigm(zf) * c[e] + sigm(zi) * tanhf(zg);
    const float hn = sigm(zo) * tanhf(cn);
    c[e] = cn;
    if (h32) h32[e] = hn;
    if (h16) h16[e] = __float2bfloat16_rn(hn);
  }
}

}  // namespace

int launch_lstm_cell(int64_t batch, int64_t hidden, const void *const *gx, int64_t ld_gx,
                     const float *const *gh, float *c, float *h32, void *h16, cudaStream_t st) {
  if (batch == 0 || hidden == 0) return DT_OK;
  CellArgs a;
  for (int g = 0; g < 4; ++g) {
    a.gx[g] = reinterpret_cast<const __nv_bfloat16 *>(gx[g]);
    a.gh[g] = gh[g];
  }
  a.ld_gx = ld_gx;
  const int64_t tot = batch * hidden;
  const unsigned grid = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  k_lstm_cell<<<grid, 256, 0, st>>>(batch, hidden, a, c, h32,
                                     reinterpret_cast<__nv_bfloat16 *>(h16));
  return check_launch("lstm_cell");
}

}  // namespace dt

// =============================================================================================
// The four recurrent gate contractions of one LSTM step (config 4: h (batch x H, fp32) through
// four reuse-geometry DeepThin layers H -> H), exact fp32 on the CUDA cores, factored exactly
// like the reuse path (kernel.py:1-16):
//   k_gates_p:  P_g[b, seg*R + k] = sum_t h[b, seg*n + t] * wf_g[k, t]        (grid: s x 4)
//   k_gates_y:  gh_g[b, j] = sum_kk P_g[b, kk] * xf_g[j*s*R + kk] + bias_g[j]   (grid: H/64 x 4)
// (xf_g viewed (H x s*R) row-major is XF2). Fixed summation order: bitwise reproducible.
// =============================================================================================
namespace dt {
namespace {

constexpr int kGB = 64;  // batch rows per pass of k_gates_y
constexpr int kPB = 16;  // batch rows per CTA of k_gates_p

struct GateArgs {
  const float *xf[4], *wf[4], *bias[4];
  float *gh[4];
};

// Stage `rows` x `cols` fp32 (cols % 4 == 0, row pitch `ld` floats) from global into shared
// memory (row pitch `sp` floats): 8 float4 loads in flight per thread before the stores.
__device__ __forceinline__ void stage_rows(float *dst, int sp, const float *src, int64_t ld, int rows,
                                           int cols) {
  const int c4 = cols / 4, n4 = rows * c4;
  for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n4) v[u] = __ldg(reinterpret_cast<const float4 *>(src + (int64_t)(i / c4) * ld) + i % c4);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n4) {
        float *d = dst + (i / c4) * sp + 4 * (i % c4);
        d[0] = v[u].x; d[1] = v[u].y; d[2] = v[u].z; d[3] = v[u].w;
      }
    }
  }
}

// one CTA per (segment, gate, 16-row block): h[rows, seg] and wf_g in shared memory; each
// thread two outputs, four interleaved partial sums (fixed order)
__global__ void __launch_bounds__(256) k_gates_p(int64_t batch, int H, int n, int R, const float *h,
                                                 GateArgs a, float *P) {
  extern __shared__ float sm[];
  const int seg = blockIdx.x, g = blockIdx.y, s = H / n, K2 = s * R;
  const int64_t b0 = (int64_t)blockIdx.z * kPB;
  const int nb = (int)(batch - b0 < kPB ? batch - b0 : kPB);
  const int npad = n + 1;  // conflict-free row reads across k
  float *hs = sm, *ws = sm + kPB * npad;
  const float *wfg = g == 0 ? a.wf[0] : g == 1 ? a.wf[1] : g == 2 ? a.wf[2] : a.wf[3];
  stage_rows(ws, npad, wfg, n, R, n);
  stage_rows(hs, npad, h + b0 * H + seg * n, H, nb, n);
  __syncthreads();
  for (int o = threadIdx.x; o < nb * R; o += blockDim.x) {
    const int b = o / R, k = o % R;
    const float *hr = hs + b * npad, *wr = ws + k * npad;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < n; t += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fmaf(hr[t + u], wr[t + u], acc[u]);
    }
    P[((int64_t)g * batch + b0 + b) * K2 + seg * R + k] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
}

// one CTA per (64-column block, gate); each thread 4 rows x 4 columns of the block
__global__ void __launch_bounds__(256) k_gates_y(int64_t batch, int H, int K2, const float *P,
                                                 GateArgs a) {
  extern __shared__ float sm[];
  const int j0 = blockIdx.x * 64, g = blockIdx.y;
  const int kp = K2 + 4;  // row pitch (16-byte aligned, staggered banks)
  float *ps = sm, *xs = sm + kGB * kp;
  const int nj = min(64, H - j0);
  const float *xfg = g == 0 ? a.xf[0] : g == 1 ? a.xf[1] : g == 2 ? a.xf[2] : a.xf[3];
  const float *bg = g == 0 ? a.bias[0] : g == 1 ? a.bias[1] : g == 2 ? a.bias[2] : a.bias[3];
  float *ghg = g == 0 ? a.gh[0] : g == 1 ? a.gh[1] : g == 2 ? a.gh[2] : a.gh[3];
  stage_rows(xs, kp, xfg + (int64_t)j0 * K2, K2, nj, K2);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;  // rows tr*4.., cols tc + 16*c
  for (int64_t b0 = 0; b0 < batch; b0 += kGB) {
    const int nb = (int)(batch - b0 < kGB ? batch - b0 : kGB);
    __syncthreads();
    stage_rows(ps, kp, P + ((int64_t)g * batch + b0) * K2, K2, nb, K2);
    __syncthreads();
    float acc[4][4] = {};
    for (int kk = 0; kk < K2; kk += 4) {
      float4 pv[4], xv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) pv[r] = *reinterpret_cast<const float4 *>(ps + (tr * 4 + r) * kp + kk);
#pragma unroll
      for (int c = 0; c < 4; ++c) xv[c] = *reinterpret_cast<const float4 *>(xs + (tc + 16 * c) * kp + kk);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[r][c] = fmaf(pv[r].x, xv[c].x, acc[r][c]);
          acc[r][c] = fmaf(pv[r].y, xv[c].y, acc[r][c]);
          acc[r][c] = fmaf(pv[r].z, xv[c].z, acc[r][c]);
          acc[r][c] = fmaf(pv[r].w, xv[c].w, acc[r][c]);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int b = tr * 4 + r;
      if (b >= nb) continue;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = tc + 16 * c;
        if (j < nj) ghg[(b0 + b) * H + j0 + j] = acc[r][c] + (bg ? bg[j0 + j] : 0.f);
      }
    }
  }
}

}  // namespace

bool lstm_gates_ok(const Geo &g) {
  return g.reuse && g.q == g.r_dim && g.rank <= 64 && g.s * g.rank <= 256 &&
         (g.s * g.rank) % 4 == 0 && g.n <= 1024 && g.n % 4 == 0;
}
size_t lstm_gates_ws(const Geo &g, int64_t batch) { return (size_t)(4 * batch * g.s * g.rank * 4); }

int lstm_gates(const Geo &g, int64_t batch, const float *h, const float *const *xf,
               const float *const *wf, const float *const *bias, float *const *gh, char *ws,
               cudaStream_t st) {
  if (batch == 0) return DT_OK;
  GateArgs a;
  for (int i = 0; i < 4; ++i) {
    a.xf[i] = xf[i]; a.wf[i] = wf[i]; a.bias[i] = bias ? bias[i] : nullptr; a.gh[i] = gh[i];
  }
  const int H = (int)g.q, n = (int)g.n, R = (int)g.rank, s = (int)g.s, K2 = s * R;
  float *P = reinterpret_cast<float *>(ws);
  const size_t smp = (size_t)(kPB + R) * (n + 1) * 4;
  const size_t smy = (size_t)(kGB + 64) * (K2 + 4) * 4;
  static bool attr = false;
  if (!attr) {
    DT_CUDA_CHECK(cudaFuncSetAttribute(k_gates_p, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    DT_CUDA_CHECK(cudaFuncSetAttribute(k_gates_y, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  k_gates_p<<<dim3((unsigned)s, 4, (unsigned)((batch + kPB - 1) / kPB)), 256, smp, st>>>(batch, H, n, R, h, a, P);
  if (int rc = check_launch("lstm_gates_p")) return rc;
  k_gates_y<<<dim3((unsigned)((H + 63) / 64), 4), 256, smy, st>>>(batch, H, K2, P, a);
  return check_launch("lstm_gates_y");
}

}  // namespace dt
