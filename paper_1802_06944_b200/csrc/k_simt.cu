#include <cstdlib>
// fp32 CUDA-core (FFMA) kernels of the DeepThin hot path — the rtol-1e-5 path.
//
// Everything here is exact-fp32 arithmetic on CUDA cores. The contractions are
// expressed as one generic register-tiled SIMT GEMM whose operand loaders are
// functors: plain strided matrices, or the DeepThin re-layout law evaluated on
// the fly (RegenW: W[i, j] = v[j*q + i] = sum_r xf[f / n, r] * wf[r, f % n],
// factor.py:87-93), so the dense W never exists in HBM.
//
//   reuse path (n | q, kernel.py:1-16 reuse with one phase):
//     P = x.view(B*s, n) @ wf^T            (run dots, each computed once)
//     y = P.view(B, s*rank) @ XF2^T + b    (XF2 = xf.view(r_dim, s*rank))
//   general path (straddling rows): y = x @ RegenW + b
//   backward (grad.py:63-95), any geometry:
//     g = up * act'(pre);  d_bias = colsum(g);  dWt = g^T @ x  (= d_v[:q*r_dim])
//     d_xf = d_aux @ wf^T; d_wf = xf^T @ d_aux (d_aux = dWt flat + zero tail)
//     d_input = g @ RegenW^T
// Split-K reductions write per-split partials and are summed in a fixed order,
// so every result is bitwise reproducible.

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <set>

#include <algorithm>
#include <atomic>
#include <type_traits>

#include "dt_internal.h"

namespace dt {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

__device__ __forceinline__ float act_apply(int act, float z, float arg) {
  switch (act) {
    case DT_ACT_RELU: return z > 0.f ? z : 0.f;
    case DT_ACT_SIGMOID: return 1.f / (1.f + expf(-z));
    case DT_ACT_TANH: return tanhf(z);
    case DT_ACT_CLIPPED_RELU: return fminf(fmaxf(z, 0.f), arg);
    default: return z;
  }
}

__device__ __forceinline__ float act_grad(int act, float z, float arg) {
  switch (act) {
    case DT_ACT_RELU: return z > 0.f ? 1.f : 0.f;
    case DT_ACT_SIGMOID: { float s = 1.f / (1.f + expf(-z)); return s * (1.f - s); }
    case DT_ACT_TANH: { float t = tanhf(z); return 1.f - t * t; }
    case DT_ACT_CLIPPED_RELU: return (z > 0.f && z < arg) ? 1.f : 0.f;
    default: return 1.f;
  }
}

// ---- operand loaders: element (row, col) of a logical matrix ------------------
// `k_fast` tells the tile loader which logical index is contiguous in memory.
struct MatF32 {
  const float *p;
  int64_t s0, s1;
  __device__ float operator()(int64_t i0, int64_t i1) const { return p[i0 * s0 + i1 * s1]; }
};
struct MatBF16 {
  const __nv_bfloat16 *p;
  int64_t s0, s1;
  __device__ float operator()(int64_t i0, int64_t i1) const {
    return __bfloat162float(p[i0 * s0 + i1 * s1]);
  }
};
// d_aux element (a, c): flat d_v[a*n + c], zero in the discarded tail (grad.py:87-91).
struct FlatPrefix {
  const float *p;  // dWt, r_dim x q row-major == d_v[:q*r_dim]
  int64_t n, qr;
  bool transpose;  // false: (a, c); true: (c, a)
  __device__ float operator()(int64_t i0, int64_t i1) const {
    int64_t a = transpose ? i1 : i0, c = transpose ? i0 : i1;
    int64_t f = a * n + c;
    return f < qr ? p[f] : 0.f;
  }
};
// W[i, j] regenerated from the factors; transpose=true serves (j, i).
struct RegenW {
  const float *xf, *wf;
  int64_t q, n, rank;
  bool transpose;
  __device__ float operator()(int64_t i0, int64_t i1) const {
    int64_t i = transpose ? i1 : i0, j = transpose ? i0 : i1;
    int64_t f = j * q + i;
    int64_t a = f / n, c = f - a * n;
    const float *xr = xf + a * rank;
    float acc = 0.f;
    for (int64_t r = 0; r < rank; ++r) acc = fmaf(xr[r], wf[r * n + c], acc);
    return acc;
  }
};

// ---- epilogues -------------------------------------------------------------------
struct EpiStore {  // out[m*ldc + n] = act(v + bias[n]) in f32 or bf16
  void *out;
  int64_t ldc;
  const float *bias;
  int act;
  float arg;
  int dtype;
  __device__ void operator()(int64_t m, int64_t n, float v) const {
    if (bias) v += bias[n];
    v = act_apply(act, v, arg);
    if (dtype == DT_BF16)
      reinterpret_cast<__nv_bfloat16 *>(out)[m * ldc + n] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float *>(out)[m * ldc + n] = v;
  }
};

// C[M x N] = sum_k A(m, k) * B(k, n) over k in [z*kchunk, min(K, (z+1)*kchunk)).
// splits > 1: partial sums go to part[z][M][N]; else epi(m, n, v).
template <bool A_KFAST, bool B_KFAST, class LA, class LB, class EPI>
__global__ void __launch_bounds__(NT) simt_gemm(int64_t M, int64_t N, int64_t K, int64_t kchunk,
                                                LA la, LB lb, EPI epi, float *part) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  const int tm = tid / 16, tn = tid % 16;
  float acc[4][4] = {};
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
    for (int l = 0; l < (BM * BK) / NT; ++l) {
      int e = tid + l * NT;
      int mm = A_KFAST ? e / BK : e % BM;
      int kk = A_KFAST ? e % BK : e / BM;
      int64_t gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < kend) ? la(gm, gk) : 0.f;
    }
#pragma unroll
    for (int l = 0; l < (BN * BK) / NT; ++l) {
      int e = tid + l * NT;
      int nn = B_KFAST ? e / BK : e % BN;
      int kk = B_KFAST ? e % BK : e / BN;
      int64_t gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < kend) ? lb(gk, gn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][tm * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + tm * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tn * 4 + j;
      if (n >= N) continue;
      if (part)
        part[((int64_t)blockIdx.z * M + m) * N + n] = acc[i][j];
      else
        epi(m, n, acc[i][j]);
    }
  }
}

// Fixed-order sum of split-K partials, then the epilogue.
template <class EPI>
__global__ void splitk_reduce(int64_t M, int64_t N, int splits, const float *part, EPI epi) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  float s = 0.f;
  for (int z = 0; z < splits; ++z) s += part[(int64_t)z * M * N + idx];
  epi(idx / N, idx % N, s);
}

// Split count: a pure function of the shape (determinism), aimed at >= ~2 waves.
int choose_splits(int64_t M, int64_t N, int64_t K) {
  int64_t tiles = std::max<int64_t>(1, ((M + BM - 1) / BM) * ((N + BN - 1) / BN));
  int64_t want = (2 * 148 + tiles - 1) / tiles;
  int64_t maxs = std::max<int64_t>(1, K / 256);
  return (int)std::max<int64_t>(1, std::min<int64_t>({want, maxs, 64}));
}

template <bool AK, bool BKF, class LA, class LB, class EPI>
int gemm(int64_t M, int64_t N, int64_t K, LA la, LB lb, EPI epi, float *part_ws,
         size_t part_bytes, cudaStream_t st, bool allow_split = true) {
  if (M == 0 || N == 0) return DT_OK;
  int splits = allow_split ? choose_splits(M, N, K) : 1;
  while (splits > 1 && (size_t)splits * M * N * sizeof(float) > part_bytes) --splits;
  if (K == 0) splits = 1;
  int64_t kchunk = splits > 1 ? ((K + splits - 1) / splits + BK - 1) / BK * BK : std::max<int64_t>(K, 1);
  splits = (int)((std::max<int64_t>(K, 1) + kchunk - 1) / kchunk);
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  simt_gemm<AK, BKF><<<grid, NT, 0, st>>>(M, N, K, kchunk, la, lb, epi,
                                          splits > 1 ? part_ws : nullptr);
  if (int rc = check_launch("simt_gemm")) return rc;
  if (splits > 1) {
    int64_t tot = M * N;
    splitk_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(M, N, splits, part_ws, epi);
    if (int rc = check_launch("splitk_reduce")) return rc;
  }
  return DT_OK;
}

size_t splitk_bytes(int64_t M, int64_t N, int64_t K) {
  return (size_t)choose_splits(M, N, K) * M * N * sizeof(float);
}

// ---- elementwise / reduction kernels ------------------------------------------------
__global__ void k_decompress(int64_t q, int64_t r_dim, int64_t rank, int64_t n, const float *xf,
                             const float *wf, float *w) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= q * r_dim) return;
  int64_t i = idx / r_dim, j = idx % r_dim;  // W row-major q x r_dim
  int64_t f = j * q + i, a = f / n, c = f - a * n;
  float acc = 0.f;
  for (int64_t r = 0; r < rank; ++r) acc = fmaf(xf[a * rank + r], wf[r * n + c], acc);
  w[idx] = acc;
}

__global__ void k_cast_bf16(int64_t count, const float *src, __nv_bfloat16 *dst) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) dst[idx] = __float2bfloat16_rn(src[idx]);
}

// g = up * act'(pre), pre already includes the bias.
__global__ void k_act_grad(int64_t count, const float *up, const float *pre, int act, float arg,
                           float *g) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) g[idx] = up[idx] * act_grad(act, pre[idx], arg);
}

// Column sums in a fixed order: part[c][j] = sum over rows of chunk c; then sum chunks.
__global__ void k_colsum_partial(int64_t rows, int64_t cols, int64_t rows_per_chunk,
                                 const float *g, float *part) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk, r1 = min(rows, r0 + rows_per_chunk);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += g[r * cols + j];
  part[(int64_t)blockIdx.y * cols + j] = s;
}
// column partial sums (as k_colsum_partial) fused with a fixed-order fp64 sum of (g*inv)^2
__global__ void __launch_bounds__(256) k_colsum_sq_partial(int64_t rows, int64_t cols, int64_t rpc,
                                                           const float *g, double inv, float *part,
                                                           double *sq_part) {
  __shared__ double red[256];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rpc, r1 = min(rows, r0 + rpc);
  float s = 0.f;
  double q = 0.0;
  if (j < cols) {
    for (int64_t r = r0; r < r1; ++r) {
      const float v = g[r * cols + j];
      s += v;
      const double d = v * inv;
      q += d * d;
    }
    part[(int64_t)blockIdx.y * cols + j] = s;
  }
  red[threadIdx.x] = q;
  __syncthreads();
  for (int h = blockDim.x / 2; h; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) sq_part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}
__global__ void k_colsum_final(int64_t cols, int chunks, const float *part, float *out) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  float s = 0.f;
  for (int c = 0; c < chunks; ++c) s += part[(int64_t)c * cols + j];
  out[j] = s;
}

// Row softmax in place (one CTA per row; fp32 reductions).
__global__ void k_row_softmax(int64_t cols, void *y, int dtype) {
  __shared__ float red[32];
  int64_t row = blockIdx.x;
  float *yf = reinterpret_cast<float *>(y) + row * cols;
  __nv_bfloat16 *yb = reinterpret_cast<__nv_bfloat16 *>(y) + row * cols;
  auto ld = [&](int64_t j) { return dtype == DT_BF16 ? __bfloat162float(yb[j]) : yf[j]; };
  float mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, ld(j));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) sum += expf(ld(j) - mx);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  float inv = 1.f / red[0];
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    float v = expf(ld(j) - mx) * inv;
    if (dtype == DT_BF16) yb[j] = __float2bfloat16_rn(v); else yf[j] = v;
  }
}

// Row softmax with the row held in registers: one warp per row, 16-byte vector loads and
// stores, max and sum by warp shuffles in a fixed order, exp2 on the log2e-prescaled
// difference (MUFU ex2, relative error ~2^-22). One HBM read and one write per element.
__device__ __forceinline__ float ex2f_approx(float x) {  // MUFU ex2, relative error ~2^-22
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int CPL, bool BF>
__global__ void __launch_bounds__(256) k_softmax_warp(int64_t rows, int cols, void *y) {
  constexpr int E = BF ? 8 : 4;  // elements per 16-byte chunk
  const int lane = threadIdx.x & 31;
  const int nch = cols / E;
  const float l2e = 1.4426950408889634f;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; row < rows;
       row += (int64_t)gridDim.x * blockDim.x / 32) {
    uint4 *yr = reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(y) + row * cols * (BF ? 2 : 4));
    float v[CPL][E];
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int ci = lane + 32 * c;
      if (ci < nch) {
        const uint4 w = yr[ci];
        if constexpr (BF) {
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            v[c][2 * k] = __uint_as_float(ws[k] << 16);
            v[c][2 * k + 1] = __uint_as_float(ws[k] & 0xffff0000u);
          }
        } else {
          v[c][0] = __uint_as_float(w.x); v[c][1] = __uint_as_float(w.y);
          v[c][2] = __uint_as_float(w.z); v[c][3] = __uint_as_float(w.w);
        }
#pragma unroll
        for (int k = 0; k < E; ++k) mx = fmaxf(mx, v[c][k]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      if (lane + 32 * c < nch) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          v[c][k] = ex2f_approx((v[c][k] - mx) * l2e);  // the difference first: exact near the max
          sum += v[c][k];
        }
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.f / sum;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int ci = lane + 32 * c;
      if (ci < nch) {
        uint4 w;
        if constexpr (BF) {
          uint32_t ws[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[c][2 * k] * inv, v[c][2 * k + 1] * inv);
            ws[k] = *reinterpret_cast<uint32_t *>(&h);
          }
          w = make_uint4(ws[0], ws[1], ws[2], ws[3]);
        } else {
          w = make_uint4(__float_as_uint(v[c][0] * inv), __float_as_uint(v[c][1] * inv),
                         __float_as_uint(v[c][2] * inv), __float_as_uint(v[c][3] * inv));
        }
        yr[ci] = w;
      }
    }
  }
}

// MSE: grad = 2 (y - t) / norm; per-block fp64 partial sums of squares, fixed order.
// grad.py:98-103 (mse): grad = 2 (y - t) / norm, per-block fp64 partial sums of (y - t)^2.
// Grid-stride over float4 groups with a grid size that depends only on `count`, so every
// partial has a fixed summation order (deterministic loss); HBM-bound (y, t read; grad written).
constexpr int kMseBlocks = 1184;  // 8 per SM
__global__ void __launch_bounds__(256) k_mse(int64_t count, const float *y, const float *t,
                                             double scale, float *grad, double *part) {
  __shared__ double red[256];
  double sq = 0.0;
  const int64_t n4 = count / 4, stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(t) |
                     reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
  if (vec) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 a = reinterpret_cast<const float4 *>(y)[i];
      const float4 b = reinterpret_cast<const float4 *>(t)[i];
      const float d0 = a.x - b.x, d1 = a.y - b.y, d2 = a.z - b.z, d3 = a.w - b.w;
      reinterpret_cast<float4 *>(grad)[i] =
          make_float4((float)(scale * d0), (float)(scale * d1), (float)(scale * d2), (float)(scale * d3));
      sq += (double)d0 * d0 + (double)d1 * d1 + (double)d2 * d2 + (double)d3 * d3;
    }
  }
  for (int64_t i = (vec ? 4 * n4 : 0) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const float d = y[i] - t[i];
    grad[i] = (float)(scale * (double)d);
    sq += (double)d * (double)d;
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// fixed-order sum of `count` fp64 partials (one block)
// fixed-order fp64 partial sums of (g * inv)^2 (the MSE loss recovered from its gradient)
__global__ void __launch_bounds__(256) k_sumsq(int64_t count, const float *g, double inv, double *part) {
  __shared__ double red[256];
  double sq = 0.0;
  const int64_t n4 = count / 4, stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  if (vec)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 a = reinterpret_cast<const float4 *>(g)[i];
      const double d0 = a.x * inv, d1 = a.y * inv, d2 = a.z * inv, d3 = a.w * inv;
      sq += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
    }
  for (int64_t i = (vec ? 4 * n4 : 0) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += stride) {
    const double d = g[i] * inv;
    sq += d * d;
  }
  red[threadIdx.x] = sq;
  __syncthreads();
  for (int s = blockDim.x / 2; s; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void __launch_bounds__(256) k_sum_f64(int64_t count, const double *part, double *out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = blockDim.x / 2; h; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

__global__ void k_sgd(int64_t count, float *p, const float *g, float lr) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < count) p[idx] -= lr * g[idx];
}

inline unsigned blocks_for(int64_t count, int tpb = 256) {
  return (unsigned)std::max<int64_t>(1, (count + tpb - 1) / tpb);
}

// Byte carving of a workspace.
struct Carver {
  char *base;
  size_t used = 0;
  template <class T> T *take(size_t count) {
    used = (used + 255) / 256 * 256;
    T *p = reinterpret_cast<T *>(base ? base + used : nullptr);
    used += count * sizeof(T);
    return p;
  }
};


// ---- reuse path, small batch: the two factored contractions in one kernel ------------------
// kernel.py:1-16 with one phase (n | q, s = q/n): column j of W is aux rows j*s .. j*s+s-1, so
//   P[b, seg, r] = sum_c x[b, seg*n + c] * wf[r, c]        (each distinct run dot once)
//   y[b, j]      = sum_{k < s*rank} P[b, k] * xf_flat[j*s*rank + k] + bias[j]
// A CTA owns one batch row x RC output columns (many small CTAs: the work is latency-bound, so
// parallelism beats reuse; the row's P is recomputed per column tile, s*rank*n FMAs). Every
// global operand it needs (the x row, wf, the XF2 tile) is staged into shared memory with
// cp.async first — all copies in flight at once — then P (warp-shuffle reductions in a fixed
// order) and the outputs (sequential s*rank-long dots) run from shared memory. Exact fp32
// FFMA; per-row results do not depend on the batch split.

// rows x cols (row stride src_ld) -> shared (row stride dst_ld), zero padded to `cols_pad`.
// fp32 sources go through cp.async (no register staging: every copy of the CTA is in flight at
// once); other types through registers. Call cp_async_wait_all() + a barrier before reading.
__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async16(float *dst, const float *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
template <typename T>
__device__ __forceinline__ void stage_rows(float *dst, int dst_ld, const T *src, int64_t src_ld,
                                           int rows, int rows_valid, int cols, int cols_pad) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if constexpr (std::is_same<T, float>::value) {
    if ((cols & 3) == 0 && (cols_pad & 3) == 0 && (dst_ld & 3) == 0 && (src_ld & 3) == 0 &&
        ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const int c4 = cols_pad / 4;
      for (int e = threadIdx.x; e < rows * c4; e += 256) {  // 16-byte copies
        const int r = e / c4, c = (e - r * c4) * 4;
        const bool ok = r < rows_valid && c < cols;
        cp_async16(dst + r * dst_ld + c, ok ? src + (int64_t)r * src_ld + c : src, ok);
      }
      return;
    }
  }
  for (int r = warp; r < rows; r += 8) {
    const bool rok = r < rows_valid;
    for (int c = lane; c < cols_pad; c += 32) {
      const bool ok = rok && c < cols;
      if constexpr (std::is_same<T, float>::value)
        cp_async4(dst + r * dst_ld + c, ok ? src + (int64_t)r * src_ld + c : src, ok);
      else
        dst[r * dst_ld + c] = ok ? (float)src[(int64_t)r * src_ld + c] : 0.f;
    }
  }
}

template <typename XT>
__global__ void __launch_bounds__(256) k_reuse_small(int64_t batch, int64_t q, int64_t r_dim,
                                                     int rank, int64_t n, int s, int RC,
                                                     const XT *x, const float *xf, const float *wf,
                                                     const float *bias, int act, float act_arg,
                                                     void *y, int y_dtype) {
  extern __shared__ __align__(16) float sm[];
  // rows padded to a multiple of 4 floats + 4: 16-byte-aligned for cp.async, and the padding
  // staggers the banks of consecutive rows
  const int SR = s * rank, SRP = (SR + 3) / 4 * 4 + 4;
  const int NP = ((int)n + 3) / 4 * 4 + 4, QP = ((int)q + 3) / 4 * 4;
  float *Xs = sm;                    // q (this CTA's batch row)
  float *Ws = Xs + QP;               // rank x NP
  float *X2 = Ws + rank * NP;        // RC x SRP
  float *Ps = X2 + RC * SRP;         // SR
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t b = blockIdx.x, j0 = (int64_t)blockIdx.y * RC;
  // 1) stage the x row, wf, the XF2 tile (rows j0.. of xf viewed r_dim x SR)
  stage_rows(Xs, (int)q, x + b * q, q, 1, 1, (int)q, (int)q);
  stage_rows(Ws, NP, wf, n, rank, rank, (int)n, (int)n);
  stage_rows(X2, SRP, xf + j0 * SR, SR, RC, (int)(r_dim - j0 < RC ? r_dim - j0 : RC), SR, SR);
  cp_async_wait_all();
  __syncthreads();
  // 2) P[seg*rank + r] = x[seg*n : (seg+1)*n] . wf[r, :]: a warp per dot, lanes along the segment,
  //    two dots per warp in flight, fixed-order shuffle reduction
  for (int d0 = warp; d0 < SR; d0 += 16) {
    const int d1 = d0 + 8;
    const float *x0 = Xs + (d0 / rank) * (int)n, *w0 = Ws + (d0 % rank) * NP;
    const float *x1 = Xs + (d1 < SR ? d1 / rank : 0) * (int)n, *w1 = Ws + (d1 < SR ? d1 % rank : 0) * NP;
    float a0 = 0.f, a1 = 0.f;
    for (int c = lane; c < (int)n; c += 32) {
      a0 = fmaf(x0[c], w0[c], a0);
      a1 = fmaf(x1[c], w1[c], a1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane == 0) {
      Ps[d0] = a0;
      if (d1 < SR) Ps[d1] = a1;
    }
  }
  __syncthreads();
  // 3) outputs j0 + jj: a thread per column, sequential SR-long dot, 4 partial sums. The
  //    tile row and P are read as float4: consecutive threads' rows are SRP (= 4 mod 32) floats
  //    apart, so scalar loads were 8-way bank conflicts; 16-byte loads of 8 threads cover 8
  //    distinct 16-byte bank groups. Partial sum kk still takes k = kk mod 4 in order.
  for (int jj = tid; jj < RC; jj += 256) {
    const int64_t j = j0 + jj;
    if (j >= r_dim) break;
    const float *xr = X2 + jj * SRP;
    const float4 *xr4 = reinterpret_cast<const float4 *>(xr);
    const float4 *p4 = reinterpret_cast<const float4 *>(Ps);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    int k = 0;
    for (; k + 4 <= SR; k += 4) {
      const float4 pv = p4[k >> 2], xv = xr4[k >> 2];
      acc[0] = fmaf(pv.x, xv.x, acc[0]);
      acc[1] = fmaf(pv.y, xv.y, acc[1]);
      acc[2] = fmaf(pv.z, xv.z, acc[2]);
      acc[3] = fmaf(pv.w, xv.w, acc[3]);
    }
    for (; k < SR; ++k) acc[0] = fmaf(Ps[k], xr[k], acc[0]);
    float v = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + (bias ? __ldg(bias + j) : 0.f);
    v = act_apply(act, v, act_arg);
    if (y_dtype == DT_BF16)
      reinterpret_cast<__nv_bfloat16 *>(y)[b * r_dim + j] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float *>(y)[b * r_dim + j] = v;
  }
}

// Launches k_reuse_small when the shape suits it (small batch, rank <= 64, tiles fit in
// shared memory); returns false to let the caller take the GEMM route.
template <typename XT>
static bool reuse_small(const Geo &g, int64_t batch, const XT *x, const float *xf, const float *wf,
                        const float *bias, int act, float act_arg, void *y, int y_dtype,
                        cudaStream_t st, int *rc) {
  const int SR = (int)(g.s * g.rank);
  if (!g.reuse || batch > 512 || g.rank > 64 || SR > 4096 || batch > 65535) return false;
  auto smem_for = [&](int rc) {
    return (size_t)((g.q + 3) / 4 * 4 + g.rank * ((g.n + 3) / 4 * 4 + 4) +
                    rc * ((SR + 3) / 4 * 4 + 4) + SR) * 4;
  };
  // output columns per CTA (DEEPTHIN_REUSE_RC overrides the cap, for tuning sweeps)
  static const int rc_cap = [] {
    const char *e = getenv("DEEPTHIN_REUSE_RC");
    const int v = e ? atoi(e) : 0;
    return (v >= 32 && v <= 512) ? v : 256;
  }();
  // up to 256 columns: <= 100 KB so two CTAs share an SM; 512 columns: one CTA per SM
  const size_t lim = rc_cap > 256 ? 200 * 1024 : 100 * 1024;
  int RC = rc_cap;
  while (RC > 32 && smem_for(RC) > lim) RC /= 2;
  const size_t smem = smem_for(RC);
  if (smem > lim) return false;
  const dim3 grid((unsigned)batch, (unsigned)((g.r_dim + RC - 1) / RC));
  cudaFuncSetAttribute(k_reuse_small<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_reuse_small<XT><<<grid, 256, smem, st>>>(batch, g.q, g.r_dim, (int)g.rank, g.n, (int)g.s, RC,
                                             x, xf, wf, bias, act, act_arg, y, y_dtype);
  *rc = check_launch("reuse_small");
  return true;
}

}  // namespace

std::atomic<int64_t> g_launches{0};

int check_launch(const char *what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return DT_E_CUDA;
  }
  return DT_OK;
}

int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void *>, int> g_smem_set;       // (device, fn) -> bytes set
std::set<std::pair<int, const void *>> g_nonportable_set;     // (device, fn)
std::set<std::pair<int, const void *>> g_carveout_set;        // (device, fn)
}  // namespace

int set_smem_limit(const void *fn, int bytes) {
  int dev = 0;
  DT_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_attr_mu);
  int &have = g_smem_set[{dev, fn}];
  if (have < bytes) {
    DT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
  }
  return DT_OK;
}

int prefer_max_smem_carveout(const void *fn) {
  int dev = 0;
  DT_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_attr_mu);
  if (g_carveout_set.insert({dev, fn}).second)
    DT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
  return DT_OK;
}

int allow_nonportable_clusters(const void *fn) {
  int dev = 0;
  DT_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_attr_mu);
  if (g_nonportable_set.insert({dev, fn}).second)
    DT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return DT_OK;
}

// ---- forward ------------------------------------------------------------------------
static size_t ffma_forward_carve(const Geo &g, int64_t batch, char *base, float **P, float **part,
                                 size_t *part_bytes) {
  Carver cv{base};
  size_t pb = 0;
  if (g.reuse) {
    *P = cv.take<float>((size_t)batch * g.s * g.rank);
    pb = std::max(splitk_bytes(batch * g.s, g.rank, g.n), splitk_bytes(batch, g.r_dim, g.s * g.rank));
  } else {
    *P = nullptr;
    pb = splitk_bytes(batch, g.r_dim, g.q);
  }
  *part = cv.take<float>(pb / sizeof(float));
  *part_bytes = pb;
  return cv.used;
}

size_t ffma_forward_ws(const Geo &g, int64_t batch) {
  float *P, *part;
  size_t pb;
  return ffma_forward_carve(g, batch, nullptr, &P, &part, &pb);
}

template <class XL>
static int ffma_forward_t(const Geo &g, int64_t batch, XL xl, const float *xf, const float *wf,
                          const float *bias, int act, float act_arg, void *y, int y_dtype, char *ws,
                          size_t ws_bytes, cudaStream_t st) {
  float *P, *part;
  size_t pb;
  size_t need = ffma_forward_carve(g, batch, ws, &P, &part, &pb);
  if (need > ws_bytes) {
    set_error("forward workspace too small: need " + std::to_string(need) + " bytes");
    return DT_E_ARG;
  }
  int sm_act = act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act;
  EpiStore out{y, g.r_dim, bias, sm_act, act_arg, y_dtype};
  int rc;
  if (g.reuse) {
    if (batch > 0) {  // small batches: both contractions in one kernel
      int src = 0;
      const bool done =
          reuse_small(g, batch, xl.p, xf, wf, bias, sm_act, act_arg, y, y_dtype, st, &src);
      if (done) {
        if (src) return src;
        if (act == DT_ACT_SOFTMAX) return launch_row_softmax(batch, g.r_dim, y, y_dtype, st);
        return DT_OK;
      }
    }
    // stage 1: P[(b*s + k), r] = sum_c x[b, k*n + c] * wf[r, c]   (one dot per distinct run)
    MatF32 wfT{wf, 1, g.n};  // (k=c, n=r) -> wf[r*n + c]
    EpiStore pst{P, g.rank, nullptr, DT_ACT_IDENTITY, 0.f, DT_F32};
    XL xseg = xl;
    xseg.s0 = g.n;  // row = segment index (b*s + k), contiguous rows of length n
    rc = gemm<true, true>(batch * g.s, g.rank, g.n, xseg, wfT, pst, part, pb, st);
    if (rc) return rc;
    // stage 2: y[b, j] = sum_kk P[b, kk] * xf[j*s*rank + kk]  (scale-after-dot combine)
    MatF32 pa{P, g.s * g.rank, 1};
    MatF32 xf2{xf, 1, g.s * g.rank};  // (k=kk, n=j)
    rc = gemm<true, true>(batch, g.r_dim, g.s * g.rank, pa, xf2, out, part, pb, st);
  } else {
    RegenW w{xf, wf, g.q, g.n, g.rank, false};  // (k=i, n=j)
    rc = gemm<true, true>(batch, g.r_dim, g.q, xl, w, out, part, pb, st);
  }
  if (rc) return rc;
  if (act == DT_ACT_SOFTMAX) return launch_row_softmax(batch, g.r_dim, y, y_dtype, st);
  return DT_OK;
}

int ffma_forward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                 const float *wf, const float *bias, int act, float act_arg, void *y, int y_dtype,
                 char *ws, size_t ws_bytes, cudaStream_t st) {
  if (x_dtype == DT_BF16)
    return ffma_forward_t(g, batch, MatBF16{(const __nv_bfloat16 *)x, g.q, 1}, xf, wf, bias, act,
                          act_arg, y, y_dtype, ws, ws_bytes, st);
  return ffma_forward_t(g, batch, MatF32{(const float *)x, g.q, 1}, xf, wf, bias, act, act_arg, y,
                        y_dtype, ws, ws_bytes, st);
}

// ---- backward -----------------------------------------------------------------------
struct BwdWs {
  float *pre, *gbuf, *dwt, *part, *colpart;
  size_t part_bytes;
  int chunks;
  int64_t rows_per_chunk;
};

static size_t ffma_backward_carve(const Geo &g, int64_t batch, char *base, BwdWs *w) {
  Carver cv{base};
  const int64_t qr = g.q * g.r_dim;
  w->pre = cv.take<float>((size_t)batch * g.r_dim);
  w->gbuf = cv.take<float>((size_t)batch * g.r_dim);
  w->dwt = cv.take<float>((size_t)qr);
  size_t pb = std::max({splitk_bytes(g.r_dim, g.q, batch), splitk_bytes(g.m, g.rank, g.n),
                        splitk_bytes(g.rank, g.n, g.m), splitk_bytes(batch, g.q, g.r_dim),
                        ffma_forward_ws(g, batch)});
  w->part = cv.take<float>(pb / sizeof(float));
  w->part_bytes = pb;
  w->rows_per_chunk = 256;
  w->chunks = (int)std::max<int64_t>(1, (batch + 255) / 256);
  w->colpart = cv.take<float>((size_t)w->chunks * g.r_dim);
  return cv.used;
}

size_t ffma_backward_ws(const Geo &g, int64_t batch) {
  BwdWs w;
  return ffma_backward_carve(g, batch, nullptr, &w);
}

template <class XL>
static int ffma_backward_t(const Geo &g, int64_t batch, XL xl, const void *x, int x_dtype,
                           const float *xf, const float *wf, const float *bias, int act,
                           float act_arg, const float *up, float *d_xf, float *d_wf, float *d_bias,
                           float *d_input, char *ws, size_t ws_bytes, cudaStream_t st) {
  BwdWs w;
  size_t need = ffma_backward_carve(g, batch, ws, &w);
  if (need > ws_bytes) {
    set_error("backward workspace too small: need " + std::to_string(need) + " bytes");
    return DT_E_ARG;
  }
  const int64_t BR = batch * g.r_dim;
  const float *gp = up;
  int rc;
  if (act != DT_ACT_IDENTITY) {  // grad.py:81-83: recompute pre, g = up * act'(pre)
    rc = ffma_forward(g, batch, x, x_dtype, xf, wf, bias, DT_ACT_IDENTITY, 0.f, w.pre, DT_F32,
                      reinterpret_cast<char *>(w.part), w.part_bytes, st);
    if (rc) return rc;
    k_act_grad<<<blocks_for(BR), 256, 0, st>>>(BR, up, w.pre, act, act_arg, w.gbuf);
    if ((rc = check_launch("act_grad"))) return rc;
    gp = w.gbuf;
  }
  if (d_bias) {  // grad.py:85
    dim3 grid(blocks_for(g.r_dim), (unsigned)w.chunks);
    k_colsum_partial<<<grid, 256, 0, st>>>(batch, g.r_dim, w.rows_per_chunk, gp, w.colpart);
    if ((rc = check_launch("colsum"))) return rc;
    k_colsum_final<<<blocks_for(g.r_dim), 256, 0, st>>>(g.r_dim, w.chunks, w.colpart, d_bias);
    if ((rc = check_launch("colsum_final"))) return rc;
  }
  // dWt[j, i] = sum_b g[b, j] x[b, i]  == d_v[:q*r_dim]  (grad.py:86-90)
  {
    MatF32 ga{gp, 1, g.r_dim};  // (m=j, k=b) -> g[b*r_dim + j]
    XL xb = xl;                 // (k=b, n=i) -> x[b*q + i]
    EpiStore st_dwt{w.dwt, g.q, nullptr, DT_ACT_IDENTITY, 0.f, DT_F32};
    rc = gemm<false, false>(g.r_dim, g.q, batch, ga, xb, st_dwt, w.part, w.part_bytes, st);
    if (rc) return rc;
  }
  const int64_t qr = g.q * g.r_dim;
  {  // d_xf[a, r] = sum_c d_aux[a, c] wf[r, c]       (grad.py:92)
    FlatPrefix da{w.dwt, g.n, qr, false};
    MatF32 wfT{wf, 1, g.n};
    EpiStore o{d_xf, g.rank, nullptr, DT_ACT_IDENTITY, 0.f, DT_F32};
    rc = gemm<true, true>(g.m, g.rank, g.n, da, wfT, o, w.part, w.part_bytes, st);
    if (rc) return rc;
  }
  {  // d_wf[r, c] = sum_a xf[a, r] d_aux[a, c]       (grad.py:93)
    MatF32 xfT{xf, 1, g.rank};  // (m=r, k=a) -> xf[a*rank + r]
    FlatPrefix da{w.dwt, g.n, qr, false};  // (k=a, n=c)
    EpiStore o{d_wf, g.n, nullptr, DT_ACT_IDENTITY, 0.f, DT_F32};
    rc = gemm<false, false>(g.rank, g.n, g.m, xfT, da, o, w.part, w.part_bytes, st);
    if (rc) return rc;
  }
  if (d_input) {  // d_input[b, i] = sum_j g[b, j] W[i, j]   (grad.py:94)
    MatF32 ga{gp, g.r_dim, 1};
    RegenW wt{xf, wf, g.q, g.n, g.rank, true};  // (k=j, n=i) -> W[i, j]
    EpiStore o{d_input, g.q, nullptr, DT_ACT_IDENTITY, 0.f, DT_F32};
    rc = gemm<true, false>(batch, g.q, g.r_dim, ga, wt, o, w.part, w.part_bytes, st);
    if (rc) return rc;
  }
  return DT_OK;
}

int ffma_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                  const float *wf, const float *bias, int act, float act_arg,
                  const float *upstream, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                  char *ws, size_t ws_bytes, cudaStream_t st) {
  if (x_dtype == DT_BF16)
    return ffma_backward_t(g, batch, MatBF16{(const __nv_bfloat16 *)x, g.q, 1}, x, x_dtype, xf,
                           wf, bias, act, act_arg, upstream, d_xf, d_wf, d_bias, d_input, ws,
                           ws_bytes, st);
  return ffma_backward_t(g, batch, MatF32{(const float *)x, g.q, 1}, x, x_dtype, xf, wf, bias, act,
                         act_arg, upstream, d_xf, d_wf, d_bias, d_input, ws, ws_bytes, st);
}

// ---- small launchers ------------------------------------------------------------------
int launch_act_grad(int64_t count, const float *up, const float *pre, int act, float act_arg,
                    float *out, cudaStream_t st) {
  if (count == 0) return DT_OK;
  k_act_grad<<<blocks_for(count), 256, 0, st>>>(count, up, pre, act, act_arg, out);
  return check_launch("act_grad");
}
size_t colsum_ws(int64_t rows, int64_t cols) {
  return (size_t)std::max<int64_t>(1, (rows + 255) / 256) * cols * sizeof(float);
}
int launch_colsum(int64_t rows, int64_t cols, const float *g, float *out, float *part,
                  cudaStream_t st) {
  const int chunks = (int)std::max<int64_t>(1, (rows + 255) / 256);
  dim3 grid(blocks_for(cols), (unsigned)chunks);
  k_colsum_partial<<<grid, 256, 0, st>>>(rows, cols, 256, g, part);
  if (int rc = check_launch("colsum")) return rc;
  k_colsum_final<<<blocks_for(cols), 256, 0, st>>>(cols, chunks, part, out);
  return check_launch("colsum_final");
}

int launch_decompress(const Geo &g, const float *xf, const float *wf, float *w, cudaStream_t st) {
  int64_t tot = g.q * g.r_dim;
  k_decompress<<<blocks_for(tot), 256, 0, st>>>(g.q, g.r_dim, g.rank, g.n, xf, wf, w);
  return check_launch("decompress");
}

int launch_cast_bf16(int64_t count, const float *src, uint16_t *dst, cudaStream_t st) {
  if (count == 0) return DT_OK;
  k_cast_bf16<<<blocks_for(count), 256, 0, st>>>(count, src, (__nv_bfloat16 *)dst);
  return check_launch("cast_bf16");
}

int launch_row_softmax(int64_t rows, int64_t cols, void *y, int y_dtype, cudaStream_t st) {
  if (rows == 0) return DT_OK;
  const bool bf = y_dtype == DT_BF16;
  const int E = bf ? 8 : 4;
  const int nch = (int)(cols / E);
  if (cols % E == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && nch <= 24 * 32) {
    const int cpl = (nch + 31) / 32;
    const unsigned grid = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 16);
    auto go = [&](auto kern) { kern<<<grid, 256, 0, st>>>(rows, (int)cols, y); };
    if (cpl <= 4) bf ? go(k_softmax_warp<4, true>) : go(k_softmax_warp<4, false>);
    else if (cpl <= 8) bf ? go(k_softmax_warp<8, true>) : go(k_softmax_warp<8, false>);
    else if (cpl <= 12) bf ? go(k_softmax_warp<12, true>) : go(k_softmax_warp<12, false>);
    else if (cpl <= 16) bf ? go(k_softmax_warp<16, true>) : go(k_softmax_warp<16, false>);
    else bf ? go(k_softmax_warp<24, true>) : go(k_softmax_warp<24, false>);
    return check_launch("row_softmax");
  }
  k_row_softmax<<<(unsigned)rows, 256, 0, st>>>(cols, y, y_dtype);
  return check_launch("row_softmax");
}

static unsigned mse_blocks(int64_t count) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(kMseBlocks, (count + 1023) / 1024));
}
size_t mse_ws(int64_t rows, int64_t cols) { return (size_t)mse_blocks(rows * cols) * sizeof(double); }

int launch_mse_grad(int64_t rows, int64_t cols, const float *y, const float *t, double norm,
                    float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st) {
  int64_t count = rows * cols;
  if (mse_ws(rows, cols) > ws_bytes) {
    set_error("mse workspace too small");
    return DT_E_ARG;
  }
  const unsigned nb = mse_blocks(count);
  k_mse<<<nb, 256, 0, st>>>(count, y, t, 2.0 / norm, grad, reinterpret_cast<double *>(ws));
  if (int rc = check_launch("mse")) return rc;
  if (loss_sum) {
    k_sum_f64<<<1, 256, 0, st>>>(nb, reinterpret_cast<double *>(ws), loss_sum);
    return check_launch("mse_sum");
  }
  return DT_OK;
}

int launch_colsum_sumsq(int64_t rows, int64_t cols, const float *g, double inv, float *out,
                        float *cpart, double *sq_part, double *loss, cudaStream_t st) {
  const int chunks = (int)std::max<int64_t>(1, (rows + 255) / 256);
  dim3 grid(blocks_for(cols), (unsigned)chunks);
  if ((int64_t)grid.x * grid.y > 1184) {  // the sq partials share the sumsq partial buffer
    set_error("colsum_sumsq: too many blocks for the partial buffer");
    return DT_E_UNSUPPORTED;
  }
  k_colsum_sq_partial<<<grid, 256, 0, st>>>(rows, cols, 256, g, inv, cpart, sq_part);
  if (int rc = check_launch("colsum_sumsq")) return rc;
  k_colsum_final<<<blocks_for(cols), 256, 0, st>>>(cols, chunks, cpart, out);
  if (int rc = check_launch("colsum_final")) return rc;
  if (!loss) return DT_OK;
  k_sum_f64<<<1, 256, 0, st>>>((int64_t)grid.x * grid.y, sq_part, loss);
  return check_launch("sumsq_sum");
}

int launch_sumsq(int64_t count, const float *g, double inv, double *part, double *out, cudaStream_t st) {
  const unsigned nb = mse_blocks(count);
  k_sumsq<<<nb, 256, 0, st>>>(count, g, inv, part);
  if (int rc = check_launch("sumsq")) return rc;
  if (!out) return DT_OK;
  k_sum_f64<<<1, 256, 0, st>>>(nb, part, out);
  return check_launch("sumsq_sum");
}

int launch_sum_f64(int64_t count, const double *part, double *out, cudaStream_t st) {
  k_sum_f64<<<1, 256, 0, st>>>(count, part, out);
  return check_launch("sum_f64");
}

int launch_sgd(int64_t count, float *p, const float *g, float lr, cudaStream_t st) {
  if (count == 0) return DT_OK;
  k_sgd<<<blocks_for(count), 256, 0, st>>>(count, p, g, lr);
  return check_launch("sgd");
}

}  // namespace dt
