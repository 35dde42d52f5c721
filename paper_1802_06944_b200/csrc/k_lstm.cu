// LSTM cell of BASELINE config 4 (speech-RNN-shaped model): the elementwise step that follows
// the eight DeepThin-compressed gate contractions. Not in the reference (SURVEY.md §8(a) a8:
// LSTM gates are "not in the reference"); its math is the standard cell, gate order i, f, g, o:
//   i = sigmoid(gx_i + gh_i), f = sigmoid(gx_f + gh_f), g = tanh(gx_g + gh_g),
//   o = sigmoid(gx_o + gh_o), c' = f c + i g, h' = o tanh(c').
// gx: input projections (bf16, batched over all time steps by the tensor-core path, biases
// included); gh: recurrent projections (fp32, this step). c is updated in place (fp32); h' is
// written in fp32 (next step's recurrent input) and bf16 (the sequence output).
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "dt_internal.h"
#include "sm100_ptx.cuh"

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
// four reuse-geometry DeepThin layers H -> H), fp32-accurate (3xTF32 mma.sync tiles), factored exactly
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
// COHERENT: L2-only loads (ld.global.cg) for data other CTAs write during the same kernel (the
// persistent recurrence's P and h); otherwise the read-only path.
template <bool COHERENT = false>
__device__ __forceinline__ void stage_rows(float *dst, int sp, const float *src, int64_t ld, int rows,
                                           int cols) {
  const int c4 = cols / 4, n4 = rows * c4;
  for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n4) {
        const float4 *a4 = reinterpret_cast<const float4 *>(src + (int64_t)(i / c4) * ld) + i % c4;
        v[u] = COHERENT ? __ldcg(a4) : __ldg(a4);
      }
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

// 64 x 64 output tile D[b][j] = sum_kk ps[b][kk] * xs[j][kk] (row pitch kp floats) on the tensor
// cores: mma.sync m16n8k8 tf32 in the 3xTF32 form (lo*hi + hi*lo + hi*hi), x = hi + lo split
// exactly by masking the low 13 mantissa bits (integer ops: cvt.rna.tf32 runs at a quarter of
// the ALU rate and made this tile conversion-bound); the MMA truncates lo to tf32, leaving
// ~2^-20 relative error per product. 8 warps, warp w owns rows 16*(w%4).. and columns
// 32*(w/4).. (4 n-tiles of 8). acc[nt][4]: m16n8 fragments.
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tile64_3xtf32(const float *ps, const float *xs, int kp, int K2,
                                              float (&acc)[4][4]) {
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32, gid = lane >> 2, tig = lane & 3;
  const int r0 = 16 * (w & 3), c0 = 32 * (w >> 2);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nt][i] = 0.f;
  for (int kk = 0; kk < K2; kk += 8) {
    const float av[4] = {ps[(r0 + gid) * kp + kk + tig], ps[(r0 + gid + 8) * kp + kk + tig],
                         ps[(r0 + gid) * kp + kk + tig + 4], ps[(r0 + gid + 8) * kp + kk + tig + 4]};
    uint32_t ah[4], al[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(av[i], ah[i], al[i]);
    uint32_t bh[4][2], bl[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float *xr = xs + (c0 + nt * 8 + gid) * kp + kk;
      split_tf32(xr[tig], bh[nt][0], bl[nt][0]);
      split_tf32(xr[tig + 4], bh[nt][1], bl[nt][1]);
    }
    // the three passes each sweep the four n-tiles, so consecutive MMAs are independent (an
    // accumulator's three products stay in the same order: lo*hi, hi*lo, hi*hi)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[nt], al, bh[nt][0], bh[nt][1]);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[nt], ah, bl[nt][0], bl[nt][1]);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) mma_tf32(acc[nt], ah, bh[nt][0], bh[nt][1]);
  }
}
// store the tile's fragments: D[b][j] + bias -> out[(b0 + b) * ld + j0 + j] (b < nb, j < nj)
__device__ __forceinline__ void tile64_store(const float (&acc)[4][4], float *out, int64_t ld,
                                             int64_t b0, int nb, int j0, int nj, const float *bias) {
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32, gid = lane >> 2, tig = lane & 3;
  const int r0 = 16 * (w & 3), c0 = 32 * (w >> 2);
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int b = r0 + gid + (i >= 2 ? 8 : 0), j = c0 + nt * 8 + 2 * tig + (i & 1);
      if (b < nb && j < nj) out[(b0 + b) * ld + j0 + j] = acc[nt][i] + (bias ? bias[j0 + j] : 0.f);
    }
}

// Segment-dot tile of the P phase on the tensor cores (3xTF32, as tile64_3xtf32):
//   P[b][k] = sum_t hs[b][t] * ws[k][t],  b < 16, k < R8 (<= 64, rows >= R zero), t < n8
// (row pitch npad = n8 + 4: conflict-free fragment loads). Warp w takes k-steps w, w + 8, ... for
// every n-tile; the 8 warp partials land in red[w][16][R8] and p_tile_sum adds them in warp order.
// Per CTA this reads 8x less shared memory than one-dot-per-thread FFMA, which was
// shared-memory-bandwidth bound.
__device__ __forceinline__ int lstm_npad(int n) { return (n + 7) / 8 * 8 + 4; }
__device__ __forceinline__ void p_tile_3xtf32(const float *hs, const float *ws, int npad, int n8, int R8,
                                              float *red) {
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32, gid = lane >> 2, tig = lane & 3;
  const int ntiles = R8 / 8;
  float acc[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[nt][i] = 0.f;
  for (int kk = 8 * w; kk < n8; kk += 64) {
    const float av[4] = {hs[gid * npad + kk + tig], hs[(gid + 8) * npad + kk + tig],
                         hs[gid * npad + kk + tig + 4], hs[(gid + 8) * npad + kk + tig + 4]};
    uint32_t ah[4], al[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) split_tf32(av[i], ah[i], al[i]);
    uint32_t bh[8][2], bl[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      if (nt < ntiles) {
        const float *wr = ws + (nt * 8 + gid) * npad + kk;
        split_tf32(wr[tig], bh[nt][0], bl[nt][0]);
        split_tf32(wr[tig + 4], bh[nt][1], bl[nt][1]);
      }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      if (nt < ntiles) mma_tf32(acc[nt], al, bh[nt][0], bh[nt][1]);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      if (nt < ntiles) mma_tf32(acc[nt], ah, bl[nt][0], bl[nt][1]);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      if (nt < ntiles) mma_tf32(acc[nt], ah, bh[nt][0], bh[nt][1]);
  }
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
    if (nt < ntiles)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        red[(w * 16 + gid + (i >= 2 ? 8 : 0)) * R8 + nt * 8 + 2 * tig + (i & 1)] = acc[nt][i];
}
// out[b * ldo + k] = sum over warps of red (fixed order), b < nb, k < R (after a __syncthreads)
__device__ __forceinline__ void p_tile_sum(const float *red, int R8, int R, int nb, float *out, int64_t ldo) {
  for (int o = threadIdx.x; o < nb * R; o += blockDim.x) {
    const int b = o / R, k = o % R;
    float v = red[b * R8 + k];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += red[(w * 16 + b) * R8 + k];
    out[(int64_t)b * ldo + k] = v;
  }
}
// zero a staged operand before its first use: the padding rows/columns the MMAs read
__device__ __forceinline__ void zero_smem(float *p, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) p[i] = 0.f;
}

// one CTA per (segment, gate, 16-row block): h[rows, seg] and wf_g in shared memory, the
// segment dots on the tensor cores (p_tile_3xtf32)
__global__ void __launch_bounds__(256) k_gates_p(int64_t batch, int H, int n, int R, const float *h,
                                                 GateArgs a, float *P) {
  extern __shared__ float sm[];
  const int seg = blockIdx.x, g = blockIdx.y, s = H / n, K2 = s * R;
  const int64_t b0 = (int64_t)blockIdx.z * kPB;
  const int nb = (int)(batch - b0 < kPB ? batch - b0 : kPB);
  const int npad = lstm_npad(n), n8 = (n + 7) / 8 * 8, R8 = (R + 7) / 8 * 8;
  float *hs = sm, *ws = hs + kPB * npad, *red = ws + R8 * npad;
  const float *wfg = g == 0 ? a.wf[0] : g == 1 ? a.wf[1] : g == 2 ? a.wf[2] : a.wf[3];
  zero_smem(sm, (kPB + R8) * npad);
  __syncthreads();
  stage_rows(ws, npad, wfg, n, R, n);
  stage_rows(hs, npad, h + b0 * H + seg * n, H, nb, n);
  __syncthreads();
  p_tile_3xtf32(hs, ws, npad, n8, R8, red);
  __syncthreads();
  p_tile_sum(red, R8, R, nb, P + ((int64_t)g * batch + b0) * K2 + seg * R, K2);
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
  for (int64_t b0 = 0; b0 < batch; b0 += kGB) {
    const int nb = (int)(batch - b0 < kGB ? batch - b0 : kGB);
    __syncthreads();
    stage_rows(ps, kp, P + ((int64_t)g * batch + b0) * K2, K2, nb, K2);
    for (int i = nb * kp + threadIdx.x; i < kGB * kp; i += blockDim.x) ps[i] = 0.f;  // pad rows
    for (int i = nj * kp + threadIdx.x; i < 64 * kp; i += blockDim.x) xs[i] = 0.f;
    __syncthreads();
    float acc[4][4];
    tile64_3xtf32(ps, xs, kp, K2, acc);
    tile64_store(acc, ghg, H, b0, nb, j0, nj, bg);
  }
}

}  // namespace

bool lstm_gates_ok(const Geo &g) {
  return g.reuse && g.q == g.r_dim && g.rank <= 64 && g.s * g.rank <= 256 &&
         (g.s * g.rank) % 8 == 0 && g.n <= 1024 && g.n % 4 == 0;
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
  const int R8 = (R + 7) / 8 * 8;
  const size_t smp = ((size_t)(kPB + R8) * ((n + 7) / 8 * 8 + 4) + (size_t)8 * 16 * R8) * 4;
  const size_t smy = (size_t)(kGB + 64) * (K2 + 4) * 4;
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(k_gates_p), 227 * 1024)) return rc;
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(k_gates_y), 227 * 1024)) return rc;
  k_gates_p<<<dim3((unsigned)s, 4, (unsigned)((batch + kPB - 1) / kPB)), 256, smp, st>>>(batch, H, n, R, h, a, P);
  if (int rc = check_launch("lstm_gates_p")) return rc;
  k_gates_y<<<dim3((unsigned)((H + 63) / 64), 4), 256, smy, st>>>(batch, H, K2, P, a);
  return check_launch("lstm_gates_y");
}

}  // namespace dt

// =============================================================================================
// The whole LSTM recurrence in ONE persistent kernel (config 4): T steps, two grid-wide
// barriers per step in the fused gate-cluster form (three in the general form), no host
// launches inside the loop. Work units (3xTF32 tiles, fp32 cell):
//   phase P, unit (gate g, segment seg, 16-row group rg):
//     P_g[rows, seg*R + k] = h[rows, seg cols] . wf_g[k, :]        (p_tile_3xtf32)
//   phase G, unit (gate g, 64-column block): gh_g[:, cols] = P_g @ XF2_g[cols]^T + b_hg
//   phase C: the cell over all of B x H (c, h in place; the bf16 sequence output)
// Same arithmetic (and summation order) as k_gates_p / k_gates_y / k_lstm_cell, so the
// per-step form gives the same bits.
// =============================================================================================
namespace dt {
namespace {

struct SeqArgs {
  const float *xf[4], *wf[4], *bias[4];
  const __nv_bfloat16 *gx[4];  // T*B x H each (biases of the input projections included)
  float *gh;                   // 4 x B x H
  float *P;                    // 4 x B x Pld (rows at the staged pitch K2 + 4: one bulk copy per gate tile)
  int Pld;
  float *c;                    // B x H cell state
  float *h;                    // B x H hidden state (fp32, the recurrent contractions' input)
  __nv_bfloat16 *out;          // T*B x H
  unsigned *bar;               // grid barrier counter (zeroed before launch)
  unsigned long long *trace;   // DEEPTHIN_LSTM_TRACE: globaltimer stamps (block 0, first steps)
  int T, B, H, n, R, s, K2;
  int vec;  // gx pointers 8-byte aligned (H % 4 == 0 always): vectorized cell
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// grid-wide barrier: monotone counter, the k-th barrier completes at k * gridDim.x arrivals
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned &target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    // release-add (cumulative over the CTA's writes ordered by the __syncthreads above); no
    // separate fence and no returned value to wait for
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (ld_acquire_gpu(bar) < target) {
    }
  }
  __syncthreads();
}

using namespace ptx;

__device__ __forceinline__ float sigm_(float z) { return 1.f / (1.f + expf(-z)); }

// Stage rows x cols fp32 (row pitch ld) into shared memory (row pitch sp) with 1-D bulk copies
// (one per row, issued by the lanes of warp 0), completion counted on `bar`; every thread
// waits. For data other CTAs wrote before the last grid barrier (P, h): the copies read L2
// through the async proxy, ordered after the barrier's acquire by fence.proxy.async. Many
// more bytes in flight than per-thread loads, so the 32-readers-per-line P broadcast no longer
// waits on two serial L2 round trips.
__device__ __forceinline__ void bulk_stage(float *dst, int sp, const float *src, int64_t ld, int rows,
                                           int cols, uint64_t *bar, uint32_t &phase) {
  if (ld == sp) {  // source rows already at the staged pitch: ONE copy of the whole block
    if (threadIdx.x == 0) {
      fence_proxy_async_global();
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, (uint32_t)(rows * sp * 4));
      bulk_load(dst, src, (uint32_t)(rows * sp * 4), bar);
    }
  } else if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      fence_proxy_async_global();
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, (uint32_t)(rows * cols * 4));
    }
    __syncwarp();
    fence_proxy_async_global();
    for (int r = threadIdx.x; r < rows; r += 32) bulk_load(dst + (size_t)r * sp, src + r * ld, cols * 4, bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
}


// FUSED: the four gate tiles of one 64-column block sit in one cluster of four CTAs (gate =
// cluster rank). After its tile each CTA scatters its gate's pre-activations into the peers'
// shared memory (DSMEM), 16 columns of the block per peer, and after one cluster barrier every
// CTA runs the cell for its 64 rows x 16 columns with c held in registers for the whole
// sequence: no gh round trip through L2, no separate cell phase and two grid barriers per step
// instead of three. Same arithmetic and order per element as the unfused phases (same bits).
template <bool FUSED>
__global__ void __launch_bounds__(256, 1) k_lstm_seq(SeqArgs a) {
  extern __shared__ float sm[];
  const int B = a.B, H = a.H, n = a.n, R = a.R, K2 = a.K2;
  const int npad = lstm_npad(n), n8 = (n + 7) / 8 * 8, R8 = (R + 7) / 8 * 8, kp = K2 + 4;
  const int rgs = (B + 15) / 16;
  const int unitsP = 4 * a.s * rgs, unitsB = 4 * ((H + 63) / 64);
  const int64_t BH = (int64_t)B * H;
  // one P unit and one gate-tile unit per CTA when the grid covers them: their factor operands
  // (wf_g, and the 64-column XF2_g block) stay resident in shared memory for all T steps
  float *hs = sm, *ws = hs + 16 * npad, *red = ws + R8 * npad, *ps = red + 128 * R8;
  ps += (4 - ((ps - sm) & 3)) & 3;  // 16-byte alignment for the staged tiles
  float *xs = ps + 64 * kp;
  float *g4 = xs + 64 * kp;  // FUSED: [4 gates][64 rows][16 columns] gate pre-activations
  const int nblk = (H + 63) / 64;
  // G unit -> (gate, column block): gate-major, or cluster rank = gate when fused
  auto unit_gate = [&](int u) { return FUSED ? (u & 3) : u / nblk; };
  auto unit_j0 = [&](int u) { return (FUSED ? (u >> 2) : u % nblk) * 64; };
  const bool resP = unitsP <= (int)gridDim.x, resB = unitsB <= (int)gridDim.x;
  auto wf_of = [&](int g) { return g == 0 ? a.wf[0] : g == 1 ? a.wf[1] : g == 2 ? a.wf[2] : a.wf[3]; };
  auto xf_of = [&](int g) { return g == 0 ? a.xf[0] : g == 1 ? a.xf[1] : g == 2 ? a.xf[2] : a.xf[3]; };
  auto stage_xs = [&](int u) {
    const int g = unit_gate(u), j0 = unit_j0(u), nj = min(64, H - j0);
    stage_rows(xs, kp, xf_of(g) + (size_t)j0 * K2, K2, nj, K2);
    for (int i = nj * kp + threadIdx.x; i < 64 * kp; i += blockDim.x) xs[i] = 0.f;
  };
  __shared__ uint64_t sbar[2];  // bulk_stage completion: [0] h rows (phase P), [1] P_g (phase G)
  uint32_t sph[2] = {0u, 0u};
  if (threadIdx.x == 0) {
    mbar_init(&sbar[0], 1);
    mbar_init(&sbar[1], 1);
    fence_mbar_init();
  }
  zero_smem(sm, (16 + R8) * npad);  // padding rows/columns of the P tile's operands stay zero
  __syncthreads();
  if (resP && (int)blockIdx.x < unitsP) stage_rows(ws, npad, wf_of((int)blockIdx.x / (a.s * rgs)), n, R, n);
  if (resB && (int)blockIdx.x < unitsB) stage_xs((int)blockIdx.x);
  unsigned target = 0;
  auto stamp = [&](int t, int k) {
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 8) {
      unsigned long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      a.trace[t * 8 + k] = v;
    }
  };
  // phase C: the cell of step t (all of B x H, grid-strided; each element owned by one thread)
  auto cell = [&](int t) {
    const size_t gxo0 = (size_t)t * BH;
    if (a.vec) {  // 4 consecutive elements per thread: all nine loads in flight at once
      const int64_t BH4 = BH / 4;
      for (int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e4 < BH4;
           e4 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = 4 * e4;
        float4 z[4];
        uint2 xg[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          z[q] = __ldcg(reinterpret_cast<const float4 *>(a.gh + q * BH + e));
          xg[q] = __ldg(reinterpret_cast<const uint2 *>(a.gx[q] + gxo0 + e));
        }
        const float4 c4 = *reinterpret_cast<const float4 *>(a.c + e);
        const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
        float zz[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162 *>(&xg[q].x);
          const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162 *>(&xg[q].y);
          zz[q][0] = __low2float(lo) + z[q].x;
          zz[q][1] = __high2float(lo) + z[q].y;
          zz[q][2] = __low2float(hi) + z[q].z;
          zz[q][3] = __high2float(hi) + z[q].w;
        }
        float cn[4], hn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          cn[k] = sigm_(zz[1][k]) * cv[k] + sigm_(zz[0][k]) * tanhf(zz[2][k]);
          hn[k] = sigm_(zz[3][k]) * tanhf(cn[k]);
        }
        *reinterpret_cast<float4 *>(a.c + e) = make_float4(cn[0], cn[1], cn[2], cn[3]);
        *reinterpret_cast<float4 *>(a.h + e) = make_float4(hn[0], hn[1], hn[2], hn[3]);
        __nv_bfloat162 o0 = __floats2bfloat162_rn(hn[0], hn[1]), o1 = __floats2bfloat162_rn(hn[2], hn[3]);
        uint2 ov;
        ov.x = *reinterpret_cast<uint32_t *>(&o0);
        ov.y = *reinterpret_cast<uint32_t *>(&o1);
        *reinterpret_cast<uint2 *>(a.out + gxo0 + e) = ov;
      }
      return;
    }
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < BH;
         e += (int64_t)gridDim.x * blockDim.x) {
      const float zi = __bfloat162float(a.gx[0][gxo0 + e]) + a.gh[e];
      const float zf = __bfloat162float(a.gx[1][gxo0 + e]) + a.gh[BH + e];
      const float zg = __bfloat162float(a.gx[2][gxo0 + e]) + a.gh[2 * BH + e];
      const float zo = __bfloat162float(a.gx[3][gxo0 + e]) + a.gh[3 * BH + e];
      const float cn = sigm_(zf) * a.c[e] + sigm_(zi) * tanhf(zg);
      const float hn = sigm_(zo) * tanhf(cn);
      a.c[e] = cn;
      a.h[e] = hn;
      a.out[gxo0 + e] = __float2bfloat16_rn(hn);
    }
  };
  float creg[4] = {0.f, 0.f, 0.f, 0.f};  // FUSED: this thread's four cell states, c(-1) = 0
  for (int t = 0; t < a.T; ++t) {
    // ---------------- phase P: P_g[rows, seg*R + k] = h[rows, seg] . wf_g[k, :] ----------------
    for (int u = blockIdx.x; u < unitsP; u += gridDim.x) {
      const int g = u / (a.s * rgs), seg = (u / rgs) % a.s, rg = u % rgs;
      const int b0 = rg * 16, nb = min(16, B - b0);
      __syncthreads();
      if (!resP) stage_rows(ws, npad, wf_of(g), n, R, n);
      bulk_stage(hs, npad, a.h + (size_t)b0 * H + seg * n, H, nb, n, &sbar[0], sph[0]);
      __syncthreads();
      p_tile_3xtf32(hs, ws, npad, n8, R8, red);
      __syncthreads();
      p_tile_sum(red, R8, R, nb, a.P + ((size_t)g * B + b0) * a.Pld + seg * R, a.Pld);
    }
    stamp(t, 0);
    grid_barrier(a.bar, target);
    stamp(t, 1);
    // ---------------- phase G: gh_g[:, 64-column block] = P_g XF2_g^T + b (3xTF32 mma) -----------
    if constexpr (FUSED) {
      // one unit per CTA (launcher: gridDim.x == unitsB, H % 64 == 0, clusters of 4)
      const int g = (int)blockIdx.x & 3, j0 = ((int)blockIdx.x >> 2) * 64;
      const float *bg = g == 0 ? a.bias[0] : g == 1 ? a.bias[1] : g == 2 ? a.bias[2] : a.bias[3];
      // this thread's cell elements: row cb, block columns 16 g + 4 cq .. + 3; their input
      // projections are independent of the recurrence: fetched before the tile
      const int cb = threadIdx.x >> 2, cq = threadIdx.x & 3, cj = j0 + 16 * g + 4 * cq;
      const size_t gxo = ((size_t)t * B + cb) * H + cj;
      uint2 xg[4];
      if (cb < B) {
#pragma unroll
        for (int q = 0; q < 4; ++q) xg[q] = __ldg(reinterpret_cast<const uint2 *>(a.gx[q] + gxo));
      }
      bulk_stage(ps, kp, a.P + (size_t)g * B * a.Pld, a.Pld, B, K2, &sbar[1], sph[1]);
      if (t == 0) {
        for (int i = B * kp + threadIdx.x; i < 64 * kp; i += blockDim.x) ps[i] = 0.f;
      }
      __syncthreads();
      stamp(t, 6);
      float acc[4][4];
      tile64_3xtf32(ps, xs, kp, K2, acc);
      __syncwarp();
      stamp(t, 7);
      {  // scatter: block column j -> peer j / 16, slot [g][row][j % 16] (column pairs: 8 bytes)
        const int w = threadIdx.x / 32, lane = threadIdx.x % 32, gid = lane >> 2, tig = lane & 3;
        const int r0 = 16 * (w & 3), c0 = 32 * (w >> 2);
        const uint32_t base = smem_u32(g4) + (uint32_t)(g * 64 * 16) * 4u;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const int j = c0 + nt * 8 + 2 * tig;
          const uint32_t peer = (uint32_t)(j >> 4);
          const float b0v = bg ? __ldg(bg + j0 + j) : 0.f, b1v = bg ? __ldg(bg + j0 + j + 1) : 0.f;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int b = r0 + gid + 8 * hh;
            const uint32_t dst = mapa_shared(base + (uint32_t)(b * 16 + (j & 15)) * 4u, peer);
            asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(dst),
                         "f"(acc[nt][2 * hh] + b0v), "f"(acc[nt][2 * hh + 1] + b1v)
                         : "memory");
          }
        }
      }
      cluster_sync();  // release / acquire at cluster scope: every peer's scatter has landed
      stamp(t, 2);
      stamp(t, 3);
      if (cb < B) {
        float4 z[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          z[q] = *reinterpret_cast<const float4 *>(g4 + (q * 64 + cb) * 16 + 4 * cq);
        float zz[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162 *>(&xg[q].x);
          const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162 *>(&xg[q].y);
          zz[q][0] = __low2float(lo) + z[q].x;
          zz[q][1] = __high2float(lo) + z[q].y;
          zz[q][2] = __low2float(hi) + z[q].z;
          zz[q][3] = __high2float(hi) + z[q].w;
        }
        float hn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          creg[k] = sigm_(zz[1][k]) * creg[k] + sigm_(zz[0][k]) * tanhf(zz[2][k]);
          hn[k] = sigm_(zz[3][k]) * tanhf(creg[k]);
        }
        *reinterpret_cast<float4 *>(a.h + (size_t)cb * H + cj) = make_float4(hn[0], hn[1], hn[2], hn[3]);
        __nv_bfloat162 o0 = __floats2bfloat162_rn(hn[0], hn[1]), o1 = __floats2bfloat162_rn(hn[2], hn[3]);
        uint2 ov;
        ov.x = *reinterpret_cast<uint32_t *>(&o0);
        ov.y = *reinterpret_cast<uint32_t *>(&o1);
        *reinterpret_cast<uint2 *>(a.out + gxo) = ov;
      }
      stamp(t, 4);
      grid_barrier(a.bar, target);
      stamp(t, 5);
    } else {
    for (int u = blockIdx.x; u < unitsB; u += gridDim.x) {
      const int g = unit_gate(u), j0 = unit_j0(u), nj = min(64, H - j0);
      const float *bg = g == 0 ? a.bias[0] : g == 1 ? a.bias[1] : g == 2 ? a.bias[2] : a.bias[3];
      __syncthreads();
      if (!resB) stage_xs(u);
      bulk_stage(ps, kp, a.P + (size_t)g * B * a.Pld, a.Pld, B, K2, &sbar[1], sph[1]);
      for (int i = B * kp + threadIdx.x; i < 64 * kp; i += blockDim.x) ps[i] = 0.f;
      __syncthreads();
      stamp(t, 6);
      float acc[4][4];
      tile64_3xtf32(ps, xs, kp, K2, acc);
      __syncwarp();
      stamp(t, 7);
      tile64_store(acc, a.gh + (size_t)g * BH, H, 0, B, j0, nj, bg);
    }
    stamp(t, 2);
    grid_barrier(a.bar, target);
    stamp(t, 3);
    cell(t);
    stamp(t, 4);
    grid_barrier(a.bar, target);
    stamp(t, 5);
    }
  }
  if constexpr (FUSED) cluster_sync();  // no CTA exits while a peer may still address its memory
}

}  // namespace

// hs (16 rows) | ws (R8 rows) | P-tile partials (8 x 16 x R8) | align | ps, xs (64 rows each)
static size_t lstm_seq_smem(const Geo &g) {
  const size_t r8 = (g.rank + 7) / 8 * 8, npad = (g.n + 7) / 8 * 8 + 4;
  return ((16 + r8) * npad + 128 * r8 + 4 + (size_t)128 * (g.s * g.rank + 4)) * 4;
}
bool lstm_seq_ok(const Geo &g, int64_t batch) {
  return lstm_gates_ok(g) && batch >= 1 && batch <= 64 && g.n <= 1024 &&
         lstm_seq_smem(g) <= 226 * 1024;  // (+ the static mbarriers)
}
size_t lstm_seq_ws(const Geo &g, int64_t batch) {
  return (size_t)4 * batch * g.q * 4 + (size_t)4 * batch * (g.s * g.rank + 4) * 4 + (size_t)2 * batch * g.q * 4 + 256;
  // gh (4 B H) | P (4 B (K2 + 4)) | c, h (2 B H) | barrier
}

int lstm_seq(const Geo &g, int64_t T, int64_t batch, const void *const *gx, const float *const *xf,
             const float *const *wf, const float *const *bias, void *out, char *ws, cudaStream_t st) {
  if (T == 0 || batch == 0) return DT_OK;
  SeqArgs a;
  for (int i = 0; i < 4; ++i) {
    a.xf[i] = xf[i]; a.wf[i] = wf[i]; a.bias[i] = bias ? bias[i] : nullptr;
    a.gx[i] = reinterpret_cast<const __nv_bfloat16 *>(gx[i]);
  }
  a.T = (int)T; a.B = (int)batch; a.H = (int)g.q; a.n = (int)g.n; a.R = (int)g.rank;
  a.s = (int)g.s; a.K2 = (int)(g.s * g.rank);
  a.vec = 1;
  for (int i = 0; i < 4; ++i) a.vec &= (reinterpret_cast<uintptr_t>(gx[i]) & 7) == 0;
  char *cur = ws;
  a.gh = reinterpret_cast<float *>(cur); cur += (size_t)4 * batch * g.q * 4;
  a.Pld = a.K2 + 4;
  a.P = reinterpret_cast<float *>(cur); cur += (size_t)4 * batch * a.Pld * 4;
  a.c = reinterpret_cast<float *>(cur); cur += (size_t)batch * g.q * 4;
  a.h = reinterpret_cast<float *>(cur); cur += (size_t)batch * g.q * 4;
  a.bar = reinterpret_cast<unsigned *>(cur);
  a.out = reinterpret_cast<__nv_bfloat16 *>(out);
  DT_CUDA_CHECK(cudaMemsetAsync(a.c, 0, (size_t)2 * batch * g.q * 4, st));  // c(-1) = h(-1) = 0
  DT_CUDA_CHECK(cudaMemsetAsync(a.bar, 0, 256, st));
  size_t smem = lstm_seq_smem(g);
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(k_lstm_seq<false>), 226 * 1024)) return rc;
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int unitsP = 4 * a.s * ((a.B + 15) / 16), unitsB = 4 * ((a.H + 63) / 64);
  int grid = std::min(nsm, std::max(unitsP, unitsB));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute coop[1], clus[1];
  coop[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: grid barriers are safe
  coop[0].val.cooperative = 1;
  cfg.attrs = coop;
  cfg.numAttrs = 1;
  // Fused gate-cluster form (k_lstm_seq<true>): one gate tile per CTA, the four gates of a
  // 64-column block in one cluster. Needs whole blocks, a CTA per unit, vectorizable gx, the
  // 16 KB exchange buffer, and every cluster resident at once (the grid barriers spin).
  // DEEPTHIN_LSTM_FUSED=0 keeps the three-phase form (A/B runs; both are complete).
  const char *fenv = getenv("DEEPTHIN_LSTM_FUSED");  // read per call (tests flip it)
  const bool want_fused = !(fenv && atoi(fenv) == 0);
  bool fused = want_fused && a.H % 64 == 0 && unitsB <= nsm && unitsP <= unitsB && a.vec &&
               smem + 16384 <= 226 * 1024;
  cudaLaunchConfig_t fc = cfg;
  if (fused) {
    if (int rc = set_smem_limit(reinterpret_cast<const void *>(k_lstm_seq<true>), 226 * 1024)) return rc;
    fc.gridDim = dim3((unsigned)unitsB);
    fc.dynamicSmemBytes = smem + 16384;
    // A plain cluster launch, not a cooperative one: ncu refuses to profile a cooperative
    // cluster launch (LaunchFailed), and the occupancy query below already establishes what
    // the cooperative attribute would — every cluster fits on the device at once, so the
    // spinning grid barriers cannot starve an unscheduled CTA (work of other streams only
    // delays residency; nothing else waits on this kernel).
    clus[0].id = cudaLaunchAttributeClusterDimension;
    clus[0].val.clusterDim.x = 4;
    clus[0].val.clusterDim.y = 1;
    clus[0].val.clusterDim.z = 1;
    fc.attrs = clus;
    fc.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k_lstm_seq<true>, &fc) != cudaSuccess || ncl < unitsB / 4) {
      cudaGetLastError();
      fused = false;
    }
  }
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_LSTM_TRACE") != 0;
  a.trace = nullptr;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&a.trace, 64 * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(a.trace, 0, 64 * 8, st));
  }
  if (fused && cudaLaunchKernelEx(&fc, k_lstm_seq<true>, a) != cudaSuccess) {
    cudaGetLastError();  // cluster launch refused: the three-phase form (cooperative launch)
    fused = false;
  }
  if (!fused) DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_lstm_seq<false>, a));
  if (tracing) {
    unsigned long long h[64];
    DT_CUDA_CHECK(cudaMemcpyAsync(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost, st));
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFree(a.trace);
    for (int t = 0; t < 8; ++t)
      fprintf(stderr, "lstm step %d: P %.2f  bar %.2f  G %.2f (stage %.2f tile %.2f)  bar %.2f  cell %.2f  bar %.2f us\n", t,
              t ? (h[t * 8] - h[t * 8 - 3]) * 1e-3 : 0.0, (h[t * 8 + 1] - h[t * 8]) * 1e-3,
              (h[t * 8 + 2] - h[t * 8 + 1]) * 1e-3, (h[t * 8 + 6] - h[t * 8 + 1]) * 1e-3,
              (h[t * 8 + 7] - h[t * 8 + 6]) * 1e-3, (h[t * 8 + 3] - h[t * 8 + 2]) * 1e-3,
              (h[t * 8 + 4] - h[t * 8 + 3]) * 1e-3, (h[t * 8 + 5] - h[t * 8 + 4]) * 1e-3);
  }
  return check_launch("lstm_seq");
}

}  // namespace dt
