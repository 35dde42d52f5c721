// Two-phase tensor-core forward — the default bf16 path for every geometry (kernel.py:222-293
// computes the same y = act(x @ W + b) on the CPU; W is factor.py:87-93's re-layout of
// I = xf @ wf).
//
// Phase 1, k_regen_wt: W^T (r_dim x ldw bf16, ldw = round_up(q, 8)) from the factors. Row j of
// W^T is the flat slice I.ravel()[j*q : (j+1)*q] (factor.py:87-93), so with ldw == q the
// buffer IS I.ravel()[:q*r_dim] and each thread stores its 8 consecutive outputs as one
// 16-byte write. W^T is 2*q*r_dim bytes — 1.8 MB at BASELINE config 2 — so it lives in L2
// between the two phases; the layer's parameters in HBM stay the factors.
//
// Phase 2, k_tc_gemm: persistent warp-specialised tcgen05 GEMM, launched with programmatic
// dependent launch so its prologue (barriers, TMEM, descriptor prefetch, the first x stages)
// overlaps phase 1. Tile = 128 output columns (UMMA M, TMEM lanes) x 256 batch rows (UMMA N);
// operands arrive by TMA in 128B-swizzled K-major layout (W^T resident per column block with
// x multicast across a cluster, or both streamed; see GemmParams) through an S-deep mbarrier
// stage ring. Accumulators double-buffer in TMEM (2 x 256
// columns) so the epilogue of tile t overlaps the MMAs of tile t+1. Epilogue: lanes are output
// columns and TMEM columns batch rows, so every warp store writes 32 consecutive outputs of
// one batch row (coalesced), fused with bias + activation.
//
// Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (one lane), warps 2.. epilogue.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <mutex>
#include <unordered_map>
#include <vector>

#include <cooperative_groups.h>

#include "act.cuh"
#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

constexpr int GM = 128;  // output columns per tile (UMMA M)
#ifndef DT_GEMM_GN
#define DT_GEMM_GN 256
#endif
constexpr int GN = DT_GEMM_GN;  // batch rows per tile (UMMA N; N = 256 runs the MMA at ~88% of peak)
constexpr int GK = 64;   // K per stage: one 128-byte swizzle row of bf16
constexpr uint32_t kABytes = GM * GK * 2;  // one W^T k-block (16 KB)
constexpr uint32_t kXBytes = GN * GK * 2;  // one x k-block (32 KB)
#ifndef DT_GEMM_EPI_WARPS
#define DT_GEMM_EPI_WARPS 8
#endif
constexpr int YDT_MSE = 7;  // epilogue "output type": the fused MSE gradient (see GemmParams)
constexpr int kEpiWarps = DT_GEMM_EPI_WARPS;  // multiple of 4 (one per TMEM lane quarter)
constexpr int kEpiParts = kEpiWarps / 4;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kSmemMax = 227 * 1024;
constexpr int kTrace = 48;
static_assert(kEpiWarps % 4 == 0, "epilogue warps cover the 4 TMEM lane quarters");

// Phase-1 tile geometry (see regen_tile) and arguments.
constexpr int RG_R = 32, RG_C = 128, RG_K = 32;  // standalone tile: 32 rows x 128 columns
constexpr int RG_RMAX = 64;                       // fused kernel: up to 64-row tiles
struct RegenArgs {
  int64_t q, r_dim, ldw;
  int rank, n, a_rows, f_dtype;
  int chain;  // pipelined forward: complete only after the previous grid (griddepcontrol.wait)
  int x_ext;  // pipelined forward with external inputs: x is never written by an in-flight grid
  const void *xf, *wf;
  __nv_bfloat16 *wt;
  // hilo: W^T as a bf16 hi + lo pair, row j = [hi(W^T[j, :]) | pad | lo(W^T[j, :]) | pad] with
  // halves of qp columns (qp = round_up(q, 64)), so one GEMM over K = 2 qp against x (read
  // twice through a wrapping tensor map) accumulates x W_hi + x W_lo: ~16 significant bits of W
  int hilo, qp;
  int tiles_x, tiles_y;  // phase-1 tile grid (filled by launch_regen_wt)
};
struct RegenSmem {
  float xt[RG_K][RG_RMAX + 4];  // +4: the transposing stores are 4-way, not 32-way, conflicted
  float ws[RG_K][RG_C];
};

// Two operand schedules:
//  * wres (W resident, K <= 512): a cluster of csize CTAs owns csize consecutive column blocks;
//    each CTA loads its W^T block once (KB x 16 KB) and the cluster walks batch tiles together,
//    each CTA TMA-loading 1/csize of every x stage and multicasting it to the whole cluster —
//    L2 serves every x tile once per cluster. (Streaming both operands per tile moved 10.5
//    bytes of operands per output through L2, which capped the kernel at the L2 throughput.)
//  * stream (larger K): W^T and x k-blocks both stream through the stage ring, csize = 1.
// Work items are (column group, batch tile), column-group-major; cluster c takes the balanced
// contiguous range [c*items/ncl, (c+1)*items/ncl), so a cluster changes W block at most a few
// times.
struct GemmParams {
  int64_t batch;
  int r_dim, ldy, KB, n_jb, n_bt, n_jg, items, ncl;
  int cpj;  // clusters per column group (> 0: every cluster stays in one group), else 0
  int wres, csize, S;
  uint32_t off_x, stage_bytes, off_bar;
  const float *bias;
  void *y;
  float arg;
  // YDT == YDT_MSE epilogue: y holds grad = scale * (z - target) (fp32), and every epilogue
  // warp writes the fp64 sum of (z - target)^2 over its share of a tile to
  // loss_part[(item * csize + crank) * kEpiWarps + warp - 2]
  const float *target;
  double scale;
  double *loss_part;
  // fused (cooperative launch): phase 1 runs inside the GEMM kernel on the epilogue warps of
  // every CTA (tiles rg_ux x rg_uy), then a grid-wide barrier, then the GEMM
  int fused, rg_ux, rg_uy, rg_rows;
  uint32_t off_rg;  // phase-1 staging (the W block area, or x stages not yet in flight)
  // wgen: no phase 1 — each pair CTA generates its own W^T block in shared memory from the
  // factors (p.rg.xf / p.rg.wf), staged at off_fs (x stages not in flight yet)
  int wgen;
  uint32_t off_fs;
  RegenArgs rg{};
  int chain;  // pipelined forward: let the next call's phase 1 launch right away
  // x may be loaded before griddepcontrol.wait: not chained (the grids ahead of phase 1 have
  // completed), or chained with inputs the caller declared external (DT_PIPELINE_EXTERNAL_X).
  // A chained forward whose x is the previous layer's output waits first: that layer's GEMM
  // may still be writing it (it signals its dependents right after its prologue).
  int x_early;
  int dbg;  // DEEPTHIN_DBG_GEMM (timing experiments only): 1 skip y stores, 2 x loads after the first S stages skipped, 4 skip TMEM loads
  unsigned long long *trace;  // DEEPTHIN_TC_TRACE: per-CTA globaltimer stamps
};

// Items of cluster cid. With cpj > 0 clusters per column group, each cluster takes a balanced
// share of one group's batch tiles, so its W block is loaded once; else balanced contiguous
// ranges of the group-major item order (a range may cross a group: the W block is reloaded).
__device__ __forceinline__ void item_range(const GemmParams &p, int cid, int &beg, int &end) {
  if (p.cpj > 0) {
    const int jg = cid / p.cpj, sub = cid % p.cpj;
    beg = jg * p.n_bt + (int)((int64_t)sub * p.n_bt / p.cpj);
    end = jg * p.n_bt + (int)((int64_t)(sub + 1) * p.n_bt / p.cpj);
  } else {
    beg = (int)((int64_t)cid * p.items / p.ncl);
    end = (int)((int64_t)(cid + 1) * p.items / p.ncl);
  }
}

__device__ __forceinline__ void gtrace(const GemmParams &p, int slot) {
  if (p.trace && slot < kTrace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    p.trace[(size_t)blockIdx.x * kTrace + slot] = t;
  }
}

// ---- phase 1 --------------------------------------------------------------------------------
template <typename FT>
__device__ __forceinline__ float ldf(const FT *p) {
  if constexpr (std::is_same<FT, float>::value)
    return __ldg(p);
  else
    return __bfloat162float(*p);
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// fp32 bits -> tf32 hi (RNA) + tf32 lo (the RNA of the remainder): hi + lo carries ~21 bits
__device__ __forceinline__ void split_tf32(uint32_t bits, uint32_t &hi, uint32_t &lo) {
  const float v = __uint_as_float(bits);
  hi = to_tf32(v);
  lo = to_tf32(v - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_m16n8k8_tf32(float (&d)[4], const uint32_t (&a)[4],
                                                 uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// CTA tile: RG_R aux rows x RG_C aux columns of I = xf @ wf, the factors staged through shared
// memory RG_K ranks at a time (coalesced loads, all in flight together; xf transposed so a
// thread's 8 rows at one rank are 32 contiguous bytes). Thread: 8 consecutive rows
// (RG_E * warp ..) x 4 consecutive columns (4 * lane ..): per rank one 128-bit load of wf (a
// warp reads 512 distinct bytes) and one broadcast 128-bit load of xf feed 16 FMAs. Only rows
// a < a_rows = ceil(q*r_dim / n) feed W (the tail of I past q*r_dim is discarded, factor.py:91).

// One regeneration tile (row block bx, column block by) by 256 threads (tid 0..255); `sync`
// is the barrier over those threads.
template <typename FT, int R, typename Sync>
__device__ __forceinline__ void regen_tile(const RegenArgs &g, int tid, int bx, int by,
                                           RegenSmem &sm, Sync sync) {
  constexpr int RG_E = R / 8;  // rows per thread (8 warps)
  static_assert(R % 32 == 0 && R <= RG_RMAX, "tile rows");
  const FT *xf = reinterpret_cast<const FT *>(g.xf);
  const FT *wf = reinterpret_cast<const FT *>(g.wf);
  const int lane = tid % 32, wrp = tid / 32;
  const int a0 = bx * R, c0 = by * RG_C;
  const int rank = g.rank, n = g.n, a_rows = g.a_rows;
  float acc[RG_E][4];
#pragma unroll
  for (int e = 0; e < RG_E; ++e)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[e][c] = 0.f;
  for (int k0 = 0; k0 < rank; k0 += RG_K) {
    const int kc = min(RG_K, rank - k0);
    // every load of the chunk issued before the first shared-memory store (one latency)
    constexpr int NX = R * RG_K / 256, NW = RG_K * RG_C / 256;
    float xv[NX], wv[NW];
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u, r = e / RG_K, k = e % RG_K;
      xv[u] = (a0 + r < a_rows && k < kc) ? ldf(xf + (int64_t)(a0 + r) * rank + k0 + k) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u, k = e / RG_C, c = e % RG_C;
      wv[u] = (k < kc && c0 + c < n) ? ldf(wf + (int64_t)(k0 + k) * n + c0 + c) : 0.f;
    }
    sync();  // the previous chunk / tile is done with the staging buffers
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u;
      sm.xt[e % RG_K][e / RG_K] = xv[u];
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u;
      sm.ws[e / RG_C][e % RG_C] = wv[u];
    }
    sync();
    // 8 ranks per unrolled group (the staged chunk is zero-padded to a multiple of 8): the
    // shared loads of later ranks issue ahead of the FMAs of earlier ones
    for (int k8 = 0; k8 < kc; k8 += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = k8 + kk;
        const float4 w4 = *reinterpret_cast<const float4 *>(&sm.ws[k][4 * lane]);
        const float wk[4] = {w4.x, w4.y, w4.z, w4.w};
        float xk[RG_E];
#pragma unroll
        for (int h = 0; h < RG_E / 4; ++h) {
          const float4 x4 = *reinterpret_cast<const float4 *>(&sm.xt[k][RG_E * wrp + 4 * h]);
          xk[4 * h] = x4.x; xk[4 * h + 1] = x4.y; xk[4 * h + 2] = x4.z; xk[4 * h + 3] = x4.w;
        }
#pragma unroll
        for (int e = 0; e < RG_E; ++e)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[e][c] = fmaf(xk[e], wk[c], acc[e][c]);
      }
    }
  }
  const int64_t q = g.q, total = q * g.r_dim;
  const bool flat = g.ldw == q && (n & 3) == 0;  // W^T == I.ravel(): 8-byte stores
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
      *reinterpret_cast<uint2 *>(g.wt + f0) =
          make_uint2(*reinterpret_cast<uint32_t *>(&v0), *reinterpret_cast<uint32_t *>(&v1));
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int64_t f = f0 + c;
        if (cc + c < n && f < total) {
          const int64_t j = f / q, i = f - j * q;
          g.wt[j * g.ldw + i] = __float2bfloat16_rn(acc[e][c]);
        }
      }
    }
  }
}

// Tensor-core form of one regeneration tile (RG_R x RG_C): the products on the warp-level
// tensor cores (mma.sync m16n8k8, tf32 operands rounded from the factors — bf16-valued factors
// are exact — fp32 accumulate); staging strides make the fragment reads conflict-free. Warp w:
// m-tile w & 1, n-tiles 4*(w >> 1) .. +3. Accumulator pairs go straight to W^T (= I.ravel()
// when ldw == q) as 4-byte bf16x2 stores.
struct RegenSmemTC {
  uint32_t xs[RG_R][RG_K + 4];   // fp32 bits (split to tf32 hi/lo at fragment load); row stride = 4 (mod 8): conflict-free A reads
  uint32_t ws[RG_K][RG_C + 8];   // row stride / 8 odd: conflict-free B reads
};
template <typename FT>
__device__ __forceinline__ void regen_tile_tc(const RegenArgs &g, int tid, int bx, int by,
                                              RegenSmemTC &sm) {
  static_assert(RG_R == 32 && RG_C == 128 && RG_K == 32, "warp tiling below");
  const FT *xf = reinterpret_cast<const FT *>(g.xf);
  const FT *wf = reinterpret_cast<const FT *>(g.wf);
  const int lane = tid % 32, w = tid / 32, gr = lane >> 2, tq = lane & 3;
  const int mt = w & 1, nt0 = 4 * (w >> 1);
  const int a0 = bx * RG_R, c0 = by * RG_C;
  const int rank = g.rank, n = g.n, a_rows = g.a_rows;
  float d[4][4];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int e = 0; e < 4; ++e) d[t][e] = 0.f;
  for (int k0 = 0; k0 < rank; k0 += RG_K) {
    const int kc = min(RG_K, rank - k0);
    constexpr int NX = RG_R * RG_K / 256, NW = RG_K * RG_C / 256;
    float xv[NX], wv[NW];
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u, r = e / RG_K, k = e % RG_K;
      xv[u] = (a0 + r < a_rows && k < kc) ? ldf(xf + (int64_t)(a0 + r) * rank + k0 + k) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u, k = e / RG_C, c = e % RG_C;
      wv[u] = (k < kc && c0 + c < n) ? ldf(wf + (int64_t)(k0 + k) * n + c0 + c) : 0.f;
    }
    if (k0 > 0) __syncthreads();  // the previous chunk's fragments are read
    // smem keeps the raw fp32 bits; fragments are split at load time
#pragma unroll
    for (int u = 0; u < NX; ++u) {
      const int e = tid + 256 * u;
      sm.xs[e / RG_K][e % RG_K] = __float_as_uint(xv[u]);
    }
#pragma unroll
    for (int u = 0; u < NW; ++u) {
      const int e = tid + 256 * u;
      sm.ws[e / RG_C][e % RG_C] = __float_as_uint(wv[u]);
    }
    __syncthreads();
    for (int ks = 0; ks < (kc + 7) / 8; ++ks) {
      uint32_t ah[4], al[4];
      const uint32_t *xr = &sm.xs[mt * 16 + gr][ks * 8 + tq];
      const uint32_t araw[4] = {xr[0], xr[8 * (RG_K + 4)], xr[4], xr[8 * (RG_K + 4) + 4]};
#pragma unroll
      for (int i = 0; i < 4; ++i) split_tf32(araw[i], ah[i], al[i]);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t *wr = &sm.ws[ks * 8 + tq][(nt0 + t) * 8 + gr];
        uint32_t bh0, bl0, bh1, bl1;
        split_tf32(wr[0], bh0, bl0);
        split_tf32(wr[4 * (RG_C + 8)], bh1, bl1);
        if constexpr (std::is_same<FT, float>::value) {
          // split TF32: hi*lo + lo*hi + hi*hi, ~fp32-accurate products, so the bf16 W^T is
          // the RNE of the (near-)exact W — the rounding the bf16 contract states
          mma_m16n8k8_tf32(d[t], ah, bl0, bl1);
          mma_m16n8k8_tf32(d[t], al, bh0, bh1);
        }
        mma_m16n8k8_tf32(d[t], ah, bh0, bh1);  // bf16 factors: exact in tf32, lo == 0
      }
    }
  }
  const int64_t q = g.q, total = q * g.r_dim;
  if (g.hilo) {
    // [hi | lo] rows: each accumulator pair (an even flat index f, so both in row f / q when q
    // is even) -> one bf16x2 hi store and one bf16x2 lo store
    const int64_t ld2 = 2 * (int64_t)g.qp;
    const bool pairs = (q & 1) == 0 && (n & 1) == 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int c = c0 + (nt0 + t) * 8 + 2 * tq;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = a0 + mt * 16 + gr + 8 * h;
        if (a >= a_rows || c >= n) continue;
        const float v0 = d[t][2 * h], v1 = d[t][2 * h + 1];
        const int64_t f = (int64_t)a * n + c;
        if (pairs && c + 1 < n && f + 2 <= total) {
          const int64_t j = f / q, i = f - j * q;
          const __nv_bfloat162 hv = __floats2bfloat162_rn(v0, v1);
          const __nv_bfloat162 lv = __floats2bfloat162_rn(v0 - __low2float(hv), v1 - __high2float(hv));
          *reinterpret_cast<__nv_bfloat162 *>(g.wt + j * ld2 + i) = hv;
          *reinterpret_cast<__nv_bfloat162 *>(g.wt + j * ld2 + g.qp + i) = lv;
        } else {
          for (int e = 0; e < 2; ++e) {
            const int64_t fe = f + e;
            if (c + e < n && fe < total) {
              const int64_t j = fe / q, i = fe - j * q;
              const float v = e ? v1 : v0;
              const __nv_bfloat16 hb = __float2bfloat16_rn(v);
              g.wt[j * ld2 + i] = hb;
              g.wt[j * ld2 + g.qp + i] = __float2bfloat16_rn(v - __bfloat162float(hb));
            }
          }
        }
      }
    }
    return;
  }
  const bool flat = g.ldw == q && (n & 1) == 0;  // W^T == I.ravel(): bf16x2 stores
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int c = c0 + (nt0 + t) * 8 + 2 * tq;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int a = a0 + mt * 16 + gr + 8 * h;
      if (a >= a_rows || c >= n) continue;
      const float v0 = d[t][2 * h], v1 = d[t][2 * h + 1];
      const int64_t f = (int64_t)a * n + c;
      if (flat && c + 1 < n && f + 2 <= total) {
        *reinterpret_cast<__nv_bfloat162 *>(g.wt + f) = __floats2bfloat162_rn(v0, v1);
      } else {
        for (int e = 0; e < 2; ++e) {
          const int64_t fe = f + e;
          if (c + e < n && fe < total) {
            const int64_t j = fe / q, i = fe - j * q;
            g.wt[j * g.ldw + i] = __float2bfloat16_rn(e ? v1 : v0);
          }
        }
      }
    }
  }
}

// Persistent over the tiles (1-D grid, tile t -> (t % tiles_x, t / tiles_x)): a pipelined launch
// caps the grid at one CTA per SM, so every CTA of this grid is resident beside the previous
// forward's GEMM (22 KB of shared memory fit next to its stages). With more CTAs than SMs the
// second wave could only start once the first wave left — which waits for that GEMM's end
// (griddepcontrol.wait below) — and ran exposed between the two GEMMs (config 2: ~7 us a step).
__global__ void __launch_bounds__(256) k_regen_wt(const RegenArgs g) {
  griddep_launch_dependents();  // the GEMM may start its prologue now
  __shared__ __align__(16) RegenSmemTC sm;
  if (g.hilo && g.qp > g.q) {
    // zero the pad columns [q, qp) of both halves (the GEMM multiplies them by x's zero fill;
    // workspace garbage could be NaN), rows strided over the CTAs
    const int64_t ld2 = 2 * (int64_t)g.qp;
    const int pad = g.qp - (int)g.q;
    for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < g.r_dim * 2 * pad;
         e += (int64_t)gridDim.x * 256) {
      const int64_t j = e / (2 * pad);
      const int k = (int)(e - j * 2 * pad);
      g.wt[j * ld2 + (k < pad ? 0 : g.qp) + g.q + (k % pad)] = __float2bfloat16_rn(0.f);
    }
  }
  const int tiles = g.tiles_x * g.tiles_y;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    if (t != (int)blockIdx.x) __syncthreads();  // the previous tile's fragments are read
    const int by = t / g.tiles_x, bx = t - by * g.tiles_x;
    if (g.f_dtype == DT_F32)
      regen_tile_tc<float>(g, threadIdx.x, bx, by, sm);
    else
      regen_tile_tc<__nv_bfloat16>(g, threadIdx.x, bx, by, sm);
  }
  // pipelined: this grid overlapped the previous forward's GEMM (it writes the other W^T
  // slot); completing only after that grid keeps the next GEMM — which waits on this grid —
  // ordered after it, so W^T slots and outputs are reused safely.
  if (g.chain) griddep_wait();
}

// Launch phase 1 (fills g.tiles_x / tiles_y; see k_regen_wt for the grid cap when pipelined).
int launch_regen_wt(RegenArgs rg, cudaStream_t st) {
  rg.tiles_x = (rg.a_rows + RG_R - 1) / RG_R;
  rg.tiles_y = (rg.n + RG_C - 1) / RG_C;
  int tiles = rg.tiles_x * rg.tiles_y;
  if (rg.chain) {
    int dev = 0, nsm = 148;
    DT_CUDA_CHECK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // the same shared-memory carveout as the GEMM it runs beside (an SM switches its L1 /
    // shared split only when idle: with the default carveout these CTAs waited for the GEMM's
    // CTAs to leave)
    if (int rc = prefer_max_smem_carveout(reinterpret_cast<const void *>(k_regen_wt))) return rc;
    cudaLaunchConfig_t rcfg{};
    rcfg.gridDim = dim3((unsigned)std::max(1, std::min(tiles, nsm)));
    rcfg.blockDim = dim3(256);
    rcfg.stream = st;
    cudaLaunchAttribute ra[1];
    ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ra[0].val.programmaticStreamSerializationAllowed = 1;
    rcfg.attrs = ra;
    rcfg.numAttrs = 1;
    DT_CUDA_CHECK(cudaLaunchKernelEx(&rcfg, k_regen_wt, rg));
  } else {
    k_regen_wt<<<(unsigned)std::max(1, tiles), 256, 0, st>>>(rg);
  }
  return check_launch("regen_wt");
}

// ---- phase 2 --------------------------------------------------------------------------------
// EL: 0 = bf16 operands (kind::f16, 64 elements per 128-byte k-block), 1 = fp32 operands
// (kind::tf32, 32 elements per k-block). Shared-memory bytes and descriptors are identical.
template <int YDT, int ACT, int EL>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
              const GemmParams p) {
  constexpr int GKE = EL ? 32 : 64;  // elements per 128-byte k-block
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *wfull = tempty + 2, *wfree = wfull + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(wfree + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int cs = p.csize;
  const uint32_t crank = cs > 1 ? cluster_ctarank() : 0u;
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  const int cid = (int)blockIdx.x / cs;
  int beg, end;
  item_range(p, cid, beg, end);
  // item -> (column block, first batch row)
  auto jb_of = [&](int it) { return (it / p.n_bt) * cs + (int)crank; };
  auto b0_of = [&](int it) { return (it % p.n_bt) * GN; };

  if (threadIdx.x == 0) {
    gtrace(p, 0);
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cs); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], kEpiWarps); }
    mbar_init(wfull, 1);
    mbar_init(wfree, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tm_w); tma_prefetch_desc(&tm_x); }
  if (warp == 1) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) gtrace(p, 1);
  if (p.chain) griddep_launch_dependents();  // the next forward's phase 1 may start

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint32_t slice_rows = GN / cs, slice_bytes = kXBytes / cs;
      int stage = 0, jg_cur = -1, u = 0;
      uint32_t phase = 0, wf_phase = 0;
      // x does not depend on phase 1: the first stages' x loads go out before griddep_wait
      // (unless x may still be in flight from a chained predecessor, see x_early).
      if (!p.x_early) griddep_wait();
      const int pre = min(p.S, p.KB);
      for (int it = beg; it < end; ++it) {
        const int jg = it / p.n_bt, j0 = jb_of(it) * GM, b0 = b0_of(it);
        if (p.wres && jg != jg_cur && jg_cur >= 0) {  // next W block: old one fully consumed
          mbar_wait(wfree, wf_phase);
          wf_phase ^= 1;
          mbar_arrive_expect_tx(wfull, (uint32_t)p.KB * kABytes);
          for (int kb = 0; kb < p.KB; ++kb)
            tma_load_2d(smem + kb * kABytes, &tm_w, wfull, kb * GKE, j0);
        }
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);  // every cluster CTA released this stage
          if (u < 10) gtrace(p, 34 + u);
          uint8_t *st = smem + p.off_x + stage * p.stage_bytes;
          mbar_arrive_expect_tx(&full[stage], p.stage_bytes);
          uint8_t *xdst = p.wres ? st : st + kABytes;
          if (cs == 1)
            tma_load_2d(xdst, &tm_x, &full[stage], kb * GKE, b0);
          else
            tma_load_2d_mc(xdst + crank * slice_bytes, &tm_x, &full[stage], kb * GKE,
                           b0 + (int)(crank * slice_rows), cmask);
          if (!p.wres && u >= pre) tma_load_2d(st, &tm_w, &full[stage], kb * GKE, j0);
          ++u;
          if (u == pre) {  // W^T is phase 1's output
            griddep_wait();
            gtrace(p, 2);
            if (p.wres) {
              mbar_arrive_expect_tx(wfull, (uint32_t)p.KB * kABytes);
              for (int k = 0; k < p.KB; ++k)
                tma_load_2d(smem + k * kABytes, &tm_w, wfull, k * GKE, j0);
            } else {
              for (int v = 0; v < pre; ++v)  // the W halves of the stages already in flight
                tma_load_2d(smem + p.off_x + v * p.stage_bytes, &tm_w, &full[v], v * GKE, j0);
            }
          }
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        jg_cur = jg;
      }
      gtrace(p, 3);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_f32acc(GM, GN, EL ? 2 : 1);
      const uint32_t s0 = smem_u32(smem);
      int stage = 0, acc = 0, jg_cur = -1;
      uint32_t phase = 0, aphase = 0, wphase = 0;
      for (int it = beg; it < end; ++it) {
        const int jg = it / p.n_bt;
        if (p.wres && jg != jg_cur) {  // this W block landed
          mbar_wait(wfull, wphase);
          wphase ^= 1;
          jg_cur = jg;
        }
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * GN);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&full[stage], phase);
          if (it == beg) gtrace(p, 20 + kb);
          tc_fence_after();
          const uint32_t st = s0 + p.off_x + (uint32_t)stage * p.stage_bytes;
          const uint32_t a_s = p.wres ? s0 + (uint32_t)kb * kABytes : st;
          const uint32_t b_s = p.wres ? st : st + kABytes;
#pragma unroll
          for (int k = 0; k < GK / 16; ++k)
            if constexpr (EL)
              mma_tf32_ss(d, smem_desc(a_s + k * 32, 16, 1024, SL_SW128),
                          smem_desc(b_s + k * 32, 16, 1024, SL_SW128), idesc, (kb | k) != 0);
            else
              mma_bf16_ss(d, smem_desc(a_s + k * 32, 16, 1024, SL_SW128),
                          smem_desc(b_s + k * 32, 16, 1024, SL_SW128), idesc, (kb | k) != 0);
          if (cs == 1)
            mma_commit(&empty[stage]);
          else  // every producer of the cluster multicasts into this stage
            mma_commit_mc(&empty[stage], cmask);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (p.wres && it + 1 < end && (it + 1) / p.n_bt != jg) mma_commit(wfree);
        gtrace(p, 4 + min(it - beg, 7));
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int wq = warp & 3;          // TMEM lane quarter this warp may read
    const int part = (warp - 2) / 4;  // which 32-row groups of the tile
    using OutT = typename std::conditional<YDT == DT_BF16, __nv_bfloat16, float>::type;
    int acc = 0;
    uint32_t aphase = 0;
    double sq = 0.0;  // YDT_MSE: this thread's share of the tile's squared error
    for (int it = beg; it < end; ++it) {
      const int j = jb_of(it) * GM + 32 * wq + lane;
      const int64_t b0 = b0_of(it);
      const bool jok = j < p.r_dim;
      const float bias_j = (p.bias && jok) ? __ldg(p.bias + j) : 0.f;
      const int nrows = (int)min((int64_t)GN, p.batch - b0);
      mbar_wait(&tfull[acc], aphase);
      if (threadIdx.x == 64 && it - beg < 2) gtrace(p, 44 + (it - beg));
      tc_fence_after();
      for (int c32 = part; c32 < GN / 32; c32 += kEpiParts) {
        if (32 * c32 >= nrows) break;
        uint32_t v[32];
        if (kTimingSwitches && (p.dbg & 4)) {
          for (int r = 0; r < 32; ++r) v[r] = 0;
        } else {
          tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(acc * GN + c32 * 32), v);
          tmem_ld_wait();
        }
        if (jok && !(kTimingSwitches && (p.dbg & 1))) {
          OutT *yp = reinterpret_cast<OutT *>(p.y) + (b0 + 32 * c32) * p.ldy + j;
          const int rmax = nrows - 32 * c32;
          if constexpr (YDT == YDT_MSE) {  // grad = scale * (z - t), sum (z - t)^2
            // fp32 per element (fp64 math per element made this epilogue the bottleneck), the
            // 32-row chunk's fp32 sum folded into the thread's fp64 total in a fixed order
            const float *tp = p.target + (b0 + 32 * c32) * p.ldy + j;
            const float sc = (float)p.scale;
            float tv[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) tv[r] = r < rmax ? __ldg(tp + (int64_t)r * p.ldy) : 0.f;
            float csq = 0.f;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              if (r < rmax) {
                const float dz = (__uint_as_float(v[r]) + bias_j) - tv[r];
                *yp = sc * dz;
                csq = fmaf(dz, dz, csq);
              }
              yp += p.ldy;
            }
            sq += (double)csq;
          } else if (rmax >= 32) {  // full chunk: no per-row predicate, pointer bumps only
            const int64_t ld = p.ldy;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
              if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
              yp += ld;
            }
          } else {
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              if (r < rmax) {
                const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
                if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
              }
              yp += p.ldy;
            }
          }
        }
      }
      if constexpr (YDT == YDT_MSE) {  // fixed-order warp reduction -> one partial per warp
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) p.loss_part[((int64_t)it * cs + crank) * kEpiWarps + (warp - 2)] = sq;
        sq = 0.0;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&tempty[acc]);  // this warp's TMEM reads are done
      if (threadIdx.x == 64) gtrace(p, 12 + min(it - beg, 7));
      if (threadIdx.x == kGemmThreads - 32 && it - beg < 2) gtrace(p, 46 + (it - beg));
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // no CTA leaves while peers may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ---- in-CTA W block generation (p.wgen) ------------------------------------------------------
// W^T rows [j0, j0 + 128) of one column block, bf16, written straight into the 128B-swizzled
// K-major A-operand layout in shared memory, so no dense W exists outside the SM. The aux rows
// a_lo..a_hi that cover the block's flat range [j0*q, (j0+128)*q) are I = xf @ wf products on
// the warp-level tensor-core path (mma.sync m16n8k8, tf32 operands rounded from the fp32
// factors — bf16-valued factors are exact — fp32 accumulate), each accumulator element scattered
// to (j, i) = divmod(a*n + c - j0*q, q) (factor.py:87-93). Factor operands are staged as fp32
// through shared memory with strides that make the fragment reads bank-conflict-free.
// byte offset of W-block element (j, i): 64-column k-blocks of 128 rows x 128 B, 16-byte chunks
// XOR-swizzled by (row mod 8) — the layout TMA SWIZZLE_128B produces for the GEMM's A operand
__device__ __forceinline__ uint32_t wsw_off(uint32_t j, uint32_t i) {
  return (i >> 6) * kABytes + j * 128u + ((((i >> 3) & 7u) ^ (j & 7u)) << 4) + (i & 7u) * 2u;
}
struct WgenGeo {  // host-computed staging geometry for one plan
  int n_ks, xs_stride, ws_stride, max_mt;
};
__host__ __device__ inline WgenGeo wgen_geo(int q, int rank, int n) {
  WgenGeo w;
  w.n_ks = (rank + 7) / 8;
  w.xs_stride = 8 * w.n_ks + 4;  // = 4 mod 8: the 8 fragment rows hit distinct bank quads
  const int n_nt = (n + 7) / 8;
  w.ws_stride = 8 * (n_nt + 1 + ((n_nt + 1) % 2 == 0 ? 1 : 0));  // /8 odd: conflict-free
  // aux rows one 128-column block touches, rounded up to whole 16-row tiles
  const int64_t rows = ((int64_t)GM * q + n - 1) / n + 1;
  w.max_mt = (int)((rows + 15) / 16);
  return w;
}
__host__ __device__ inline uint32_t wgen_stage_bytes(int q, int rank, int n) {
  const WgenGeo w = wgen_geo(q, rank, n);
  return (uint32_t)(w.max_mt * 16 * w.xs_stride + w.n_ks * 8 * w.ws_stride) * 4u;
}

// Integer work here is latency-bound (8 warps, 2 per scheduler): the loops are division-free
// (warp-per-row staging, the flat offset of a row split once per m-tile and advanced by +8
// per n-tile) and two n-tiles are in flight per iteration.
template <typename FT>
__device__ void wgen_block(const GemmParams &p, int j0, uint8_t *smem, int tid) {
  const RegenArgs &g = p.rg;
  const int q = (int)g.q, n = g.n, rank = g.rank;
  const int jrows = max(0, min(GM, (int)g.r_dim - j0));
  const int KP = p.KB * GK;
  const WgenGeo wg = wgen_geo(q, rank, n);
  const int w = tid / 32, lane = tid % 32;
  // 1) zeros: the K padding [q8, KP) of every row (q8 = q rounded down to 8), rows >= jrows
  {
    const int q8 = q & ~7;
    for (int j = tid >> 3; j < GM; j += 32) {  // 8 threads per row
      const int i_start = j >= jrows ? 0 : q8;
      for (int i8 = i_start + 8 * (tid & 7); i8 < KP; i8 += 64) {
        if (j >= jrows || i8 >= q) {
          *reinterpret_cast<uint4 *>(smem + wsw_off(j, i8)) = make_uint4(0, 0, 0, 0);
        } else {  // the unit straddling q: only its tail
          for (int i = q; i < i8 + 8; ++i) *reinterpret_cast<uint16_t *>(smem + wsw_off(j, i)) = 0;
        }
      }
    }
  }
  if (tid == 0) gtrace(p, 28);
  if (jrows == 0) return;
  const int f_lo = j0 * q, f_span = jrows * q;  // flat range of the block (< 2^31: host check)
  const int a_lo = f_lo / n, a_hi = (f_lo + f_span - 1) / n;
  const int n_mt = (a_hi - a_lo + 16) / 16, n_nt = (n + 7) / 8, n_ks = wg.n_ks;
  const int XS = wg.xs_stride, WS = wg.ws_stride;
  uint32_t *xs = reinterpret_cast<uint32_t *>(smem + p.off_fs);  // tf32 bit patterns
  uint32_t *ws = xs + wg.max_mt * 16 * XS;
  // 2) stage xf rows a_lo.. (n_mt*16 x n_ks*8) and wf (n_ks*8 x n_nt*8) as tf32, zero padded;
  //    a warp per row, lanes along the contiguous dimension, loads batched ahead of the stores
  const FT *xf = reinterpret_cast<const FT *>(g.xf);
  const FT *wf = reinterpret_cast<const FT *>(g.wf);
  const int kx = n_ks * 8, cx = n_nt * 8;
  {
    constexpr int B = 8;
    const int rows = n_mt * 16;
    for (int r0 = w; r0 < rows; r0 += 8 * B) {
      float v[B][2];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int r = r0 + 8 * u, a = a_lo + r;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = lane + 32 * h;
          v[u][h] = (r < rows && a <= a_hi && k < rank) ? ldf(xf + (int64_t)a * rank + k) : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int r = r0 + 8 * u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = lane + 32 * h;
          if (r < rows && k < kx) xs[r * XS + k] = to_tf32(v[u][h]);
        }
      }
    }
    for (int k = w; k < kx; k += 8) {
      const bool kok = k < rank;
      for (int c0 = 0; c0 < cx; c0 += 32 * B) {
        float v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int c = c0 + lane + 32 * u;
          v[u] = (kok && c < n) ? ldf(wf + (int64_t)k * n + c) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          const int c = c0 + lane + 32 * u;
          if (c < cx) ws[k * WS + c] = to_tf32(v[u]);
        }
      }
    }
  }
  named_bar_sync(1, 256);
  if (tid == 0) gtrace(p, 29);
  // 3) tensor-core products + scatter; warp w owns n-tiles w, w+8, ... (two per iteration)
  const int gr = lane >> 2, tq = lane & 3;
  // 8 consecutive columns of a row land on 8 consecutive, 16-byte-aligned elements of one W
  // row: the quad's four bf16 pairs are gathered into one lane and stored as 16 bytes
  const bool vec8 = (q % 8) == 0 && (n % 8) == 0 && (f_lo % 8) == 0;
  auto split = [&](int rel, int &j, int &i) {  // rel >= 0
    j = rel / q;
    i = rel - j * q;
  };
  auto put1 = [&](int rel, uint16_t hb) {  // one element at flat offset rel (any range)
    if (rel < 0 || rel >= f_span) return;
    int j, i;
    split(rel, j, i);
    *reinterpret_cast<uint16_t *>(smem + wsw_off(j, i)) = hb;
  };
  // this lane's store row for the vector path: quad lane 0 stores row g, lane 1 row g + 8
  const int my_half = tq == 1 ? 8 : 0;
  for (int mt = 0; mt < n_mt; ++mt) {
    uint32_t af[8][4];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      if (ks < n_ks) {
        const uint32_t *xr = xs + (mt * 16 + gr) * XS + ks * 8 + tq;
        af[ks][0] = xr[0];
        af[ks][1] = xr[8 * XS];
        af[ks][2] = xr[4];
        af[ks][3] = xr[8 * XS + 4];
      }
    }
    const int ra = a_lo + mt * 16 + gr;
    const int rel_g = ra * n - f_lo, rel_g8 = (ra + 8) * n - f_lo;
    // the vector path's row: flat offset at column 0, split once; advanced per n-tile below
    const int my_row = ra + my_half, my_rel0 = my_half ? rel_g8 : rel_g;
    const bool my_rowok = my_row <= a_hi;
    int jv = 0, iv = 0;
    if (my_rel0 >= 0) split(my_rel0, jv, iv);
    for (int nt0 = w; nt0 < n_nt; nt0 += 16) {
      float d[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      const bool second = nt0 + 8 < n_nt;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks < n_ks) {
          const uint32_t *wr = ws + (ks * 8 + tq) * WS + nt0 * 8 + gr;
          mma_m16n8k8_tf32(d[0], af[ks], wr[0], wr[4 * WS]);
          if (second) mma_m16n8k8_tf32(d[1], af[ks], wr[64], wr[4 * WS + 64]);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !second) break;
        const int nt = nt0 + 8 * h, c0 = nt * 8;
        if (vec8 && c0 + 8 <= n) {
          __nv_bfloat162 hg = __floats2bfloat162_rn(d[h][0], d[h][1]);
          __nv_bfloat162 hg8 = __floats2bfloat162_rn(d[h][2], d[h][3]);
          const uint32_t w0 = *reinterpret_cast<uint32_t *>(&hg);
          const uint32_t w8 = *reinterpret_cast<uint32_t *>(&hg8);
          uint32_t u[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t a0 = __shfl_sync(0xffffffffu, w0, (lane & ~3) + k);
            const uint32_t a8 = __shfl_sync(0xffffffffu, w8, (lane & ~3) + k);
            u[k] = my_half ? a8 : a0;
          }
          if (tq < 2 && my_rowok) {
            const int rel = my_rel0 + c0;
            if (rel >= 0 && rel + 8 <= f_span) {
              int j = jv, i = iv + c0;  // advance the row's split by c0 (c0 < n)
              if (my_rel0 < 0) split(rel, j, i);
              while (i >= q) { i -= q; ++j; }
              *reinterpret_cast<uint4 *>(smem + wsw_off(j, i)) = make_uint4(u[0], u[1], u[2], u[3]);
            } else {  // the block's first / last row: element-wise
              for (int e = 0; e < 8; ++e) {
                const uint32_t word = u[e >> 1];
                put1(rel + e, (uint16_t)(e & 1 ? word >> 16 : word & 0xFFFFu));
              }
            }
          }
        } else {
          const int c = c0 + 2 * tq;
          auto hb = [](float v) {
            __nv_bfloat16 t = __float2bfloat16_rn(v);
            return *reinterpret_cast<uint16_t *>(&t);
          };
          if (c < n) {
            if (ra <= a_hi) put1(rel_g + c, hb(d[h][0]));
            if (ra + 8 <= a_hi) put1(rel_g8 + c, hb(d[h][2]));
          }
          if (c + 1 < n) {
            if (ra <= a_hi) put1(rel_g + c + 1, hb(d[h][1]));
            if (ra + 8 <= a_hi) put1(rel_g8 + c + 1, hb(d[h][3]));
          }
        }
      }
    }
  }
  if (tid == 0) gtrace(p, 30);
}

// ---- phase 2, CTA-pair variant (tcgen05 cta_group::2) ---------------------------------------
// A cluster of two CTAs owns two consecutive column blocks (UMMA M = 256: each CTA's W^T block
// resident in its own shared memory, loaded once per column group, one mbarrier per k-block so
// the first MMAs need not wait for the whole block) and walks 256-row batch tiles, each CTA
// TMA-loading its 128-row half of every x k-block (16 KB stages, S ~ 7 deep). The leader
// (cluster rank 0) issues every MMA (M = 256, N = 256) and its commits multicast to both CTAs;
// each CTA's TMEM holds its own 128 columns x 256 rows. Per SM this halves the x bytes per
// output of the single-CTA schedule and doubles the stages in flight, with no multicast copy.
constexpr uint32_t kXHalf = (GN / 2) * GK * 2;  // one CTA's half of an x k-block (16 KB)
constexpr int kMaxKB = 8;

__device__ __forceinline__ void arrive_leader(uint64_t *bar, uint32_t crank) {
  if (crank == 0)
    mbar_arrive(bar);
  else
    mbar_arrive_remote(bar, 0);
}
// "TMEM read" signals of the epilogue: relaxed (see mbar_arrive_relaxed)
__device__ __forceinline__ void arrive_leader_tmem(uint64_t *bar, uint32_t crank) {
  if (crank == 0)
    mbar_arrive_relaxed(bar);
  else
    mbar_arrive_remote_relaxed(bar, 0);
}

template <int YDT, int ACT, int EL>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_tc_gemm_pair(const __grid_constant__ CUtensorMap tm_w,
                   const __grid_constant__ CUtensorMap tm_x, const GemmParams p) {
  constexpr int GKE = EL ? 32 : 64;  // elements per 128-byte k-block
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *wfull = tempty + 2, *wfree = wfull + kMaxKB, *wgen_done = wfree + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(wgen_done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int cid = (int)blockIdx.x / 2;
  int beg, end;
  item_range(p, cid, beg, end);
  auto jb_of = [&](int it) { return (it / p.n_bt) * 2 + (int)crank; };
  auto b0_of = [&](int it) { return (it % p.n_bt) * GN; };

  if (threadIdx.x == 0) {
    gtrace(p, 0);
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * kEpiWarps); }
    for (int k = 0; k < kMaxKB; ++k) mbar_init(&wfull[k], 1);
    if (p.wgen) mbar_init(&wfull[0], 2);  // both CTAs generated their W block (leader's copy)
    mbar_init(wfree, 1);
    mbar_init(wgen_done, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch_desc(&tm_w); tma_prefetch_desc(&tm_x); }
  if (warp == 1) tmem_alloc_pair(tslot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers initialised before any pair TMA / commit lands
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) gtrace(p, 1);
  if (p.chain) griddep_launch_dependents();  // the next forward's phase 1 may start

  // ---------------- TMA producer state (warp 0, lane 0) ----------------
  // Issue order for the first column group: the first x stages before W^T is known to be
  // ready (they do not depend on phase 1), then W^T k-blocks interleaved one ahead of the
  // x stages (W0 W1 x2 W2 x3 ...), so the first MMAs wait for ~3 k-blocks of operands, not for
  // the whole W block queued behind the x prefetch (operand delivery is L2-throughput-bound).
  const bool producer = warp == 0 && lane == 0;
  int pstage = 0, pu = 0, w_next = p.KB, w_j0 = 0;
  uint32_t pphase = 0;
  const int pre = min(2, min(p.S, p.KB));
  auto issue_w = [&](int upto) {
    for (; w_next < min(upto, p.KB); ++w_next) {
      if (leader) mbar_arrive_expect_tx(&wfull[w_next], 2 * kABytes);
      tma_load_2d_pair(smem + w_next * kABytes, &tm_w, &wfull[w_next], w_next * GKE, w_j0);
    }
  };
  auto issue_x = [&](int it, int kb) {
    const int xb0 = b0_of(it) + (int)crank * (GN / 2);
    if (kTimingSwitches && (p.dbg & 2) && pu >= p.S) {  // timing experiment: stale x, no L2 traffic
      if (leader) mbar_arrive(&full[pstage]);
    } else {
      if (leader) mbar_arrive_expect_tx(&full[pstage], 2 * kXHalf);
      tma_load_2d_pair(smem + p.off_x + pstage * kXHalf, &tm_x, &full[pstage], kb * GKE, xb0);
    }
    ++pu;
    if (++pstage == p.S) { pstage = 0; pphase ^= 1; }
  };
  if (producer && beg < end) {
    if (!p.x_early && !p.wgen && !p.fused) griddep_wait();  // x may be a chained predecessor's output
    for (int kb = 0; kb < pre; ++kb) issue_x(beg, kb);  // fresh stages: no empty wait
  }

  if (p.fused) {
    // ---------------- phase 1 inside the kernel: W^T tiles on the epilogue warps ----------
    if (warp >= 2) {
      RegenSmem &rs = *reinterpret_cast<RegenSmem *>(smem + p.off_rg);  // no TMA lands here yet
      auto sync = [] { named_bar_sync(1, 256); };
      const int n_units = p.rg_ux * p.rg_uy;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int bx = u % p.rg_ux, by = u / p.rg_ux, t = threadIdx.x - 64;
        if (p.rg_rows == 64) {
          if (p.rg.f_dtype == DT_F32) regen_tile<float, 64>(p.rg, t, bx, by, rs, sync);
          else regen_tile<__nv_bfloat16, 64>(p.rg, t, bx, by, rs, sync);
        } else {
          if (p.rg.f_dtype == DT_F32) regen_tile<float, 32>(p.rg, t, bx, by, rs, sync);
          else regen_tile<__nv_bfloat16, 32>(p.rg, t, bx, by, rs, sync);
        }
      }
      fence_proxy_async_global();  // W^T stores -> the TMA reads of every CTA
      fence_proxy_async_smem();    // staging stores -> the W block TMA writes to the same bytes
    }
    if (threadIdx.x == 64) gtrace(p, 42);
    cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0) gtrace(p, 43);
  }

  if (p.wgen && warp >= 2 && beg < end) {
    // ---------------- W block generated in shared memory (epilogue warps) ----------------
    if (p.rg.f_dtype == DT_F32)
      wgen_block<float>(p, jb_of(beg) * GM, smem, threadIdx.x - 64);
    else
      wgen_block<__nv_bfloat16>(p, jb_of(beg) * GM, smem, threadIdx.x - 64);
    fence_proxy_async_smem();  // generic-proxy W stores -> the tensor cores' operand reads
    named_bar_sync(1, 256);
    if (threadIdx.x == 64) {
      gtrace(p, 42);
      mbar_arrive(wgen_done);             // the factor staging area may take x stages now
      arrive_leader(&wfull[0], crank);    // the leader's MMAs read both CTAs' W blocks
    }
  }

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own W block, own half of each x tile) -------
    if (lane == 0) {
      int jg_cur = -1;
      uint32_t wf_phase = 0;
      for (int it = beg; it < end; ++it) {
        const int jg = it / p.n_bt, j0 = jb_of(it) * GM;
        if (jg != jg_cur && jg_cur >= 0) {  // next W block once the MMAs on the old one retired
          issue_w(p.KB);
          mbar_wait(wfree, wf_phase);
          wf_phase ^= 1;
          w_next = 0;
          w_j0 = j0;
          issue_w(p.KB);
        }
        if (it == beg && p.wgen) {  // stages past `pre` hold the factor staging until then
          mbar_wait(wgen_done, 0);
          gtrace(p, 2);
        } else if (it == beg) {  // W^T is phase 1's output
          if (p.fused)
            fence_proxy_async_global();
          else
            griddep_wait();
          gtrace(p, 2);
          w_next = 0;
          w_j0 = j0;
          issue_w(2);
        }
        for (int kb = it == beg ? pre : 0; kb < p.KB; ++kb) {
          issue_w(pu - pre + 3);
          if (pstage == 0 && pu >= p.S) issue_w(p.KB);  // before the first wait on a stage
          mbar_wait(&empty[pstage], pphase ^ 1);
          if (pu < 8) gtrace(p, 34 + pu);
          issue_x(it, kb);
        }
        jg_cur = jg;
      }
      issue_w(p.KB);
      gtrace(p, 3);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (lane == 0 && leader) {
      const uint32_t idesc = idesc_f32acc(2 * GM, GN, EL ? 2 : 1);
      const uint32_t s0 = smem_u32(smem);
      int stage = 0, acc = 0, jg_cur = -1;
      uint32_t phase = 0, aphase = 0, wphase = 0;
      for (int it = beg; it < end; ++it) {
        const int jg = it / p.n_bt;
        const bool first_of_group = jg != jg_cur;
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * GN);
        for (int kb = 0; kb < p.KB; ++kb) {
          if (first_of_group && (!p.wgen || kb == 0))  // both CTAs' W k-block (or block) ready
            mbar_wait(&wfull[kb], wphase);
          mbar_wait(&full[stage], phase);
          if (it == beg) gtrace(p, 20 + kb);
          tc_fence_after();
          const uint32_t a_s = s0 + (uint32_t)kb * kABytes;
          const uint32_t b_s = s0 + p.off_x + (uint32_t)stage * kXHalf;
#pragma unroll
          for (int k = 0; k < GK / 16; ++k)
            if constexpr (EL)
              mma_tf32_ss_pair(d, smem_desc(a_s + k * 32, 16, 1024, SL_SW128),
                               smem_desc(b_s + k * 32, 16, 1024, SL_SW128), idesc, (kb | k) != 0);
            else
              mma_bf16_ss_pair(d, smem_desc(a_s + k * 32, 16, 1024, SL_SW128),
                               smem_desc(b_s + k * 32, 16, 1024, SL_SW128), idesc, (kb | k) != 0);
          mma_commit_pair(&empty[stage]);  // frees the stage in both CTAs
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        if (first_of_group) { wphase ^= 1; jg_cur = jg; }
        mma_commit_pair(&tfull[acc]);
        if (it + 1 < end && (it + 1) / p.n_bt != jg) mma_commit_pair(wfree);
        gtrace(p, 4 + min(it - beg, 7));
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (both CTAs: own 128 columns x 256 rows) ----------------
    const int wq = warp & 3;
    const int part = (warp - 2) / 4;
    using OutT = typename std::conditional<YDT == DT_BF16, __nv_bfloat16, float>::type;
    int acc = 0;
    uint32_t aphase = 0;
    double sq = 0.0;  // YDT_MSE: this thread's share of the tile's squared error
    for (int it = beg; it < end; ++it) {
      const int j = jb_of(it) * GM + 32 * wq + lane;
      const int64_t b0 = b0_of(it);
      const bool jok = j < p.r_dim;
      const float bias_j = (p.bias && jok) ? __ldg(p.bias + j) : 0.f;
      const int nrows = (int)min((int64_t)GN, p.batch - b0);
      mbar_wait(&tfull[acc], aphase);
      if (threadIdx.x == 64 && it - beg < 2) gtrace(p, 44 + (it - beg));
      tc_fence_after();
      for (int c32 = part; c32 < GN / 32; c32 += kEpiParts) {
        if (32 * c32 >= nrows) break;
        uint32_t v[32];
        if (kTimingSwitches && (p.dbg & 4)) {
          for (int r = 0; r < 32; ++r) v[r] = 0;
        } else {
          tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(acc * GN + c32 * 32), v);
          tmem_ld_wait();
        }
        if (jok && !(kTimingSwitches && (p.dbg & 1))) {
          OutT *yp = reinterpret_cast<OutT *>(p.y) + (b0 + 32 * c32) * p.ldy + j;
          const int rmax = nrows - 32 * c32;
          if constexpr (YDT == YDT_MSE) {  // grad = scale * (z - t), sum (z - t)^2
            // fp32 per element (fp64 math per element made this epilogue the bottleneck), the
            // 32-row chunk's fp32 sum folded into the thread's fp64 total in a fixed order
            const float *tp = p.target + (b0 + 32 * c32) * p.ldy + j;
            const float sc = (float)p.scale;
            float tv[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) tv[r] = r < rmax ? __ldg(tp + (int64_t)r * p.ldy) : 0.f;
            float csq = 0.f;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              if (r < rmax) {
                const float dz = (__uint_as_float(v[r]) + bias_j) - tv[r];
                *yp = sc * dz;
                csq = fmaf(dz, dz, csq);
              }
              yp += p.ldy;
            }
            sq += (double)csq;
          } else if (rmax >= 32) {  // full chunk: no per-row predicate, pointer bumps only
            const int64_t ld = p.ldy;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
              if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
              yp += ld;
            }
          } else {
#pragma unroll
            for (int r = 0; r < 32; ++r) {
              if (r < rmax) {
                const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
                if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
              }
              yp += p.ldy;
            }
          }
        }
      }
      if constexpr (YDT == YDT_MSE) {  // fixed-order warp reduction -> one partial per warp
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) p.loss_part[((int64_t)it * 2 + crank) * kEpiWarps + (warp - 2)] = sq;
        sq = 0.0;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader_tmem(&tempty[acc], crank);  // the leader's MMAs reuse it
      if (threadIdx.x == 64) gtrace(p, 12 + min(it - beg, 7));
      if (threadIdx.x == kGemmThreads - 32 && it - beg < 2) gtrace(p, 46 + (it - beg));
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

typedef void (*GemmFn)(CUtensorMap, CUtensorMap, GemmParams);

template <int YDT, int EL>
GemmFn pick_gemm_el(int act, bool pair) {
  if (pair) switch (act) {
      case DT_ACT_RELU: return k_tc_gemm_pair<YDT, DT_ACT_RELU, EL>;
      case DT_ACT_SIGMOID: return k_tc_gemm_pair<YDT, DT_ACT_SIGMOID, EL>;
      case DT_ACT_TANH: return k_tc_gemm_pair<YDT, DT_ACT_TANH, EL>;
      case DT_ACT_CLIPPED_RELU: return k_tc_gemm_pair<YDT, DT_ACT_CLIPPED_RELU, EL>;
      default: return k_tc_gemm_pair<YDT, DT_ACT_IDENTITY, EL>;
    }
  switch (act) {
    case DT_ACT_RELU: return k_tc_gemm<YDT, DT_ACT_RELU, EL>;
    case DT_ACT_SIGMOID: return k_tc_gemm<YDT, DT_ACT_SIGMOID, EL>;
    case DT_ACT_TANH: return k_tc_gemm<YDT, DT_ACT_TANH, EL>;
    case DT_ACT_CLIPPED_RELU: return k_tc_gemm<YDT, DT_ACT_CLIPPED_RELU, EL>;
    default: return k_tc_gemm<YDT, DT_ACT_IDENTITY, EL>;
  }
}
GemmFn pick_gemm(int y_dtype, int act, bool pair, int el) {
  if (y_dtype == YDT_MSE) {  // identity activation only
    if (el) return pair ? k_tc_gemm_pair<YDT_MSE, DT_ACT_IDENTITY, 1> : k_tc_gemm<YDT_MSE, DT_ACT_IDENTITY, 1>;
    return pair ? k_tc_gemm_pair<YDT_MSE, DT_ACT_IDENTITY, 0> : k_tc_gemm<YDT_MSE, DT_ACT_IDENTITY, 0>;
  }
  if (el)
    return y_dtype == DT_BF16 ? pick_gemm_el<DT_BF16, 1>(act, pair) : pick_gemm_el<DT_F32, 1>(act, pair);
  return y_dtype == DT_BF16 ? pick_gemm_el<DT_BF16, 0>(act, pair) : pick_gemm_el<DT_F32, 0>(act, pair);
}

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

void print_gemm_trace(const std::vector<unsigned long long> &h, int grid, int n_tiles) {
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int c = 0; c < grid; ++c) {
    if (h[(size_t)c * kTrace]) t0 = std::min(t0, h[(size_t)c * kTrace]);
    for (int s = 0; s < kTrace; ++s) t1 = std::max(t1, h[(size_t)c * kTrace + s]);
  }
  fprintf(stderr, "[gemm trace] grid %d items %d span %.2f us\n", grid, n_tiles, (t1 - t0) / 1e3);
  {  // per-CTA start / end distribution
    std::vector<double> st, en;
    for (int c = 0; c < grid; ++c) {
      const unsigned long long *r = &h[(size_t)c * kTrace];
      unsigned long long e = 0;
      for (int s = 0; s < kTrace; ++s) e = std::max(e, r[s]);
      st.push_back((r[0] - t0) / 1e3);
      en.push_back((e - t0) / 1e3);
    }
    std::sort(st.begin(), st.end());
    std::sort(en.begin(), en.end());
    auto q = [&](const std::vector<double> &v, double f) { return v[(size_t)(f * (v.size() - 1))]; };
    fprintf(stderr, "  CTA start min/med/p90/max %.2f %.2f %.2f %.2f | end min/med/p90/max %.2f %.2f %.2f %.2f\n",
            q(st, 0), q(st, .5), q(st, .9), q(st, 1), q(en, 0), q(en, .5), q(en, .9), q(en, 1));
  }
  std::vector<int> show;
  for (int c = 0; c < grid; c += std::max(1, grid / 6)) show.push_back(c);
  for (int c = 0; c < grid; ++c) {  // plus the three latest-finishing CTAs
    unsigned long long e = 0;
    for (int s = 0; s < kTrace; ++s) e = std::max(e, h[(size_t)c * kTrace + s]);
    if (e + 1500 >= t1 && show.size() < 10) show.push_back(c);
  }
  for (int c : show) {
    const unsigned long long *r = &h[(size_t)c * kTrace];
    auto rel = [&](int s) { return r[s] ? (double)(r[s] - t0) / 1e3 : -1.0; };
    fprintf(stderr, "  cta %3d: start %.2f setup %.2f wgen zero/stage/mma %.2f %.2f %.2f regen-done %.2f gsync %.2f W-ready %.2f prod-done %.2f | mma",
            c, rel(0), rel(1), rel(28), rel(29), rel(30), rel(42), rel(43), rel(2), rel(3));
    for (int k = 0; k < 8; ++k)
      if (r[4 + k]) fprintf(stderr, " %.2f", rel(4 + k));
    fprintf(stderr, " | epi");
    for (int k = 0; k < 8; ++k)
      if (r[12 + k]) fprintf(stderr, " %.2f", rel(12 + k));
    fprintf(stderr, "\n        first tile full[kb]:");
    for (int k = 0; k < 14; ++k)
      if (r[20 + k]) fprintf(stderr, " %.2f", rel(20 + k));
    fprintf(stderr, " | epi-start %.2f %.2f last-warp-done %.2f %.2f", rel(44), rel(45), rel(46),
            rel(47));
    fprintf(stderr, " | producer empty-ok[u]:");
    for (int k = 0; k < 8; ++k)
      if (r[34 + k]) fprintf(stderr, " %.2f", rel(34 + k));
    fprintf(stderr, "\n");
  }
}

}  // namespace

// One phase-2 launch: y[rows x cols] (pitch ldy) = act(x[rows x K] @ wt[cols x K]^T + bias),
// bf16 operands with 16-byte-aligned pitches, fp32 accumulation. `rg` non-null: wt is the output
// of the phase-1 regeneration described by rg, launched here first (PDL / fused / wgen
// schedules apply); null: wt is ready in memory.
struct GemmCall {
  const void *x;
  int64_t ldx, rows, K;
  const void *wt;
  int64_t ldw, cols;
  const float *bias;
  int act;
  float act_arg;
  void *y;
  int64_t ldy;
  int y_dtype;
  const RegenArgs *rg;
  bool profile;  // the forward's dominant kernel: dt_profile_kernel_events brackets it
  int el = 0;    // operand element type: 0 bf16 (kind::f16), 1 fp32 (kind::tf32)
  // y_dtype == YDT_MSE: fused MSE gradient against `target`, partials into loss_part
  const float *target = nullptr;
  double scale = 0.0;
  double *loss_part = nullptr;
  int64_t *n_part = nullptr;  // out: number of partials written
};

static int run_gemm(const GemmCall &c, cudaStream_t st) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  static const int max_sm = getenv("DEEPTHIN_GEMM_MAXSM") ? atoi(getenv("DEEPTHIN_GEMM_MAXSM")) : 0;
  if (max_sm > 0) nsm = std::min(nsm, max_sm);
  GemmParams p{};
  const int64_t n_bt = (c.rows + GN - 1) / GN;
  const int64_t n_jb = (c.cols + GM - 1) / GM;
  const int gke = c.el ? 32 : 64;  // elements per 128-byte k-block
  p.KB = (int)((c.K + gke - 1) / gke);
  // operand schedule + shared-memory layout (see GemmParams)
  const uint32_t kFixed = 256 /*barriers*/ + 1024 /*alignment slack*/;
  const uint32_t wbytes = (uint32_t)p.KB * kABytes;
  static const int want_cs = getenv("DEEPTHIN_GEMM_CLUSTER") ? atoi(getenv("DEEPTHIN_GEMM_CLUSTER")) : 4;
  static const int want_wres = getenv("DEEPTHIN_GEMM_WRES") ? atoi(getenv("DEEPTHIN_GEMM_WRES")) : 1;
  static const int want_pair = getenv("DEEPTHIN_GEMM_PAIR") ? atoi(getenv("DEEPTHIN_GEMM_PAIR")) : 1;
  bool pair = false;
  if (want_pair && n_jb >= 2 && p.KB <= kMaxKB &&
      wbytes + 4 * kXHalf + kFixed <= (uint32_t)kSmemMax) {
    pair = true;
    p.wres = 1;
    p.stage_bytes = kXHalf;
    p.off_x = wbytes;
    // stages: DEEPTHIN_GEMM_STAGES caps them (fewer stages leave shared memory for a
    // co-resident phase-1 CTA of the next pipelined forward)
    static const int max_stages = getenv("DEEPTHIN_GEMM_STAGES") ? atoi(getenv("DEEPTHIN_GEMM_STAGES")) : 8;
    p.S = (int)std::min<uint32_t>((uint32_t)std::max(4, max_stages),
                                  (kSmemMax - kFixed - wbytes) / kXHalf);
    p.csize = 2;
  } else if (want_wres && p.KB <= 8 && wbytes + 3 * kXBytes + kFixed <= (uint32_t)kSmemMax) {
    p.wres = 1;
    p.stage_bytes = kXBytes;
    p.off_x = wbytes;
    p.S = (int)std::min<uint32_t>(6, (kSmemMax - kFixed - wbytes) / kXBytes);
    p.csize = 1;
    for (int cs : {16, 8, 4, 2})
      if (cs <= want_cs && n_jb >= cs) { p.csize = cs; break; }
  } else {
    p.wres = 0;
    p.stage_bytes = kABytes + kXBytes;
    p.off_x = 0;
    p.S = (int)std::min<uint32_t>(6, (kSmemMax - kFixed) / p.stage_bytes);
    p.csize = 1;
  }
  p.off_bar = p.off_x + (uint32_t)p.S * p.stage_bytes;
  const uint32_t smem_bytes = p.off_bar + kFixed;
  const int64_t n_jg = (n_jb + p.csize - 1) / p.csize;
  if (n_jg * n_bt > INT32_MAX / 2 || c.cols > INT32_MAX / 2 || c.ldy > INT32_MAX) {
    set_error("tensor-core GEMM: too many tiles");
    return DT_E_UNSUPPORTED;
  }
  p.n_jb = (int)n_jb;
  p.n_bt = (int)n_bt;
  p.n_jg = (int)n_jg;
  p.items = (int)(n_jg * n_bt);
  p.ncl = std::min(p.items, nsm / p.csize);
  // whole column groups per cluster when every group gets at least one cluster (no W reloads)
  p.cpj = p.ncl >= p.n_jg ? std::min(p.ncl / p.n_jg, p.n_bt) : 0;
  if (p.cpj > 0) p.ncl = p.cpj * p.n_jg;
  const int grid = p.ncl * p.csize;
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_TC_TRACE") != 0;
  unsigned long long *tbuf = nullptr;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&tbuf, (size_t)grid * kTrace * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(tbuf, 0, (size_t)grid * kTrace * 8, st));
  }

  // DEEPTHIN_DBG_PHASE=1 / 2: launch only phase 1 / phase 2 (timing experiments only — the
  // output is wrong).
  static const int dbg_phase = DT_DBG_ENV("DEEPTHIN_DBG_PHASE");
  // DEEPTHIN_GEMM_FUSED=1: phase 1 inside the (cooperatively launched) pair kernel, a grid
  // barrier between the phases (a refused cooperative launch falls back to two kernels).
  // Measured slower than the two-kernel form at BASELINE config 2 (20.2 vs 18.7 us/step: the
  // grid barrier ~1.6 us and one 64-row tile per CTA ~3.3 us), so off by default.
  const int want_fused = getenv("DEEPTHIN_GEMM_FUSED") ? atoi(getenv("DEEPTHIN_GEMM_FUSED")) : 0;

  CUtensorMap tm_w, tm_x;
  const int tdt = c.el ? DT_F32 : DT_BF16, esz = c.el ? 4 : 2;
  if (int rc = encode_tensor_map_2d(&tm_w, tdt, const_cast<void *>(c.wt), (uint64_t)c.K,
                                    (uint64_t)c.cols, (uint64_t)c.ldw * esz, gke, GM, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_x, tdt, const_cast<void *>(c.x), (uint64_t)c.K,
                                    (uint64_t)c.rows, (uint64_t)c.ldx * esz, gke, GN / p.csize, true))
    return rc;
  p.batch = c.rows;
  p.r_dim = (int)c.cols;
  p.ldy = (int)c.ldy;
  p.trace = tbuf;
  static const int dbg_gemm = DT_DBG_ENV("DEEPTHIN_DBG_GEMM");
  p.dbg = dbg_gemm;
  p.bias = c.bias;
  p.y = c.y;
  p.arg = c.act_arg;
  p.target = c.target;
  p.scale = c.scale;
  p.loss_part = c.loss_part;
  if (c.n_part) *c.n_part = (int64_t)p.items * p.csize * kEpiWarps;
  if (c.loss_part)
    DT_CUDA_CHECK(cudaMemsetAsync(c.loss_part, 0,
                                  (size_t)p.items * p.csize * kEpiWarps * sizeof(double), st));
  dim3 rgrid(1, 1);
  if (c.rg) {
    const RegenArgs &rg = *c.rg;
    rgrid = dim3((unsigned)((rg.a_rows + RG_R - 1) / RG_R), (unsigned)((rg.n + RG_C - 1) / RG_C));
    p.rg = rg;
    p.chain = rg.chain;
    p.x_early = (!rg.chain || rg.x_ext) ? 1 : 0;
    // fused phase 1: 64-row tiles when that makes one tile per CTA, else 32-row tiles
    p.rg_rows = ((rg.a_rows + 63) / 64) * (int64_t)rgrid.y <= (int64_t)grid ? 64 : 32;
    p.rg_ux = (int)((rg.a_rows + p.rg_rows - 1) / p.rg_rows);
    p.rg_uy = (int)rgrid.y;
  }
  const int eact = c.act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : c.act;
  GemmFn fn = pick_gemm(c.y_dtype, eact, pair, c.el);
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  if (p.csize > 8)
    if (int rc = allow_nonportable_clusters(reinterpret_cast<const void *>(fn))) return rc;

  static const int use_pdl = getenv("DEEPTHIN_PDL") ? atoi(getenv("DEEPTHIN_PDL")) : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  auto launch = [&](bool fused) {
    int na = 0;
    if (fused) {
      attr[na].id = cudaLaunchAttributeCooperative;
      attr[na].val.cooperative = 1;
      ++na;
    } else if (use_pdl && c.rg && !p.wgen) {  // overlap the prologue with phase 1
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (p.csize > 1) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = (unsigned)p.csize;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    p.fused = fused ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, tm_w, tm_x, p);
  };
  // phase-1 staging inside the fused kernel: the W block area, else x stages past the ones
  // prefetched during phase 1
  const uint32_t pre_stages = (uint32_t)std::min(2, std::min(p.S, p.KB));
  // DEEPTHIN_GEMM_WGEN=1: every CTA generates its own W^T block in shared memory (no phase-1
  // kernel, no W^T outside the SM). Needs one column group per cluster (cpj > 0), rank <= 64
  // and the factor staging to fit in the x stages not prefetched. Measured slower than the
  // two-kernel form at config 2 (~40 vs 20.7 us/step): the per-element scatter is
  // instruction-latency-bound on 8 warps and its one-pass code runs from a cold I-cache.
  const int want_wgen = getenv("DEEPTHIN_GEMM_WGEN") ? atoi(getenv("DEEPTHIN_GEMM_WGEN")) : 0;
  p.off_fs = p.off_x + pre_stages * p.stage_bytes;
  p.wgen = (c.rg && !c.el && pair && want_wgen && p.cpj > 0 && c.rg->rank <= 64 && dbg_phase == 0 &&
            p.off_fs + wgen_stage_bytes((int)c.rg->q, c.rg->rank, c.rg->n) <= p.off_bar)
               ? 1
               : 0;
  p.off_rg = wbytes >= sizeof(RegenSmem) ? 0u : p.off_x + pre_stages * p.stage_bytes;
  const bool rg_fits = p.off_rg + sizeof(RegenSmem) <= p.off_bar;
  cudaEvent_t ev_b = nullptr, ev_a = nullptr;  // dt_profile_kernel_events: bracket the GEMM
  if (c.profile) profile_next(&ev_b, &ev_a, DT_PROF_GEMM);
  bool done = false;
  if (p.wgen) {
    if (ev_b) DT_CUDA_CHECK(cudaEventRecord(ev_b, st));
    DT_CUDA_CHECK(launch(false));
    done = true;
  } else if (c.rg && pair && want_fused && rg_fits && dbg_phase == 0) {
    if (ev_b) DT_CUDA_CHECK(cudaEventRecord(ev_b, st));
    const cudaError_t e = launch(true);
    if (e == cudaSuccess) {
      done = true;
    } else if (e == cudaErrorCooperativeLaunchTooLarge) {
      (void)cudaGetLastError();  // not all CTAs co-resident right now: two kernels instead
    } else {
      set_error(std::string("tc_gemm (fused) launch: ") + cudaGetErrorString(e));
      return DT_E_CUDA;
    }
  }
  if (!done) {
    if (c.rg && dbg_phase != 2) {
      if (int rc = launch_regen_wt(*c.rg, st)) return rc;
    }
    if (c.rg && dbg_phase == 1) return DT_OK;
    if (ev_b) DT_CUDA_CHECK(cudaEventRecord(ev_b, st));
    DT_CUDA_CHECK(launch(false));
  }
  if (ev_a) DT_CUDA_CHECK(cudaEventRecord(ev_a, st));
  if (int rc = check_launch("tc_gemm")) return rc;
  if (tracing) {
    std::vector<unsigned long long> h((size_t)grid * kTrace);
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    DT_CUDA_CHECK(cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(tbuf);
    print_gemm_trace(h, grid, p.items);
  }
  if (c.act == DT_ACT_SOFTMAX) return launch_row_softmax(c.rows, c.cols, c.y, c.y_dtype, st);
  return DT_OK;
}

// Factored reuse forward on the tensor cores (n | q, s = q/n; kernel.py:1-16 with one phase):
//   P  (B*s x rank) = x.view(B*s, n) @ wf^T        GEMM 1: bf16 operands, fp32 P
//   y  (B x r_dim)  = P.view(B, s*rank) @ XF2^T    GEMM 2: kind::tf32 on the fp32 P and the
//                                                  fp32 master xf viewed (r_dim x s*rank)
// 2*B*s*rank*(n + r_dim) flops instead of the dense 2*B*q*r_dim, and no intermediate bf16
// rounding (P stays fp32; rounding it to bf16 measured 2.5e-3 rel_error at config 1 — over the
// 2e-3 contract — while tf32 products keep the two-GEMM error at the operand-rounding level).
// Needs aligned views: n % 8 == 0 (bf16 rows), s*rank % 4 == 0 (fp32 rows); fp32 factors.
// DEEPTHIN_RUNS=0 routes low-rank straddling layers to the two-phase path instead (comparisons)
static bool runs_disabled() {
  static const bool off = getenv("DEEPTHIN_RUNS") && atoi(getenv("DEEPTHIN_RUNS")) == 0;
  return off;
}

static bool reuse_factored_ok(const Geo &g) {
  const int want = getenv("DEEPTHIN_REUSE_FACTORED") ? atoi(getenv("DEEPTHIN_REUSE_FACTORED")) : 1;
  return want && g.reuse && g.n % 8 == 0 && (g.s * g.rank) % 4 == 0;
}
static size_t reuse_factored_ws(const Geo &g, int64_t batch) {
  return (size_t)round_up(g.rank * g.n * 2, 256) + (size_t)round_up(batch * g.s * g.rank * 4, 256) +
         (size_t)round_up(batch * g.q * 2, 256);
}

// W^T slot of a pipelined forward: consecutive calls with one workspace alternate between two
// slots, so a call's phase 1 never overwrites the W^T the previous call's GEMM is reading.
static int pipeline_slot(const void *ws) {
  static std::mutex mu;
  static std::unordered_map<const void *, unsigned> next;
  std::lock_guard<std::mutex> lock(mu);
  return (int)(next[ws]++ & 1u);
}

// W^T slot of the two-phase forward: the hi | lo rows (2 x round_up(q, 64) bf16 per row)
static int64_t wt_slot_bytes(const Geo &g) {
  return round_up(g.r_dim * 2 * round_up(g.q, 64) * 2, 256);
}

size_t tc_gemm_ws(const Geo &g, int64_t batch) {
  const int64_t ldw = round_up(g.q, 8);
  const size_t two_phase =  // two W^T slots (pipelined forwards alternate) + packed x
      2 * (size_t)wt_slot_bytes(g) + (size_t)round_up(batch * ldw * 2, 256);
  return std::max(std::max(std::max(two_phase, reuse_factored_ok(g) ? reuse_factored_ws(g, batch)
                                                                     : (size_t)0),
                           tc_rows_ws(g)),
                  tc_runs_ws(g));
}

struct MseArgs {
  const float *target;
  double scale;
  double *loss_sum;
  double *part;     // workspace for the per-warp partials
  float *d_bias;    // nullable: the column sums of grad (grad.py:85) in the loss pass
  float *p_out;     // nullable: keep P (B x s*rank fp32) for the backward
};
static int64_t mse_parts_bound(const Geo &g, int64_t batch) {
  return ((g.r_dim + GM - 1) / GM + 2) * ((batch + GN - 1) / GN) * kEpiWarps;
}


static int tc_forward_impl(const Geo &g, int64_t batch, const void *x, int x_dtype,
                           const void *xf, const void *wf, int f_dtype, const float *bias,
                           int act, float act_arg, void *y, int y_dtype, char *ws,
                           size_t ws_bytes, cudaStream_t st, const MseArgs *mse);

int tc_gemm_forward(const Geo &g, int64_t batch, const void *x, int x_dtype, const void *xf,
                    const void *wf, int f_dtype, const float *bias, int act, float act_arg,
                    void *y, int y_dtype, char *ws, size_t ws_bytes, cudaStream_t st) {
  return tc_forward_impl(g, batch, x, x_dtype, xf, wf, f_dtype, bias, act, act_arg, y, y_dtype,
                         ws, ws_bytes, st, nullptr);
}

size_t tc_forward_mse_ws(const Geo &g, int64_t batch) {
  const size_t own = tc_gemm_ws(g, batch) + (size_t)round_up(mse_parts_bound(g, batch) * 8, 256) +
                     (size_t)round_up(g.r_dim * 4, 256) + (size_t)round_up(1184 * 8, 256) +
                     (size_t)round_up(colsum_ws(batch, g.r_dim), 256);
  return std::max(own, xtrain_ok(g) ? xtrain_forward_mse_ws(g, batch) : (size_t)0);
}

int tc_forward_mse(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                   const float *wf, const float *bias, const float *target, double scale,
                   float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st,
                   float *d_bias, float *p_out) {
  if (xtrain_ok(g) && x_dtype == DT_BF16) {  // k_train.cu: our tcgen05 GEMMs, fused MSE + d_bias
    if (batch == 0) {
      if (loss_sum) DT_CUDA_CHECK(cudaMemsetAsync(loss_sum, 0, sizeof(double), st));
      if (d_bias) DT_CUDA_CHECK(cudaMemsetAsync(d_bias, 0, (size_t)g.r_dim * 4, st));
      return DT_OK;
    }
    return xtrain_forward_mse(g, batch, x, x_dtype, xf, wf, bias, target, scale, grad, loss_sum,
                              ws, ws_bytes, st, d_bias, p_out);
  }
  if (p_out && !(reuse_factored_ok(g))) {
    set_error("forward_mse: P is kept only on reuse geometries (factored path)");
    return DT_E_UNSUPPORTED;
  }
  if (ws_bytes < tc_forward_mse_ws(g, batch)) {
    set_error("forward+mse workspace too small: need " + std::to_string(tc_forward_mse_ws(g, batch)));
    return DT_E_ARG;
  }
  if (batch == 0) {
    if (loss_sum) DT_CUDA_CHECK(cudaMemsetAsync(loss_sum, 0, sizeof(double), st));
    return DT_OK;
  }
  const size_t base = tc_gemm_ws(g, batch);
  MseArgs m{target, scale, loss_sum, reinterpret_cast<double *>(ws + base), d_bias, p_out};
  int rc = tc_forward_impl(g, batch, x, x_dtype, xf, wf, DT_F32, bias, DT_ACT_IDENTITY, 0.f, grad,
                           YDT_MSE, ws, base, st, &m);
  if (rc == DT_OK && m.d_bias) {  // paths without the fused column sums: a separate pass
    char *tail = ws + base + round_up(mse_parts_bound(g, batch) * 8, 256) + round_up(g.r_dim * 4, 256) +
                 round_up(1184 * 8, 256);
    rc = launch_colsum(batch, g.r_dim, grad, d_bias, reinterpret_cast<float *>(tail), st);
  }
  return rc;
}

int tc_forward_path(const Geo &g, int x_dtype, int f_dtype, int y_dtype) {
  // mirrors tc_forward_impl's order below (non-MSE launch, 16-byte-aligned operands)
  if (f_dtype != DT_F32 && f_dtype != DT_BF16) return -DT_E_ARG;
  if (g.m * g.n > INT32_MAX || g.r_dim > INT32_MAX / 2) return -DT_E_UNSUPPORTED;
  if (f_dtype == DT_F32 && tc_rows_ok(g, x_dtype, y_dtype)) return DT_PATH_ROWS;
  if (reuse_factored_ok(g) && f_dtype == DT_F32) return DT_PATH_FACTORED;
  if (f_dtype == DT_F32 && tc_runs_ok(g, x_dtype, y_dtype) && !runs_disabled()) return DT_PATH_RUNS;
  if (y_dtype == DT_F32 && g.q * 2 * round_up(g.q, 64) < INT32_MAX) return DT_PATH_HILO;
  return DT_PATH_PAIR;
}

static int tc_forward_impl(const Geo &g, int64_t batch, const void *x, int x_dtype,
                           const void *xf, const void *wf, int f_dtype, const float *bias,
                           int act, float act_arg, void *y, int y_dtype, char *ws,
                           size_t ws_bytes, cudaStream_t st, const MseArgs *mse) {
  if (batch == 0) return DT_OK;
  int64_t n_part = 0;
  auto finish_mse = [&](int rc) {
    if (rc || !mse) return rc;
    if (n_part > mse_parts_bound(g, batch)) {
      set_error("mse partials exceed the workspace bound");
      return (int)DT_E_ARG;
    }
    return mse->loss_sum ? launch_sum_f64(n_part, mse->part, mse->loss_sum, st) : (int)DT_OK;
  };
  if (f_dtype != DT_F32 && f_dtype != DT_BF16) {
    set_error("tensor-core path: factors must be DT_F32 or DT_BF16");
    return DT_E_ARG;
  }
  if (g.m * g.n > INT32_MAX || g.r_dim > INT32_MAX / 2) {
    set_error("tensor-core path: m*n must fit in 32 bits");
    return DT_E_UNSUPPORTED;
  }
  if (ws_bytes < tc_gemm_ws(g, batch)) {
    set_error("forward workspace too small: need " + std::to_string(tc_gemm_ws(g, batch)));
    return DT_E_ARG;
  }

  // one-kernel row-tile form (k_tc_rows.cu) when the geometry and operands allow it; it pads
  // each segment's rank to 4, so it also serves reuse geometries whose s*rank % 4 != 0
  if (f_dtype == DT_F32 && !mse && tc_rows_ok(g, x_dtype, y_dtype) &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
        reinterpret_cast<uintptr_t>(bias)) & 15) == 0) {
    // (softmax: fused into the epilogue when it fits, else a post pass inside)
    return tc_rows_forward(g, batch, x, reinterpret_cast<const float *>(wf),
                           reinterpret_cast<const float *>(xf), bias, act, act_arg, y, y_dtype,
                           ws, st);
  }
  if (reuse_factored_ok(g) && f_dtype == DT_F32) {
    // ---- factored reuse path: two GEMMs ----
    char *cur = ws;
    auto take = [&](int64_t bytes) {
      char *r = cur;
      cur += round_up(bytes, 256);
      return r;
    };
    char *wf16 = take(g.rank * g.n * 2);
    float *P = reinterpret_cast<float *>(take(batch * g.s * g.rank * 4));
    char *x_ws = take(batch * g.q * 2);
    if (int rc = launch_cast_bf16(g.rank * g.n, reinterpret_cast<const float *>(wf),
                                  reinterpret_cast<uint16_t *>(wf16), st))
      return rc;
    const void *xt = x;
    if (x_dtype != DT_BF16 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
      if (int rc = launch_pack_x(batch, g.q, g.q, x, x_dtype, x_ws, st)) return rc;
      xt = x_ws;
    }
    const int64_t SR = g.s * g.rank;
    if (mse && mse->p_out) P = mse->p_out;  // kept for the backward (dt_backward_ex)
    GemmCall c1{xt, g.n, batch * g.s, g.n, wf16, g.n, g.rank, nullptr, DT_ACT_IDENTITY, 0.f,
                P, g.rank, DT_F32, nullptr, false, 0};
    if (int rc = run_gemm(c1, st)) return rc;
    GemmCall c2{P, SR, batch, SR, xf, SR, g.r_dim, bias, act, act_arg,
                y, g.r_dim, y_dtype, nullptr, true, 1};
    if (mse) {
      c2.target = mse->target; c2.scale = mse->scale; c2.loss_part = mse->part;
      c2.n_part = &n_part;
    }
    return finish_mse(run_gemm(c2, st));
  }

  // ---- low-rank straddling layers, bf16 in / out: the memoized runs (k_tc_runs.cu) ----
  if (!mse && f_dtype == DT_F32 && tc_runs_ok(g, x_dtype, y_dtype) && !runs_disabled() &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0)
    return tc_runs_forward(g, batch, x, reinterpret_cast<const float *>(wf),
                           reinterpret_cast<const float *>(xf), bias, act, act_arg, y, ws, st);

  // ---- two-phase: W^T regenerated into the workspace, then the GEMM ----
  const int64_t ldw = round_up(g.q, 8);
  const bool pipe = forward_pipeline();
  const int64_t slot_bytes = wt_slot_bytes(g);
  if (!mse && y_dtype == DT_F32 && g.q * 2 * round_up(g.q, 64) < INT32_MAX) {
    // fp32 outputs: W^T as bf16 hi + lo. Phase 1 writes rows [hi | lo] (K = 2 qp), phase 2 is
    // the any-major tcgen05 GEMM (k_tc_xgemm.cu) with x read twice through a wrapping tensor
    // map, epilogue transposed into y's row-major layout with bias + activation. W keeps ~16
    // significant bits: rel_error ~3e-6 instead of the 1.7-1.9e-3 of a single bf16 rounding
    // (SURVEY §0.6), at twice the tensor work (config 2: 33 vs 20 us per step).
    // bf16 outputs keep the single rounding (the W-resident pair kernel below): the output's
    // own bf16 rounding (2^-9 relative per element) is of the same size as W's.
    const int64_t qp = round_up(g.q, 64);
    __nv_bfloat16 *w2 =
        reinterpret_cast<__nv_bfloat16 *>(ws + (pipe ? pipeline_slot(ws) : 0) * slot_bytes);
    char *xws = ws + 2 * slot_bytes;
    const void *xt = x;
    int64_t ldx = g.q;
    if (x_dtype != DT_BF16 || (g.q % 8) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
      ldx = ldw;
      if (int rc = launch_pack_x(batch, g.q, ldx, x, x_dtype, xws, st)) return rc;
      xt = xws;
    }
    RegenArgs rg{};
    rg.q = g.q; rg.r_dim = g.r_dim; rg.ldw = 2 * qp;
    rg.rank = (int)g.rank; rg.n = (int)g.n;
    rg.a_rows = (int)((g.q * g.r_dim + g.n - 1) / g.n);
    rg.f_dtype = f_dtype;
    rg.xf = xf; rg.wf = wf; rg.wt = w2;
    rg.chain = pipe ? 1 : 0;
    rg.hilo = 1;
    rg.qp = (int)qp;
    if (int rc = launch_regen_wt(rg, st)) return rc;  // pipelined: overlaps the previous forward's GEMM
    XGemm xg;
    // K = qp with the lo half riding in the same stages (dual A): x is read once per tile
    xg.M = g.r_dim; xg.N = batch; xg.K = qp;
    xg.A = w2; xg.lda = 2 * qp; xg.a_mn = 0;
    xg.dual_k = qp;
    xg.B = xt; xg.ldb = ldx; xg.b_mn = 0; xg.b_rows = g.q;
    xg.el = 0;
    xg.BN = 256;
    xg.epi = 4;  // transposed store: y[b][j] = act(D[j][b] + bias[j])
    xg.out_t = y; xg.ldo = g.r_dim;
    xg.y_dtype = y_dtype;
    xg.act = act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act;
    xg.act_arg = act_arg;
    xg.bias = bias;
    xg.chain = pipe ? 1 : 0;
    if (int rc = xgemm(xg, st)) return rc;
    if (act == DT_ACT_SOFTMAX) return launch_row_softmax(batch, g.r_dim, y, y_dtype, st);
    return DT_OK;
  }
  __nv_bfloat16 *wt =
      reinterpret_cast<__nv_bfloat16 *>(ws + (pipe ? pipeline_slot(ws) : 0) * slot_bytes);
  char *xws = ws + 2 * slot_bytes;
  // TMA needs a bf16 x whose base and row pitch are 16-byte aligned.
  const void *xt = x;
  int64_t ldx = g.q;
  if (x_dtype != DT_BF16 || (g.q % 8) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
    ldx = ldw;
    if (int rc = launch_pack_x(batch, g.q, ldx, x, x_dtype, xws, st)) return rc;
    xt = xws;
  }
  RegenArgs rg{};
  rg.q = g.q; rg.r_dim = g.r_dim; rg.ldw = ldw;
  rg.rank = (int)g.rank; rg.n = (int)g.n;
  rg.a_rows = (int)((g.q * g.r_dim + g.n - 1) / g.n);
  rg.f_dtype = f_dtype;
  rg.xf = xf; rg.wf = wf; rg.wt = wt;
  rg.chain = pipe ? 1 : 0;
  rg.x_ext = forward_pipeline_external_x() ? 1 : 0;
  GemmCall c{xt, ldx, batch, g.q, wt, ldw, g.r_dim, bias, act, act_arg,
             y, g.r_dim, y_dtype, &rg, true};
  if (mse) {
    c.target = mse->target; c.scale = mse->scale; c.loss_part = mse->part;
    c.n_part = &n_part;
  }
  return finish_mse(run_gemm(c, st));
}


// Backward of reuse geometries on the tensor cores: k_train.cu (our tcgen05 GEMMs throughout).
bool tc_backward_ok(const Geo &g) { return xtrain_ok(g); }

size_t tc_backward_ws(const Geo &g, int64_t batch) { return xtrain_backward_ws(g, batch); }

int tc_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                const float *wf, const float *bias, int act, float act_arg,
                const float *up, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                char *ws, size_t ws_bytes, cudaStream_t st, const float *p_in) {
  if (!tc_backward_ok(g)) {
    set_error("tensor-core backward: reuse geometries with n % 8 == 0, rank % 4 == 0, rank <= 128");
    return DT_E_UNSUPPORTED;
  }
  return xtrain_backward(g, batch, x, x_dtype, xf, wf, bias, act, act_arg, up, d_xf, d_wf, d_bias,
                         d_input, ws, ws_bytes, st, p_in);
}

}  // namespace dt
