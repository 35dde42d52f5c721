// Fused layer chain: several reuse-geometry DeepThin layers (n_f | q) in ONE persistent kernel,
// each 128-row tile carried through every layer without its activations leaving the SM cluster.
//
// Reference: the network forward runs layer_forward per layer (kernel.py:296-320; the reference
// model runs its layers one after another, model_io.py:46-63), each the reuse identity of
// kernel.py:1-16. Per layer and tile this is the row-tile kernel's arithmetic (k_tc_rows.cu):
//
//   phase A  P[b, seg, k] = x[b, seg*n : (seg+1)*n] . wf[k]     bf16 (wf hi + lo), fp32 in TMEM
//   phase B  y[b, j] = act(P2[b, :] . XF2[j, :] (+ bias))      tf32, XF2 = xf viewed (r_dim x s*r)
//
// B200 design: a cluster of cs CTAs owns a row tile. CTA c contracts the input segments
// seg = c, c + cs, ... and — for every hidden layer — computes exactly the output columns that
// form those same segments of the NEXT layer's input (chunks seg*n/128 ... of 128 columns). So
// the epilogue writes each hidden layer's activations (bias + sigmoid + bf16) straight into the
// CTA's own shared-memory activation buffer, in the 128B-swizzled K-major layout the next
// layer's phase-A MMAs read. Only P crosses the cluster (distributed shared memory bulk copies,
// as in the row-tile kernel). HBM sees the chain's input once and its last layer's output once:
// for config 3's layers 1-6 that is 64 + 98 MB instead of 6 x (64 + 64..98) MB.
//
// Per CTA (cs = 4, s = 8, n = 256): activation buffer 2 segments x 4 k-blocks x 16 KB = 128 KB
// (also the TMA destination of the chain's input tile), A2 (the tf32 P operand) 2 x 16 KB, wf
// ring 2 x 8 KB, XF2 chunk ring 2 x 16 KB. The next tile's input loads as soon as the last
// layer's phase A has read the buffer (act_free), overlapping that layer's exchange, phase B
// and epilogue.
//
// Warp roles (as k_tc_rows.cu): 0 input TMA producer, 1 wf / XF2 producer, 2 TMEM owner + MMA
// issuer, 3-6 P exchange, 7-22 epilogue (16 warps: TMEM lane quarter = warp % 4, 32 of each
// chunk's 128 columns).

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

// This (opt-in, measured-slower) kernel keeps the bounded mbarrier waits: with the bare
// try_wait loops of sm100_ptx.cuh its layer-chain test hangs (a wait that never completes —
// a phase race in this kernel's single-buffered activation hand-off that the slower bounded
// waits do not expose; unresolved). The bounded loops also turn any such hang into a trap.
#define DEEPTHIN_BOUNDED_WAITS 1
#include "act.cuh"
#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

constexpr int cTM = 128;                    // rows per tile (UMMA M, TMEM lanes)
constexpr int cNc = 128;                    // output columns per chunk (phase-B UMMA N)
constexpr int cPW = 4, cEpi = 16;
constexpr int cThreads = 32 * (3 + cPW + cEpi);
constexpr uint32_t cKB = cTM * 128;         // one 64-column bf16 k-block of the tile (16 KB)
constexpr uint32_t cB = cNc * 128;          // one XF2 chunk: 128 columns x 32 fp32 (16 KB)
constexpr uint32_t cA2 = cTM * 128;         // tf32 P operand: 128 rows x 32 fp32 (16 KB)
constexpr uint32_t cDCol = 256;             // TMEM column of the first D buffer
constexpr int cMaxL = 8;

struct ChainMaps {
  CUtensorMap x;             // chain input (batch x q0 bf16), box 64 x 128, SW128
  CUtensorMap wf[cMaxL];     // per layer: [wf_hi; wf_lo] (2r x n bf16), box 64 x np, SW128
  CUtensorMap xf2[cMaxL];    // per layer: XF2p (r_dim x k2 fp32), box 32 x 128, SW128
};

struct ChainParams {
  int64_t batch;
  int L, n_tiles, cs, s, nkb, np, rank, rp, k2, bslot;
  int r_dim[cMaxL];
  int sps;                   // segments per CTA (s / cs)
  void *y;                   // last layer output (batch x r_dim[L-1], bf16)
  float arg;
  uint32_t off_act, off_a2, off_wf, off_b, off_bar;
  unsigned long long *trace;  // DEEPTHIN_CHAIN_TRACE (timing builds): stamps of cluster 0
};

constexpr int cTr = 6 * 40;  // per CTA: 6 stamps x 40 layer steps
__device__ __forceinline__ void ctrace(const ChainParams &p, int step, int k) {
  if (kTimingSwitches && p.trace && blockIdx.x < 4 && step < 40) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * cTr + step * 6 + k] = t;
  }
}

__device__ __forceinline__ uint32_t a2n_off_c(int row, int kk) {  // as k_tc_rows.cu a2n_off
  return (uint32_t)(kk >> 2) * 2048u + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u +
         (uint32_t)(kk & 3) * 4u;
}
__device__ __forceinline__ void bulk_s2c_c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                           uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}
// hidden-layer activation on bf16 outputs: the prepared operands pre-scale a sigmoid layer's
// contraction and bias by 1/2, so sigmoid = 1/2 + tanh(z/2)/2 is one MUFU op (as k_tc_rows.cu)
template <int ACT>
__device__ __forceinline__ float act_out_chain(float z, float arg) {
  if constexpr (ACT == DT_ACT_SIGMOID) return fmaf(0.5f, tanh_approx(z), 0.5f);
  return act_out_bf16<DT_BF16, ACT>(z, arg);
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}

// Owned output chunks of CTA c in layer l: hidden layers own the chunks that form this CTA's
// input segments of layer l+1 (segment seg = c + k*cs -> chunks seg*cps .. seg*cps + cps - 1,
// cps = n / 128); the last layer owns chunks c, c + cs, ...
__device__ __forceinline__ int owned_chunks(const ChainParams &p, int l, int crank) {
  if (l < p.L - 1) return p.sps * (p.nkb / 2);
  const int nch = (p.r_dim[l] + cNc - 1) / cNc;
  return crank < nch ? (nch - crank + p.cs - 1) / p.cs : 0;
}
__device__ __forceinline__ int chunk_id(const ChainParams &p, int l, int crank, int k) {
  if (l < p.L - 1) {
    const int cps = p.nkb / 2;
    return (crank + (k / cps) * p.cs) * cps + (k % cps);
  }
  return crank + k * p.cs;
}

template <int ACT>
__global__ void __launch_bounds__(cThreads, 1)
    k_tc_chain(const __grid_constant__ ChainMaps tm, const ChainParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *xk_full = bars;                    // [16] input k-block landed (one phase per tile)
  uint64_t *act_full = xk_full + 16;           // hidden layer written by the epilogue (cEpi)
  uint64_t *act_free = act_full + 1;           // last layer's phase A read the buffer
  uint64_t *wf_full = act_free + 1, *wf_empty = wf_full + 2;
  uint64_t *b_full = wf_empty + 2, *b_empty = b_full + 2;
  uint64_t *d_full = b_empty + 2, *d_empty = d_full + 2;
  uint64_t *a2_full = d_empty + 2, *a2_free = a2_full + 2;
  uint64_t *p_full = a2_free + 2, *p_empty = p_full + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(p_empty + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int cs = p.cs;
  const int crank = cs > 1 ? (int)cluster_ctarank() : 0;
  const int cid = (int)blockIdx.x / cs, ncl = (int)gridDim.x / cs;
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  const int nkb_act = p.sps * p.nkb;           // k-blocks of this CTA's activation buffer
  const int ntl = cid < p.n_tiles ? (p.n_tiles - cid + ncl - 1) / ncl : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&xk_full[i], 1);
    mbar_init(act_full, cEpi);
    mbar_init(act_free, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&wf_full[i], 1); mbar_init(&wf_empty[i], 1);
      mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1);
      mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], cEpi);
      mbar_init(&a2_full[i], 1); mbar_init(&a2_free[i], cs);
    }
    mbar_init(p_full, 1);
    mbar_init(p_empty, cPW);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm.x);
    for (int l = 0; l < p.L; ++l) { tma_prefetch_desc(&tm.wf[l]); tma_prefetch_desc(&tm.xf2[l]); }
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  griddep_wait();  // the chain's input is the previous kernel's output
  griddep_launch_dependents();

  const uint32_t s0 = smem_u32(smem);
  if (warp == 0) {
    // ---------------- input producer: this CTA's segments of each tile, into the act buffer ---
    if (lane == 0) {
      int i = 0;
      for (int t = cid; t < p.n_tiles; t += ncl, ++i) {
        if (i > 0) mbar_wait(act_free, (uint32_t)(i - 1) & 1u);  // last layer of tile i-1 read it
        for (int j = 0; j < p.sps; ++j)
          for (int kb = 0; kb < p.nkb; ++kb) {
            const int a = j * p.nkb + kb, seg = crank + j * cs;
            mbar_arrive_expect_tx(&xk_full[a], cKB);
            tma_load_2d(smem + p.off_act + a * cKB, &tm.x, &xk_full[a], seg * p.nkb * 64 + kb * 64,
                        t * cTM);
          }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- operand producer: wf per layer, then the layer's owned XF2 chunks -------
    if (lane == 0) {
      int ws = 0, bs = 0;
      uint32_t wph = 0, bph = 0;
      const uint32_t wbytes = (uint32_t)(p.nkb * p.np * 128);
      for (int i = 0; i < ntl; ++i)
        for (int l = 0; l < p.L; ++l) {
          mbar_wait(&wf_empty[ws], wph ^ 1);
          mbar_arrive_expect_tx(&wf_full[ws], wbytes);
          for (int kb = 0; kb < p.nkb; ++kb)
            tma_load_2d(smem + p.off_wf + ws * wbytes + kb * p.np * 128, &tm.wf[l], &wf_full[ws],
                        kb * 64, 0);
          if (++ws == 2) { ws = 0; wph ^= 1; }
          const int oc = owned_chunks(p, l, crank);
          for (int k = 0; k < oc; ++k) {
            mbar_wait(&b_empty[bs], bph ^ 1);
            mbar_arrive_expect_tx(&b_full[bs], cB);
            tma_load_2d(smem + p.off_b + bs * cB, &tm.xf2[l], &b_full[bs], 0,
                        chunk_id(p, l, crank, k) * cNc);
            if (++bs == 2) { bs = 0; bph ^= 1; }
          }
        }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idA = idesc_f32acc(cTM, (uint32_t)p.np, 1);
      const uint32_t idB = idesc_f32acc(cTM, cNc, 2);
      const uint32_t wbytes = (uint32_t)(p.nkb * p.np * 128);
      int ws = 0, bs = 0, db = 0;
      uint32_t wph = 0, bph = 0, dph = 0, afph = 0, peph = 0;
      int step = 0;  // global layer step (tile i, layer l): A2 buffer parity
      for (int i = 0; i < ntl; ++i) {
        for (int l = 0; l < p.L; ++l, ++step) {
          // phase A: P of this CTA's segments (TMEM columns [0, sps*np)), once the P warps have
          // read the previous step's P out of TMEM
          if (step > 0) { mbar_wait(p_empty, peph); peph ^= 1; }
          mbar_wait(&wf_full[ws], wph);
          if (l > 0) { mbar_wait(act_full, afph); afph ^= 1; }
          ctrace(p, step, 0);
          tc_fence_after();
          const uint32_t wf_s = s0 + p.off_wf + (uint32_t)ws * wbytes;
          for (int j = 0; j < p.sps; ++j) {
            const uint32_t d = tbase + (uint32_t)(j * p.np);
            for (int kb = 0; kb < p.nkb; ++kb) {
              const int a = j * p.nkb + kb;
              if (l == 0) mbar_wait(&xk_full[a], (uint32_t)i & 1u);
              tc_fence_after();
              const uint32_t as = s0 + p.off_act + (uint32_t)a * cKB;
              const uint32_t bsw = wf_s + (uint32_t)(kb * p.np * 128);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(d, smem_desc(as + k * 32, 16, 1024, SL_SW128),
                            smem_desc(bsw + k * 32, 16, 1024, SL_SW128), idA, (kb | k) != 0);
            }
          }
          mma_commit(&p_full[0]);
          mma_commit(&wf_empty[ws]);
          if (++ws == 2) { ws = 0; wph ^= 1; }
          if (l == p.L - 1) mma_commit(act_free);  // the next tile's input may land
          // phase B: every cluster CTA's P landed in A2[step & 1]
          const int ab = step & 1;
          mbar_wait_cluster(&a2_full[ab], (uint32_t)(step >> 1) & 1u);
          ctrace(p, step, 2);
          tc_fence_after();
          const uint32_t a2_s = s0 + p.off_a2 + (uint32_t)ab * cA2;
          const int oc = owned_chunks(p, l, crank);
          for (int k = 0; k < oc; ++k) {
            mbar_wait(&b_full[bs], bph);
            mbar_wait(&d_empty[db], dph ^ 1);
            tc_fence_after();
            const uint32_t d = tbase + cDCol + (uint32_t)(db * cNc);
            const uint32_t b = s0 + p.off_b + (uint32_t)bs * cB;
            for (int k8 = 0; k8 < p.k2 / 8; ++k8)
              mma_tf32_ss(d, smem_desc(a2_s + k8 * 4096, 2048, 128, SL_NONE),
                          smem_desc(b + k8 * 32, 16, 1024, SL_SW128), idB, k8 != 0);
            mma_commit(&b_empty[bs]);
            if (++bs == 2) { bs = 0; bph ^= 1; }
            mma_commit(&d_full[db]);
            if (++db == 2) { db = 0; dph ^= 1; }
          }
          if (cs > 1) mma_commit_mc(&a2_free[ab], cmask); else mma_commit(&a2_free[ab]);
          ctrace(p, step, 3);
        }
      }
    }
    __syncwarp();
  } else if (warp < 3 + cPW) {
    // ---------------- P exchange: TMEM -> tf32 A operand of every cluster CTA ----------------
    const int sp = warp & 3, row = 32 * sp + lane;
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    const uint32_t a2_local = s0 + p.off_a2;
    for (int b = 0; b < 2; ++b)  // K padding of the tf32 operand (never overwritten)
      for (int kk = p.s * p.rp; kk < p.k2; kk += 4)
        sts_v4(a2_local + (uint32_t)b * cA2 + a2n_off_c(row, kk), kk == p.bslot ? 0x3f800000u : 0u,
               0u, 0u, 0u);
    uint32_t pph = 0;
    int step = 0;
    for (int i = 0; i < ntl; ++i)
      for (int l = 0; l < p.L; ++l, ++step) {
        const int ab = step & 1;
        mbar_wait(p_full, pph);
        pph ^= 1;
        if (warp == 3 && lane == 0) ctrace(p, step, 1);
        tc_fence_after();
        mbar_wait(&a2_free[ab], (uint32_t)((step >> 1) & 1) ^ 1u);
        const uint32_t a2b = a2_local + (uint32_t)ab * cA2;
        for (int j = 0; j < p.sps; ++j) {
          const int seg = crank + j * cs;
          const uint32_t pcol = tbase + lane_t + (uint32_t)(j * p.np);
          uint32_t vh[32], vl[32];
          tmem_ld_32x32b_x32(pcol, vh);
          tmem_ld_32x32b_x32(pcol + (uint32_t)p.rank, vl);
          tmem_ld_wait();
          if (j == p.sps - 1) {  // P read out: the next phase A may overwrite it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_empty);
          }
#pragma unroll
          for (int k0 = 0; k0 < 32; k0 += 4) {
            if (k0 < p.rp) {
              uint32_t w[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int k = k0 + q;
                w[q] = (k < p.rank) ? __float_as_uint(__uint_as_float(vh[k]) + __uint_as_float(vl[k]))
                       : (seg == 0 && k == p.bslot) ? 0x3f800000u : 0u;
              }
              sts_v4(a2b + a2n_off_c(row, seg * p.rp + k0), w[0], w[1], w[2], w[3]);
            }
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        named_bar_sync(1, 32 * cPW);
        if (warp == 3) {
          if (lane >= 1 && lane < cs) {
            const uint32_t peer = (uint32_t)((crank + lane) % cs);
            const uint32_t bar = mapa_shared(smem_u32(&a2_full[ab]), peer);
            for (int j = 0; j < p.sps; ++j) {
              const int seg = crank + j * cs;
              for (int c4 = seg * p.rp / 4; c4 < (seg + 1) * p.rp / 4; ++c4) {
                const uint32_t src = a2b + (uint32_t)c4 * 2048u;
                bulk_s2c_c(mapa_shared(src, peer), src, 2048u, bar);
              }
            }
          }
          if (lane == 0) {
            const int own = p.sps * (p.rp / 4);
            mbar_arrive_expect_tx(&a2_full[ab], (uint32_t)(p.s * p.rp / 4 - own) * 2048u);
          }
          __syncwarp();
        }
      }
  } else {
    // ---------------- epilogue: hidden layers -> act buffer (smem), last layer -> y ----------
    const int sp = warp & 3;
    const int e = warp - 3 - cPW;
    const int qc = e / 4;               // which 32 columns of each 128-column chunk
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    const int row_in_tile = 32 * sp + lane;
    int db = 0;
    uint32_t dph = 0;
    int step = 0;
    for (int i = 0; i < ntl; ++i) {
      const int t = cid + i * ncl;
      const int64_t row = (int64_t)t * cTM + row_in_tile;
      for (int l = 0; l < p.L; ++l, ++step) {
        const bool last = l == p.L - 1;
        const int oc = owned_chunks(p, l, crank);
        for (int k = 0; k < oc; ++k) {
          mbar_wait(&d_full[db], dph);
          if (e == 0 && lane == 0 && k == 0) ctrace(p, step, 5);
          tc_fence_after();
          uint32_t v[32];
          tmem_ld_32x32b_x32(tbase + lane_t + cDCol + (uint32_t)(db * cNc + 32 * qc), v);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[db]);
          if (++db == 2) { db = 0; dph ^= 1; }
          float o[32];
          if (!last) {
#pragma unroll
            for (int q = 0; q < 32; ++q) o[q] = act_out_chain<ACT>(__uint_as_float(v[q]), p.arg);
            // into the act buffer: this CTA's segment j = k / cps, 128-column half hh = k % cps,
            // 64-column k-block kb = hh * 2 + qc / 2, 16-byte chunks (qc % 2) * 4 .. + 3
            const int cps = p.nkb / 2, j = k / cps, hh = k % cps;
            const int kb = hh * 2 + (qc >> 1);
            const uint32_t base = s0 + p.off_act + (uint32_t)(j * p.nkb + kb) * cKB +
                                  (uint32_t)row_in_tile * 128u;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int c16 = (qc & 1) * 4 + c;
              const float *f = o + 8 * c;
              sts_v4(base + ((uint32_t)(c16 ^ (row_in_tile & 7)) << 4), pack2(f[0], f[1]),
                     pack2(f[2], f[3]), pack2(f[4], f[5]), pack2(f[6], f[7]));
            }
          } else {
            const int col0 = chunk_id(p, l, crank, k) * cNc + 32 * qc;
            const int rd = p.r_dim[l];
            if (col0 < rd && row < p.batch) {
#pragma unroll
              for (int q = 0; q < 32; ++q) o[q] = __uint_as_float(v[q]);
              __nv_bfloat16 *yp = reinterpret_cast<__nv_bfloat16 *>(p.y) + row * rd + col0;
              if (col0 + 32 <= rd) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                  const float *f = o + 8 * c;
                  reinterpret_cast<uint4 *>(yp)[c] = make_uint4(pack2(f[0], f[1]), pack2(f[2], f[3]),
                                                                pack2(f[4], f[5]), pack2(f[6], f[7]));
                }
              } else {
                for (int q = 0; q < 32 && col0 + q < rd; ++q) yp[q] = __float2bfloat16_rn(o[q]);
              }
            }
          }
        }
        if (!last) {  // this warp's share of the next layer's input is in shared memory
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(act_full);
        }
        if (e == 0 && lane == 0) ctrace(p, step, 4);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

using ChainFn = void (*)(ChainMaps, ChainParams);

}  // namespace

bool tc_chain_ok(const Geo *g, int L) {
  if (L < 2 || L > cMaxL) return false;
  for (int l = 0; l < L; ++l) {
    if (!g[l].reuse || g[l].n != g[0].n || g[l].s != g[0].s || g[l].rank != g[0].rank) return false;
    if (!tc_rows_ok(g[l], DT_BF16, DT_BF16)) return false;
    if (l > 0 && g[l].q != g[l - 1].r_dim) return false;
  }
  const int cs = 4;
  return g[0].n % 128 == 0 && g[0].s % cs == 0 && g[0].r_dim % 8 == 0 &&
         (g[0].s / cs) * (g[0].n / 64) <= 16;
}

int tc_chain_forward(const Geo *g, int L, int64_t batch, const void *x, void *const *prepared,
                     int hidden_act, float act_arg, void *y, cudaStream_t st) {
  if (!tc_chain_ok(g, L)) {
    set_error("layer chain: geometry not eligible (reuse layers sharing n, s, rank; q = previous r_dim)");
    return DT_E_UNSUPPORTED;
  }
  if (batch == 0) return DT_OK;
  ChainParams p{};
  p.batch = batch;
  p.L = L;
  p.n_tiles = (int)((batch + cTM - 1) / cTM);
  p.cs = 4;
  p.s = (int)g[0].s;
  p.nkb = (int)(g[0].n / 64);
  p.sps = p.s / p.cs;
  p.rank = (int)g[0].rank;
  p.np = (int)((2 * g[0].rank + 15) / 16 * 16);
  p.rp = (int)((g[0].rank + 3) / 4 * 4);
  p.k2 = (int)((g[0].s * p.rp + 7) / 8 * 8);
  p.bslot = g[0].rank < p.rp ? (int)g[0].rank : (p.k2 > g[0].s * p.rp ? (int)(g[0].s * p.rp) : -1);
  for (int l = 0; l < L; ++l) p.r_dim[l] = (int)g[l].r_dim;
  p.y = y;
  p.arg = act_arg;
  const uint32_t wbytes = (uint32_t)(p.nkb * p.np * 128);
  p.off_act = 0;
  p.off_a2 = (uint32_t)(p.sps * p.nkb) * cKB;
  p.off_wf = p.off_a2 + 2 * cA2;
  p.off_b = (p.off_wf + 2 * wbytes + 1023) & ~1023u;
  p.off_bar = p.off_b + 2 * cB;
  const uint32_t smem_bytes = p.off_bar + 512 + 1024;
  if (smem_bytes > 227 * 1024) {
    set_error("layer chain: shared memory budget exceeded");
    return DT_E_UNSUPPORTED;
  }
  ChainMaps tm;
  memset(&tm, 0, sizeof(tm));
  if (int rc = encode_tensor_map_2d(&tm.x, DT_BF16, const_cast<void *>(x), (uint64_t)g[0].q,
                                    (uint64_t)batch, (uint64_t)g[0].q * 2, 64, cTM, true))
    return rc;
  for (int l = 0; l < L; ++l) {
    char *ws = reinterpret_cast<char *>(prepared[l]);
    const int64_t wfb = (2 * g[l].rank * g[l].n * 2 + 255) / 256 * 256;
    if (int rc = encode_tensor_map_2d(&tm.wf[l], DT_BF16, ws, (uint64_t)g[l].n,
                                      (uint64_t)(2 * g[l].rank), (uint64_t)g[l].n * 2, 64,
                                      (uint32_t)p.np, true))
      return rc;
    if (int rc = encode_tensor_map_2d(&tm.xf2[l], DT_F32, ws + wfb, (uint64_t)p.k2,
                                      (uint64_t)g[l].r_dim, (uint64_t)p.k2 * 4, 32, cNc, true))
      return rc;
  }
  ChainFn fn;
  switch (hidden_act) {
    case DT_ACT_SIGMOID: fn = k_tc_chain<DT_ACT_SIGMOID>; break;
    case DT_ACT_RELU: fn = k_tc_chain<DT_ACT_RELU>; break;
    case DT_ACT_TANH: fn = k_tc_chain<DT_ACT_TANH>; break;
    case DT_ACT_CLIPPED_RELU: fn = k_tc_chain<DT_ACT_CLIPPED_RELU>; break;
    default: fn = k_tc_chain<DT_ACT_IDENTITY>; break;
  }
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(cThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)p.cs;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, int> occ;
  int max_cl = 0;
  {
    int dev = 0;
    DT_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    int &slot = occ[{dev, reinterpret_cast<const void *>(fn)}];
    if (!slot) {
      cfg.gridDim = dim3((unsigned)(p.cs * 64));
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        n = nsm / p.cs;
      }
      slot = n;
    }
    max_cl = slot;
  }
  const int ncl = std::max(1, std::min(p.n_tiles, max_cl));
  cfg.gridDim = dim3((unsigned)(ncl * p.cs));
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_CHAIN_TRACE") != 0;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&p.trace, 4 * cTr * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, 4 * cTr * 8, st));
  }
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm, p));
  if (tracing) {
    std::vector<unsigned long long> h(4 * cTr);
    DT_CUDA_CHECK(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFree(p.trace);
    unsigned long long t0 = ~0ull;
    for (auto v : h) if (v && v < t0) t0 = v;
    fprintf(stderr, "chain trace: %d clusters x %d, %d tiles, %d layers (us: A-issue P-seen A2-seen B-issued epi-first epi-done)\n",
            ncl, p.cs, p.n_tiles, p.L);
    for (int b = 0; b < 4; ++b) {
      fprintf(stderr, " cta %d:\n", b);
      for (int s2 = 0; s2 < 40; ++s2) {
        const unsigned long long *r = &h[b * cTr + s2 * 6];
        if (!r[0]) continue;
        fprintf(stderr, "  step %2d:", s2);
        for (int k : {0, 1, 2, 3, 5, 4}) fprintf(stderr, " %7.2f", r[k] ? (r[k] - t0) * 1e-3 : -1.0);
        fprintf(stderr, "\n");
      }
    }
  }
  return check_launch("tc_chain");
}

}  // namespace dt
