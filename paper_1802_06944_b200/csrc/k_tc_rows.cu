// Row-tile tensor-core forward for reuse geometries (n_f | q): the factored DeepThin layer in
// ONE persistent kernel, batch rows on the MMA M axis, output written through TMA stores.
//
// Reference: kernel.py:1-16 / 99-164 (the reuse identity: every output column reads s = q/n
// whole rows of I = xf @ wf, so each distinct run dot x_seg . wf[k] is computed once) and
// kernel.py:296-320 (layer_forward = act(x W + b)). In BASELINE notation, per 128-row tile:
//
//   phase A:  P[b, seg, k] = sum_t x[b, seg*n + t] * wf[k, t]        (bf16 x bf16 -> fp32, TMEM)
//   phase B:  y[b, j] = act(sum_{seg,k} xf[j*s + seg, k] * P[b, seg, k] + bias[j])
//             = act(P2[b, :] . XF2[j, :] + bias[j]),  XF2 = xf viewed (r_dim x s*rank)
//             (kind::tf32 on the fp32 P and the fp32 master xf, fp32 accumulate)
//
// No W and no P ever touch HBM: per row the kernel reads q bf16 inputs and writes r_dim
// outputs, so it is HBM-bound (config 3: 8 KB per row per 2048-wide layer, ~13 flop/B).
//
// A cluster of cs CTAs (8 when s allows) shares each 128-row tile: CTA c contracts only
// segments c, c+cs, ... (so x is read from HBM exactly once and every SM streams), broadcasts
// its P values into the tf32 A operand of every cluster CTA through distributed shared memory,
// then computes and stores output chunks c, c+cs, ... Clusters are persistent over tiles.
//
// Warp roles (768 threads, one CTA per SM):
//   warp 0  TMA producer of x k-blocks (128 rows x 64 bf16, SW128) into a ring sized to the
//           shared memory left (5-8 deep)
//   warp 1  TMA producer of XF2 chunks (128 output columns x 32 fp32, SW128), 2-deep ring
//   warp 2  TMEM allocator + single-thread tcgen05.mma issuer of phase A
//   warps 3-6  P exchange: P (TMEM) -> tf32 A operand of every cluster CTA (DSMEM bulk copies)
//   warps 7-22 epilogue: D chunks (TMEM, double-buffered 2 x 128 columns) -> bias +
//           activation -> bf16/fp32 -> swizzled shared staging -> TMA store (each warp its
//           own 32 x 32 box)
//   warp 23 single-thread tcgen05.mma issuer of phase B (decoupled from phase A: B of tile i
//           never waits for tile i+1's x, A of tile i+1 never waits for the epilogue)
#include <cuda_bf16.h>

#include <algorithm>
#include <unordered_map>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "act.cuh"
#include "dt_internal.h"
#include "rows_common.cuh"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;
using namespace rowsdev;

constexpr int kTM = 128;           // batch rows per tile (UMMA M = TMEM lanes)
constexpr int kNc = 128;           // output columns per D chunk (UMMA N of phase B)
constexpr int kXSMax = 8;          // x ring depth cap (the launcher sizes it to the smem left)
constexpr int kBS = 2;             // XF2 chunk ring depth (resident when a CTA has <= 2 chunks)
constexpr int kPW = 4;             // P-exchange warps (one per TMEM lane quarter)
constexpr int kEpi = 16;           // epilogue warps (four per TMEM lane quarter)
constexpr int kBWarp = 3 + kPW + kEpi;  // the phase-B MMA issuer (last warp)
constexpr int kRowsThreads = 32 * (4 + kPW + kEpi);
constexpr uint32_t kXBytes = kTM * 128;   // 128 rows x 64 bf16
constexpr uint32_t kBBytes = kNc * 128;   // 128 columns x 32 fp32
constexpr uint32_t kA2Bytes = kTM * 128;  // 128 rows x 32 fp32 (k2 <= 32)
// A2 descriptor strides (see a2n_off)
constexpr uint32_t kA2Lbo = 2048, kA2Sbo = 128;

struct RowsParams {
  int64_t batch;
  int r_dim, n_tiles, s, nkb, np, rank, rp, k2, n_chunks, cs, xs, pcols;
  const float *bias;
  void *y;
  float arg;
  int softmax;         // fused row softmax over the full output width (see the epilogue)
  int tma_y;           // epilogue stores through TMA (tm_y, 32 x 32 boxes) instead of st.global
  int nd;              // D buffers in TMEM (2-3, 128 columns each, from column dcol0)
  uint32_t dcol0;
  int nstage;          // output staging boxes per epilogue warp (1-2, TMA stores in flight)
  int wide;            // bf16 TMA epilogue in two teams of 8 warps on alternate chunks, each warp
                       // 32 rows x 64 columns per chunk: 128-byte rows per TMA store request
  uint32_t off_sm;     // softmax: 2 x cs x 128 (max, sum) cluster partials
  uint32_t off_red;    // softmax: [4][128] column-warp partials
  int bslot;  // K slot carrying the bias (P = 1 there, XF2p = bias * scale), -1: epilogue adds it
  uint32_t off_x, off_a2, off_wf, off_b, off_out, off_bar;
  unsigned long long *trace;  // DEEPTHIN_ROWS_TRACE: globaltimer stamps of cluster 0
  // layer chaining (dt_rows_chain): x row tile t is loaded once wait_flags[t] >= wait_target
  // (the previous layer's epilogue warps post to it) instead of after the whole previous grid;
  // this layer's epilogue warps post their finished tiles to post_flags
  const unsigned *wait_flags;
  unsigned wait_target;
  unsigned *post_flags;
};

constexpr int kTr = 64;  // trace slots per CTA
__device__ __forceinline__ void rtrace(const RowsParams &p, int slot) {
  if (p.trace && slot < kTr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * kTr + slot] = t;
  }
}

// No-swizzle K-major layout of the 128-row x k2 tf32 A operand: core matrices of 8 rows x 16 B
// (4 K values); M-adjacent core matrices 128 B apart (SBO), K-adjacent 2 KB apart (LBO) — so
// every 4-K column block of all 128 rows is one contiguous 2 KB run (bulk-copyable).
__device__ __forceinline__ uint32_t a2n_off(int row, int kk) {
  return (uint32_t)(kk >> 2) * 2048u + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u +
         (uint32_t)(kk & 3) * 4u;
}
// shared::cta -> shared::cluster bulk copy, completion counted on the destination's mbarrier
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                         uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst_cluster),
      "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
      : "memory");
}

// Cluster of cs CTAs per 128-row tile. CTA c of the cluster:
//   * loads and contracts only its own segments seg = c, c + cs, ... (x read once from HBM);
//   * pushes its P values (rank per segment per row, padded to rp) into the tf32 A operand of
//     every cluster CTA with shared->shared bulk copies (A2 double-buffered by tile parity);
//   * computes and stores its own output chunks ch = c, c + cs, ... (128 columns each).
// Tiles are strided over the clusters (persistent); the MMA issuer runs phase A of tile i+1
// before phase B of tile i (P double-buffered in TMEM), so the exchange latency is hidden.
template <int YDT, int ACT>
__global__ void __launch_bounds__(kRowsThreads, 1)
    k_tc_rows_reuse(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_wf,
                    const __grid_constant__ CUtensorMap tm_xf2, const __grid_constant__ CUtensorMap tm_y,
                    const RowsParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *x_full = bars, *x_empty = bars + kXSMax;
  uint64_t *b_full = bars + 2 * kXSMax, *b_empty = b_full + kBS;
  uint64_t *d_full = b_empty + kBS, *d_empty = d_full + 4;
  uint64_t *a2_full = d_empty + 4, *a2_free = a2_full + 2;
  uint64_t *p_full = a2_free + 2, *wf_full = p_full + 2;
  uint64_t *sm_full = wf_full + 1;  // softmax partials of every cluster CTA landed (2, by tile)
  uint64_t *p_free = sm_full + 2;   // the P warps read P[i & 1] out of TMEM (2, by tile)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(p_free + 2);
  // (the shuffles make the warp index, the cluster rank and the TMEM base provably warp-uniform
  // for the compiler: the producer / issuer loops below run on all 32 lanes with only the
  // asynchronous instructions predicated on lane 0, so their operands stay in uniform registers
  // instead of a per-instruction ELECT / R2UR waterfall — ~200 -> ~40 clocks per MMA issue,
  // measured on the slab kernel, k_tc_slab.cu)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const bool l0 = lane == 0;
  const int cs = p.cs;
  const int crank = (int)(blockIdx.x & (unsigned)(cs - 1));  // rank in the cluster of cs (power of 2) along x
  const int cid = (int)blockIdx.x / cs, ncl = (int)gridDim.x / cs;
  const uint16_t cmask = (uint16_t)((1u << cs) - 1u);
  const int my_chunks = crank < p.n_chunks ? (p.n_chunks - crank + cs - 1) / cs : 0;
  const bool b_res = my_chunks <= kBS;  // XF2 chunks loaded once, resident for every tile

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.xs; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < kBS; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], p.wide ? kEpi / 2 : kEpi);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a2_full[i], 1);   // local arm (expect_tx of the peers' bytes)
      mbar_init(&a2_free[i], cs);  // every cluster CTA's MMAs on this buffer done
      mbar_init(&p_full[i], 1);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(wf_full, 1);
    mbar_init(&sm_full[0], 1);
    mbar_init(&sm_full[1], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wf);
    tma_prefetch_desc(&tm_xf2);
    if (p.tma_y) tma_prefetch_desc(&tm_y);
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // peers' barriers initialised before any remote copy/arrive
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tslot, 0);
  if (threadIdx.x == 0) rtrace(p, 0);
  // Everything below reads buffers an earlier kernel on the stream may write (x is the previous
  // layer's output; factors/bias may come from an SGD step): wait for it, let the next start.
  // (chained layers wait per row tile on the previous layer's flags instead, in the x producer)
  if (!p.wait_flags) griddep_wait();
  griddep_launch_dependents();
  if (threadIdx.x == 0) rtrace(p, 1);

  const int n = p.nkb * 64;
  if (warp == 0) {
    // ---------------- x producer: this CTA's segments of each tile ----------------
    {
      // wf (rank x n bf16, rows rank..np-1 zero-filled by TMA) stays resident: nkb blocks of
      // np rows x 128 B
      const uint32_t s0 = smem_u32(smem);
      if (l0) {
        mbar_arrive_expect_tx(wf_full, (uint32_t)(p.nkb * p.np * 128));
        for (int kb = 0; kb < p.nkb; ++kb)
          tma_load_2d_s(s0 + p.off_wf + (uint32_t)(kb * p.np * 128), &tm_wf, smem_u32(wf_full), kb * 64, 0);
      }
      int st = 0;
      uint32_t ph = 0;
      for (int t = cid; t < p.n_tiles; t += ncl) {
        if (p.wait_flags) {  // rows of tile t written (and released) by the previous layer
          uint32_t spins = 0;
          while (ld_acquire_u32(p.wait_flags + t) < p.wait_target) {
            if (++spins == (1u << 28)) {
              printf("deepthin: layer-chain flag timeout (tile %d)\n", t);
              __trap();
            }
          }
          fence_proxy_async_global();  // the TMA (async proxy) reads below see those writes
        }
        for (int seg = crank; seg < p.s; seg += cs)
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&x_empty[st], ph ^ 1);
            if (l0) {
              mbar_arrive_expect_tx(&x_full[st], kXBytes);
              tma_load_2d_s(s0 + p.off_x + (uint32_t)st * kXBytes, &tm_x, smem_u32(&x_full[st]),
                            seg * n + kb * 64, t * kTM);
            }
            if (++st == p.xs) { st = 0; ph ^= 1; }
          }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- XF2 chunk producer: this CTA's output chunks ----------------
    {
      const uint32_t s0 = smem_u32(smem);
      if (b_res) {
        int i = 0;
        for (int c = crank; c < p.n_chunks; c += cs, ++i)
          if (l0) {
            mbar_arrive_expect_tx(&b_full[i], kBBytes);
            tma_load_2d_s(s0 + p.off_b + (uint32_t)i * kBBytes, &tm_xf2, smem_u32(&b_full[i]), 0, c * kNc);
          }
      } else {
        int st = 0;
        uint32_t ph = 0;
        for (int t = cid; t < p.n_tiles; t += ncl)
          for (int pass = 0; pass < (p.softmax ? 2 : 1); ++pass)
          for (int c = crank; c < p.n_chunks; c += cs) {
            mbar_wait(&b_empty[st], ph ^ 1);
            if (l0) {
              mbar_arrive_expect_tx(&b_full[st], kBBytes);
              tma_load_2d_s(s0 + p.off_b + (uint32_t)st * kBBytes, &tm_xf2, smem_u32(&b_full[st]), 0, c * kNc);
            }
            if (++st == kBS) { st = 0; ph ^= 1; }
          }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ---------------- phase-A MMA issuer: P[i & 1] = x_seg . [wf_hi | wf_lo] ----------------
    // (phase B runs on its own issuer warp, so A of the next tiles never waits behind the
    // epilogue's D buffers, and B never waits for the next tile's x)
    {
      const uint32_t s0 = smem_u32(smem);
      const uint32_t idA = idesc_f32acc(kTM, (uint32_t)p.np, 1);
      const uint64_t descX0 = smem_desc(s0 + p.off_x, 16, 1024, SL_SW128);
      const uint64_t descW0 = smem_desc(s0 + p.off_wf, 16, 1024, SL_SW128);
      const uint32_t wstep = (uint32_t)(p.np * 128) >> 4;  // descriptor units per wf k-block
      mbar_wait(wf_full, 0);
      const int ntl = cid < p.n_tiles ? (p.n_tiles - cid + ncl - 1) / ncl : 0;
      int xs = 0;
      uint32_t xph = 0;
      for (int i = 0; i < ntl; ++i) {
        mbar_wait(&p_free[i & 1], ((uint32_t)(i >> 1) & 1u) ^ 1u);  // P warps read tile i-2
        tc_fence_after();
        const uint32_t pc = tbase + (uint32_t)((i & 1) * p.pcols);
        int j = 0;
        for (int seg = crank; seg < p.s; seg += cs, ++j) {
          const uint32_t d = pc + (uint32_t)(j * p.np);
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&x_full[xs], xph);
            if (l0 && kb == 0 && j == 0) rtrace(p, 2 + 5 * min(i, 9));
            if (l0 && kb == p.nkb - 1 && seg + cs >= p.s) rtrace(p, 3 + 5 * min(i, 9));
            tc_fence_after();
            const uint64_t a = descX0 + (uint64_t)((uint32_t)xs * (kXBytes >> 4));
            const uint64_t b = descW0 + (uint64_t)((uint32_t)kb * wstep);
            if (l0) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(d, a + (uint64_t)(2 * k), b + (uint64_t)(2 * k), idA, (kb | k) != 0);
              mma_commit(&x_empty[xs]);
            }
            if (++xs == p.xs) { xs = 0; xph ^= 1; }
          }
        }
        if (l0) mma_commit(&p_full[i & 1]);
      }
    }
    __syncwarp();
  } else if (warp == kBWarp) {
    // ---------------- phase-B MMA issuer: D = A2 . XF2 chunk (tf32) ----------------
    {
      const uint32_t s0 = smem_u32(smem);
      const uint32_t idB = idesc_f32acc(kTM, kNc, 2);
      const uint64_t descA20 = smem_desc(s0 + p.off_a2, kA2Lbo, kA2Sbo, SL_NONE);
      const uint64_t descXF0 = smem_desc(s0 + p.off_b, 16, 1024, SL_SW128);
      const int nk = p.k2 / 8;
      const int ntl = cid < p.n_tiles ? (p.n_tiles - cid + ncl - 1) / ncl : 0;
      int bs = 0, db = 0;
      uint32_t bph = 0, dph = 0;
      for (int tb = 0; tb < ntl; ++tb) {
        // every cluster CTA's P landed in A2[tb & 1]
        const int ab = tb & 1;
        mbar_wait_cluster(&a2_full[ab], (uint32_t)(tb >> 1) & 1u);
        if (l0) rtrace(p, 4 + 5 * min(tb, 9));
        tc_fence_after();
        const uint64_t a2d = descA20 + (uint64_t)((uint32_t)ab * (kA2Bytes >> 4));
        // softmax: two passes over the chunks (statistics, then normalised stores), the tf32
        // MMA recomputed from the A2 tile still resident — no logits round trip through HBM
        for (int pass = 0; pass < (p.softmax ? 2 : 1); ++pass) {
          int ci = 0;
          for (int c = crank; c < p.n_chunks; c += cs, ++ci) {
            const int slot = b_res ? ci : bs;
            mbar_wait(&b_full[slot], b_res ? 0u : bph);
            mbar_wait(&d_empty[db], dph ^ 1);
            tc_fence_after();
            const uint32_t d = tbase + p.dcol0 + (uint32_t)(db * kNc);
            const uint64_t b = descXF0 + (uint64_t)((uint32_t)slot * (kBBytes >> 4));
            if (l0) {
#pragma unroll
              for (int k = 0; k < 4; ++k)  // A2: 4 KB (256 descriptor units) per K step of 8
                if (k < nk) mma_tf32_ss(d, a2d + (uint64_t)(256 * k), b + (uint64_t)(2 * k), idB, k != 0);
              if (!b_res) mma_commit(&b_empty[bs]);
              mma_commit(&d_full[db]);
            }
            if (!b_res && ++bs == kBS) { bs = 0; bph ^= 1; }
            if (++db == p.nd) { db = 0; dph ^= 1; }
          }
        }
        // this CTA's reads of A2[ab] are done when these MMAs complete: tell every writer
        if (l0) {
          if (cs > 1) mma_commit_mc(&a2_free[ab], cmask); else mma_commit(&a2_free[ab]);
        }
      }
    }
    __syncwarp();
  } else if (warp < 3 + kPW) {
    // ---------------- P exchange: TMEM -> tf32 A operand of every cluster CTA ----------------
    const int sp = warp & 3, row = 32 * sp + lane;
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    const uint32_t a2_local = smem_u32(smem) + p.off_a2;
    for (int b = 0; b < 2; ++b)  // K padding of the tf32 operand (never overwritten)
      for (int kk = p.s * p.rp; kk < p.k2; kk += 4)
        st_shared_v4(a2_local + (uint32_t)b * kA2Bytes + a2n_off(row, kk),
                     kk == p.bslot ? 0x3f800000u : 0u, 0u, 0u, 0u);
    uint32_t it = 0;
    for (int t = cid; t < p.n_tiles; t += ncl, ++it) {
      const int ab = (int)(it & 1);
      mbar_wait(&p_full[ab], (it >> 1) & 1);
      tc_fence_after();
      mbar_wait(&a2_free[ab], ((it >> 1) & 1) ^ 1);  // all readers of tile it-2 finished
      const uint32_t a2b = a2_local + (uint32_t)ab * kA2Bytes;
      // own P values (rank padded to rp with zeros) into this CTA's A2[ab], one 16-byte store
      // per 4 K values
      int j = 0;
      for (int seg = crank; seg < p.s; seg += cs, ++j) {
        // columns [0, rank) hold x . wf_hi, [rank, 2 rank) x . wf_lo: two loads, the second
        // offset by rank columns, so P = hi + lo pairs up register by register
        const uint32_t pcol = tbase + lane_t + (uint32_t)(ab * p.pcols + j * p.np);
        uint32_t vh[32], vl[32];
        tmem_ld_32x32b_x32(pcol, vh);
        tmem_ld_32x32b_x32(pcol + (uint32_t)p.rank, vl);
        tmem_ld_wait();
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
          if (k0 < p.rp) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int k = k0 + i;
              w[i] = (k < p.rank) ? __float_as_uint(__uint_as_float(vh[k]) + __uint_as_float(vl[k]))
                     : (seg == 0 && k == p.bslot) ? 0x3f800000u : 0u;  // 1.0f
            }
            st_shared_v4(a2b + a2n_off(row, seg * p.rp + k0), w[0], w[1], w[2], w[3]);
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();  // visible to the local MMAs and to the bulk-copy engine
      named_bar_sync(1, 32 * kPW);
      if (warp == 3 && lane == 0) mbar_arrive(&p_free[ab]);  // P[ab] read out of TMEM
      if (warp == 3) {
        // lane r (1..cs-1) pushes this CTA's blocks into peer (crank + r) % cs, completion
        // counted on the peer's a2_full[ab]; lane 0 arms the local barrier for the peers' bytes
        if (lane >= 1 && lane < cs) {
          const uint32_t peer = (uint32_t)((crank + lane) % cs);
          const uint32_t bar = mapa_shared(smem_u32(&a2_full[ab]), peer);
          for (int seg = crank; seg < p.s; seg += cs)
            for (int c4 = seg * p.rp / 4; c4 < (seg + 1) * p.rp / 4; ++c4) {
              const uint32_t src = a2b + (uint32_t)c4 * 2048u;
              bulk_s2c(mapa_shared(src, peer), src, 2048u, bar);
            }
        }
        if (lane == 0) {
          const int own = ((p.s - crank + cs - 1) / cs) * (p.rp / 4);
          mbar_arrive_expect_tx(&a2_full[ab], (uint32_t)(p.s * p.rp / 4 - own) * 2048u);
        }
        __syncwarp();
      }
    }
  } else if (warp < kBWarp) {
    // ---------------- epilogue ----------------
    if (p.softmax) {
      // Fused row softmax (the output layer of config 3), two passes over the tile's chunks with
      // the tf32 contraction recomputed in between (the B issuer runs it twice):
      //   pass 1: per row, the online (max, sum 2^((z - max) log2 e)) over this warp's 32
      //           columns of every chunk of this CTA, combined over the four column warps in
      //           shared memory, then over the cluster: each CTA bulk-copies its 128 partials
      //           into every peer (completion on the peer's sm_full) and every CTA combines the
      //           cs partials in rank order (fixed order: deterministic);
      //   pass 2: p = 2^((z - M) log2 e) / L, staged and TMA-stored like the logits path.
      // The logits never leave the SM (one HBM write of p instead of z written, read, rewritten).
      const int sp = warp & 3, e = warp - 3 - kPW, qc = e / 4, row = 32 * sp + lane;
      const uint32_t s0 = smem_u32(smem);
      const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
      constexpr int E = YDT == DT_BF16 ? 2 : 4;
      constexpr int RB = 32 * E, SWM = RB / 16 - 1;
      const uint32_t out_s = s0 + p.off_out + (uint32_t)e * (32u * RB);
      float2 *red = reinterpret_cast<float2 *>(smem + p.off_red);  // [4][128]
      const float l2e = 1.4426950408889634f;
      int db = 0;
      uint32_t dph = 0, it = 0;
      for (int t = cid; t < p.n_tiles; t += ncl, ++it) {
        const int sb = (int)(it & 1);
        float2 *part = reinterpret_cast<float2 *>(smem + p.off_sm) + sb * cs * kTM;  // [cs][128]
        float m = -INFINITY, l = 0.f;
        for (int c = crank; c < p.n_chunks; c += cs) {
          mbar_wait(&d_full[db], dph);
          tc_fence_after();
          uint32_t v[32];
          tmem_ld_32x32b_x32(tbase + lane_t + p.dcol0 + (uint32_t)(db * kNc + 32 * qc), v);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[db]);
          if (++db == p.nd) { db = 0; dph ^= 1; }
          const int nv = min(32, p.r_dim - (c * kNc + 32 * qc));
          if (nv <= 0) continue;
          float cm = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nv) cm = fmaxf(cm, __uint_as_float(v[i]));
          const float nm = fmaxf(m, cm);
          float cl = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i < nv) cl += ex2_approx((__uint_as_float(v[i]) - nm) * l2e);
          l = (m > -INFINITY ? l * ex2_approx((m - nm) * l2e) : 0.f) + cl;
          m = nm;
        }
        red[qc * kTM + row] = make_float2(m, l);
        named_bar_sync(2, 32 * kEpi);
        if (qc == 0) {  // the CTA's partial for this row, column warps in order
          float M = -INFINITY, L = 0.f;
          for (int k = 0; k < 4; ++k) {
            const float2 q = red[k * kTM + row];
            if (q.x > -INFINITY) {
              const float nm = fmaxf(M, q.x);
              L = L * exp2f((M - nm) * l2e) + q.y * exp2f((q.x - nm) * l2e);
              M = nm;
            }
          }
          part[crank * kTM + row] = make_float2(M, L);
        }
        fence_proxy_async_smem();
        named_bar_sync(2, 32 * kEpi);
        if (warp == 3 + kPW) {
          if (lane >= 1 && lane < cs) {
            const uint32_t peer = (uint32_t)((crank + lane) % cs);
            const uint32_t src = smem_u32(part + crank * kTM);
            bulk_s2c(mapa_shared(src, peer), src, kTM * 8u,
                     mapa_shared(smem_u32(&sm_full[sb]), peer));
          }
          if (lane == 0) mbar_arrive_expect_tx(&sm_full[sb], (uint32_t)(cs - 1) * kTM * 8u);
          __syncwarp();
        }
        if (cs > 1) mbar_wait_cluster(&sm_full[sb], (it >> 1) & 1);
        float M = -INFINITY, L = 0.f;
        for (int k = 0; k < cs; ++k) {
          const float2 q = part[k * kTM + row];
          if (q.x > -INFINITY) {
            const float nm = fmaxf(M, q.x);
            L = L * exp2f((M - nm) * l2e) + q.y * exp2f((q.x - nm) * l2e);
            M = nm;
          }
        }
        const float inv = 1.f / L;  // the difference first below: exact near the max
        // pass 2: the recomputed chunks, normalised, through the staging box and TMA stores
        const int64_t row0 = (int64_t)t * kTM + 32 * sp;
        for (int c = crank; c < p.n_chunks; c += cs) {
          mbar_wait(&d_full[db], dph);
          tc_fence_after();
          uint32_t v[32];
          tmem_ld_32x32b_x32(tbase + lane_t + p.dcol0 + (uint32_t)(db * kNc + 32 * qc), v);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[db]);
          if (++db == p.nd) { db = 0; dph ^= 1; }
          const int col0 = c * kNc + 32 * qc;
          if (col0 >= p.r_dim) continue;
          float o[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = ex2_approx((__uint_as_float(v[i]) - M) * l2e) * inv;
          if (lane == 0) bulk_wait_group_read<0>();
          __syncwarp();
          const uint32_t rb = out_s + (uint32_t)lane * RB;
#pragma unroll
          for (int ch = 0; ch < RB / 16; ++ch) {
            uint32_t w0, w1, w2, w3;
            if constexpr (E == 2) {
              const float *f = o + ch * 8;
              w0 = pack_bf16(f[0], f[1]); w1 = pack_bf16(f[2], f[3]);
              w2 = pack_bf16(f[4], f[5]); w3 = pack_bf16(f[6], f[7]);
            } else {
              const float *f = o + ch * 4;
              w0 = __float_as_uint(f[0]); w1 = __float_as_uint(f[1]);
              w2 = __float_as_uint(f[2]); w3 = __float_as_uint(f[3]);
            }
            const int sw = E == 2 ? ((lane >> 1) & SWM) : (lane & SWM);
            st_shared_v4(rb + ((uint32_t)(ch ^ sw) << 4), w0, w1, w2, w3);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_y, smem + (out_s - s0), col0, (int32_t)row0);
            bulk_commit_group();
          }
        }
      }
      if (lane == 0) bulk_wait_group<0>();
    } else if (p.wide) {
      // bf16 outputs through TMA, two teams of 8 warps: team (n & 1) takes the CTA's n-th chunk
      // (= D buffer n & 1, nd == 2), a warp 32 rows (its TMEM lane quarter) x 64 columns of it in
      // two 32-column steps, staged as ONE 32 x 64 box of 128-byte rows: half the TMA store
      // requests of the 32-column boxes (fp32 outputs — 128-byte rows, twice the bytes — take
      // only 1.4x as long, which suggested a per-request cost), and the teams run out of phase
      // (one reads TMEM while the other computes and stores). Opt-in (DEEPTHIN_ROWS_WIDE=1):
      // measured no faster than the 32-column epilogue.
      const int sp = warp & 3;
      const int e = warp - 3 - kPW;      // 0..15
      const int team = (e >> 2) & 1, half = e >> 3;
      const uint32_t s0 = smem_u32(smem);
      const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
      const uint32_t out_s = s0 + p.off_out + (uint32_t)e * 4096u;  // 32 rows x 128 bytes
      const uint32_t rb = out_s + (uint32_t)lane * 128u;
      const uint32_t dcol = p.dcol0 + (uint32_t)(team * kNc + 64 * half);
      uint32_t n = 0, dph = 0, it = 0;
      for (int t = cid; t < p.n_tiles; t += ncl, ++it) {
        const int64_t row0 = (int64_t)t * kTM + 32 * sp;
        for (int c = crank; c < p.n_chunks; c += cs, ++n) {
          if ((int)(n & 1u) != team) continue;
          mbar_wait(&d_full[team], dph);
          dph ^= 1;
          if (warp == 3 + kPW && c == crank) rtrace(p, 5 + 5 * (int)min(it, 9u));
          tc_fence_after();
          const int col0 = c * kNc + 64 * half;
          if (lane == 0) bulk_wait_group_read<0>();  // the staging box's previous store has read it
          __syncwarp();
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tbase + lane_t + dcol + (uint32_t)(32 * h2), v);
            tmem_ld_wait();
            if (h2 == 1) {  // both halves read: the D buffer may be overwritten
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&d_empty[team]);
            }
            const int colh = col0 + 32 * h2;
            if (colh >= p.r_dim) continue;
            float o[32];
            if (p.bias && p.bslot < 0) {
              constexpr float bsc = (YDT == DT_BF16 && ACT == DT_ACT_SIGMOID) ? 0.5f : 1.f;
              const float bl = colh + lane < p.r_dim ? bsc * __ldg(p.bias + colh + lane) : 0.f;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]) + __shfl_sync(0xffffffffu, bl, i), p.arg);
            } else {  // bias folded into the tf32 contraction (or absent)
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]), p.arg);
            }
            // this lane's row: 16-byte chunk ch of the 128-byte row at ch ^ (row & 7) (TMA SW128)
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              const float *f = o + ch * 8;
              st_shared_v4(rb + ((uint32_t)((4 * h2 + ch) ^ (lane & 7)) << 4), pack_bf16(f[0], f[1]),
                           pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
            }
          }
          if (col0 >= p.r_dim) continue;
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_y, smem + (out_s - s0), col0, (int32_t)row0);
            bulk_commit_group();
          }
        }
        if (warp == 3 + kPW) rtrace(p, 6 + 5 * (int)min(it, 9u));
      }
      if (lane == 0) bulk_wait_group<0>();  // staging read + y written before exit
      if (warp == 3 + kPW) rtrace(p, 60);
    } else {
    // 16 warps: four per TMEM lane quarter, each owning 32 of the chunk's 128 columns
    const int sp = warp & 3;           // TMEM lane quarter this warp may access
    const int e = warp - 3 - kPW;      // 0..15
    const int qc = e / 4;              // which 32 columns of each 128-column chunk
    const uint32_t s0 = smem_u32(smem);
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    constexpr int E = YDT == DT_BF16 ? 2 : 4;
    constexpr int RB = 32 * E;         // bytes per row of this warp's 32 columns (64 or 128)
    constexpr int LPR = RB / 16;       // lanes per row when storing (4 or 8)
    constexpr int RPI = 32 / LPR;      // rows per store instruction (8 or 4)
    constexpr int SWM = RB / 16 - 1;   // swizzle mask over the row's 16-byte chunks
    const uint32_t out_s0 = s0 + p.off_out + (uint32_t)(e * p.nstage) * (32u * RB);
    int db = 0, sb = 0;
    uint32_t dph = 0, it = 0;
    for (int t = cid; t < p.n_tiles; t += ncl, ++it) {
      const int64_t row0 = (int64_t)t * kTM + 32 * sp;
      for (int c = crank; c < p.n_chunks; c += cs) {
        mbar_wait(&d_full[db], dph);
        if (warp == 3 + kPW && c == crank) rtrace(p, 5 + 5 * (int)min(it, 9u));
        tc_fence_after();
        const int col0 = c * kNc + 32 * qc;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_t + p.dcol0 + (uint32_t)(db * kNc + 32 * qc), v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[db]);
        if (++db == p.nd) { db = 0; dph ^= 1; }
        if (col0 >= p.r_dim) continue;
        float o[32];
        if (p.bias && p.bslot < 0) {
          constexpr float bsc = (YDT == DT_BF16 && ACT == DT_ACT_SIGMOID) ? 0.5f : 1.f;
          const float bl = col0 + lane < p.r_dim ? bsc * __ldg(p.bias + col0 + lane) : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]) + __shfl_sync(0xffffffffu, bl, i), p.arg);
        } else {  // bias folded into the tf32 contraction (or absent)
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]), p.arg);
        }
        // this lane's row (RB bytes) into the warp's swizzled staging box (the TMA SW64 / SW128
        // pattern: 16-byte chunk ch of row r at ch ^ (r >> 1 & 3) / ch ^ (r & 7)), then either one
        // TMA store of the 32 x 32 box or, read back RPI rows per instruction, st.global.v4
        const uint32_t out_s = out_s0 + (uint32_t)sb * (32u * RB);
        if (p.nstage == 2) sb ^= 1;
        if (p.tma_y) {  // the staging box's previous TMA store has read it
          if (lane == 0) {
            if (p.nstage == 2) bulk_wait_group_read<1>(); else bulk_wait_group_read<0>();
          }
          __syncwarp();
        }
        const uint32_t rb = out_s + (uint32_t)lane * RB;
#pragma unroll
        for (int ch = 0; ch < RB / 16; ++ch) {
          uint32_t w0, w1, w2, w3;
          if constexpr (E == 2) {
            const float *f = o + ch * 8;
            w0 = pack_bf16(f[0], f[1]); w1 = pack_bf16(f[2], f[3]);
            w2 = pack_bf16(f[4], f[5]); w3 = pack_bf16(f[6], f[7]);
          } else {
            const float *f = o + ch * 4;
            w0 = __float_as_uint(f[0]); w1 = __float_as_uint(f[1]);
            w2 = __float_as_uint(f[2]); w3 = __float_as_uint(f[3]);
          }
          const int sw = E == 2 ? ((lane >> 1) & SWM) : (lane & SWM);
          st_shared_v4(rb + ((uint32_t)(ch ^ sw) << 4), w0, w1, w2, w3);
        }
        if (p.tma_y) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_y, smem + (out_s - s0), col0, (int32_t)row0);
            bulk_commit_group();
          }
          continue;
        }
        __syncwarp();
        const int ch = lane % LPR;
        const int cb = col0 + ch * (16 / E);  // first column of this lane's 16 bytes
        uint32_t w[RPI == 8 ? 4 : 8][4];
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int r = RPI * i + lane / LPR;
          const int sw = E == 2 ? ((r >> 1) & SWM) : (r & SWM);
          ld_shared_v4(out_s + (uint32_t)r * RB + ((uint32_t)(ch ^ sw) << 4), w[i][0], w[i][1],
                       w[i][2], w[i][3]);
        }
#pragma unroll
        for (int i = 0; i < 32 / RPI; ++i) {
          const int r = RPI * i + lane / LPR;
          if (row0 + r < p.batch && cb < p.r_dim)
            st_global_v4(reinterpret_cast<uint8_t *>(p.y) + ((row0 + r) * p.r_dim + cb) * E, w[i][0],
                         w[i][1], w[i][2], w[i][3]);
        }
        __syncwarp();
      }
      if (p.post_flags) {  // this warp's stores of tile t are done: release them to the next layer
        __syncwarp();
        if (lane == 0) {
          if (p.tma_y) {
            bulk_wait_group<0>();
            fence_proxy_async_global();
          }
          __threadfence();
          red_release_add(p.post_flags + t, 1u);
        }
      }
      if (warp == 3 + kPW) rtrace(p, 6 + 5 * (int)min(it, 9u));
    }
    if (p.tma_y && lane == 0) bulk_wait_group<0>();  // staging read + y written before exit
    if (warp == 3 + kPW) rtrace(p, 60);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (cs > 1) cluster_sync();  // no CTA leaves while peers may still copy into / arrive on it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

using RowsFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, RowsParams);

template <int YDT>
RowsFn pick_act(int act) {
  switch (act) {
    case DT_ACT_RELU: return k_tc_rows_reuse<YDT, DT_ACT_RELU>;
    case DT_ACT_SIGMOID: return k_tc_rows_reuse<YDT, DT_ACT_SIGMOID>;
    case DT_ACT_TANH: return k_tc_rows_reuse<YDT, DT_ACT_TANH>;
    case DT_ACT_CLIPPED_RELU: return k_tc_rows_reuse<YDT, DT_ACT_CLIPPED_RELU>;
    default: return k_tc_rows_reuse<YDT, DT_ACT_IDENTITY>;
  }
}

int g_nsm() {
  static int nsm = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return nsm;
}

}  // namespace

// wf enters phase A as a bf16 hi + lo pair (rows [0, rank) = bf16(wf), rows [rank, 2 rank) =
// bf16(wf - hi)): the P columns of the two halves are added in fp32 before phase B, so P carries
// ~16 significant bits of wf instead of 8 — the bf16 rounding of fp32 factors (~2^-9 relative
// per product, 1.7-2.1e-3 rel_error at config 3) drops to the tf32 level. The extra N columns
// are free while 2 * rank <= 16 (the UMMA N floor). np = 2 * rank padded to 16.
static inline int64_t rows_np(const Geo &g) { return (2 * g.rank + 15) / 16 * 16; }
static inline int64_t rows_wf_bytes(const Geo &g) { return (2 * g.rank * g.n * 2 + 255) / 256 * 256; }

// Cluster size: CTAs sharing one row tile (segments and output chunks split among them).
// Default 4: clusters of 4 fill all 148 SMs (37 clusters; clusters of 8 fit only 15 times =
// 120 SMs), measured 298 vs 316 us per config-3 forward.
static int rows_cluster(const Geo &g) {
  static const int want = getenv("DEEPTHIN_ROWS_CS") ? atoi(getenv("DEEPTHIN_ROWS_CS")) : 4;
  for (int cs : {8, 4, 2})
    if (cs <= want && g.s % cs == 0) return cs;
  return 1;
}

// Geometries the row-tile kernel takes: reuse (n | q), 64-aligned segments, the padded rank's
// wf block resident (<= 32 KB), s * round_up(rank, 4) <= 32 (one 128-byte tf32 K atom),
// TMA-legal output pitch.
bool tc_rows_ok(const Geo &g, int x_dtype, int y_dtype) {
  static const int want = getenv("DEEPTHIN_ROWS") ? atoi(getenv("DEEPTHIN_ROWS")) : 1;
  if (!want || !g.reuse || g.n % 64 != 0 || x_dtype != DT_BF16) return false;
  const int64_t np = rows_np(g);
  const int64_t rp = (g.rank + 3) / 4 * 4;
  if (np > 32) return false;  // the P exchange reads all np columns of a segment in one x32 load
  if (g.s * rp > 32 || (g.s / rows_cluster(g)) * np > 128) return false;
  if ((g.n / 64) * np * 128 > 32 * 1024) return false;
  const int E = y_dtype == DT_BF16 ? 2 : 4;
  if ((g.r_dim * E) % 16 != 0) return false;
  return true;
}

static int64_t rows_k2(const Geo &g) { return (g.s * ((g.rank + 3) / 4 * 4) + 7) / 8 * 8; }

size_t tc_rows_ws(const Geo &g) {
  if (!g.reuse) return 0;
  return (size_t)rows_wf_bytes(g) + (size_t)((g.r_dim * rows_k2(g) * 4 + 255) / 256 * 256);
}

namespace {
// Per-call operand prep (the analogue of the reference's per-pair derived copies,
// kernel.py:157-164): wf -> bf16, and XF2 re-laid with each segment's rank values padded to rp
// (zeros), K padded to k2: XF2p[j, seg*rp + k] = xf[j*s + seg, k].
__global__ void k_rows_prep(int64_t wf_count, const float *wf, __nv_bfloat16 *wf16, int r_dim, int s,
                            int rank, int rp, int k2, const float *xf, float *xf2p, const float *bias,
                            int bslot, float scale) {
  griddep_wait();
  griddep_launch_dependents();
  const int64_t tot = wf_count + (int64_t)r_dim * k2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < wf_count) {  // hi (rows 0..rank-1) and lo (rows rank..2 rank-1) parts of wf
      const float v = wf[i];
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      wf16[i] = hi;
      wf16[wf_count + i] = __float2bfloat16_rn(v - __bfloat162float(hi));
    } else {
      const int64_t e = i - wf_count;
      const int64_t j = e / k2;
      const int kk = (int)(e - j * k2), seg = kk / rp, k = kk - seg * rp;
      float v = (seg < s && k < rank) ? xf[(j * s + seg) * rank + k] : 0.f;
      if (kk == bslot) v = bias ? bias[j] : 0.f;
      xf2p[e] = v * scale;
    }
  }
}
}  // namespace

int tc_rows_prepare(const Geo &g, const float *wf, const float *xf, const float *bias, int act,
                    int y_dtype, char *ws, cudaStream_t st) {
  const int rp = (int)((g.rank + 3) / 4 * 4), k2 = (int)rows_k2(g);
  const int bslot = !bias ? -1 : (g.rank < rp ? (int)g.rank : (k2 > g.s * rp ? (int)(g.s * rp) : -1));
  const float scale = (y_dtype == DT_BF16 && act == DT_ACT_SIGMOID) ? 0.5f : 1.f;
  __nv_bfloat16 *wf16 = reinterpret_cast<__nv_bfloat16 *>(ws);
  float *xf2p = reinterpret_cast<float *>(ws + rows_wf_bytes(g));
  const int64_t tot = g.rank * g.n + g.r_dim * (int64_t)k2;
  cudaLaunchConfig_t pc{};
  pc.gridDim = dim3((unsigned)std::min<int64_t>((tot + 255) / 256, 4 * g_nsm()));
  pc.blockDim = dim3(256);
  pc.stream = st;
  cudaLaunchAttribute pa[1];
  pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pa[0].val.programmaticStreamSerializationAllowed = 1;
  pc.attrs = pa;
  pc.numAttrs = 1;
  DT_CUDA_CHECK(cudaLaunchKernelEx(&pc, k_rows_prep, (int64_t)(g.rank * g.n), wf, wf16, (int)g.r_dim,
                                   (int)g.s, (int)g.rank, rp, k2, xf, xf2p, bias, bslot, scale));
  return check_launch("rows_prep");
}

namespace {
thread_local const unsigned *g_chain_wait = nullptr;
thread_local unsigned g_chain_target = 0;
thread_local unsigned *g_chain_post = nullptr;
}  // namespace

void rows_chain(const unsigned *wait, unsigned target, unsigned *post) {
  g_chain_wait = wait;
  g_chain_target = target;
  g_chain_post = post;
}
int rows_posts_per_tile(const Geo &g) { return rows_cluster(g) * kEpi; }

int tc_rows_forward(const Geo &g, int64_t batch, const void *x, const float *wf, const float *xf,
                    const float *bias, int act, float act_arg, void *y, int y_dtype, char *ws,
                    cudaStream_t st, bool prepared) {
  if (batch == 0) return DT_OK;
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15) ||
      (reinterpret_cast<uintptr_t>(ws) & 255)) {
    set_error("row-tile kernel: operands must be 16-byte aligned");
    return DT_E_ARG;
  }
  RowsParams p{};
  p.batch = batch;
  p.r_dim = (int)g.r_dim;
  p.n_tiles = (int)((batch + kTM - 1) / kTM);
  p.s = (int)g.s;
  p.nkb = (int)(g.n / 64);
  p.np = (int)rows_np(g);
  p.rank = (int)g.rank;
  p.rp = (int)((g.rank + 3) / 4 * 4);
  p.k2 = (int)rows_k2(g);
  p.n_chunks = (int)((g.r_dim + kNc - 1) / kNc);
  p.cs = rows_cluster(g);
  p.bias = bias;
  p.y = y;
  p.arg = act_arg;
  // one-shot chain request (dt_rows_chain), honoured only with prepared operands (a per-call
  // prep kernel would itself be the dependency)
  if (prepared) {
    p.wait_flags = g_chain_wait;
    p.wait_target = g_chain_target;
    p.post_flags = g_chain_post;
  }
  g_chain_wait = nullptr;
  g_chain_post = nullptr;
  // a zero K slot for the bias: the rank padding of segment 0, else an all-zero pad chunk
  p.bslot = !bias ? -1 : (g.rank < p.rp ? (int)g.rank : (p.k2 > g.s * p.rp ? (int)(g.s * p.rp) : -1));
  p.pcols = (int)((g.s / p.cs) * p.np);
  // row softmax fused into the epilogue (two passes, the contraction recomputed: see the
  // kernel) when the bias rides in the contraction; DEEPTHIN_ROWS_SOFTMAX=0: logits, then the
  // separate register softmax kernel (A/B runs)
  const bool want_sm = act == DT_ACT_SOFTMAX;
  const char *fenv = getenv("DEEPTHIN_ROWS_SOFTMAX");  // read per call (tests flip it)
  const int fuse_sm = fenv ? atoi(fenv) : 1;
  p.softmax = (want_sm && fuse_sm && (!bias || p.bslot >= 0)) ? 1 : 0;
  if (want_sm) act = DT_ACT_IDENTITY;
  // bf16 sigmoid runs as 1/2 + tanh(z/2)/2: the contraction (and bias) pre-scaled by 1/2
  const float scale = (y_dtype == DT_BF16 && act == DT_ACT_SIGMOID) ? 0.5f : 1.f;
  // shared memory: A2 x 2 | wf | XF2 ring | output staging | x ring (what is left) | barriers
  const uint32_t wf_bytes = (uint32_t)(p.nkb * p.np * 128);
  p.off_a2 = 0;
  p.off_wf = 2 * kA2Bytes;
  p.off_b = (p.off_wf + wf_bytes + 1023) & ~1023u;
  p.off_out = p.off_b + kBS * kBBytes;
  // TMEM: P double buffer in columns [0, 2 pcols), nd D buffers of 128 columns at the top;
  // output staging: nstage boxes per epilogue warp (DEEPTHIN_ROWS_ND / _STG: A/B runs)
  static const int want_nd = getenv("DEEPTHIN_ROWS_ND") ? atoi(getenv("DEEPTHIN_ROWS_ND")) : 2;
  static const int want_stg = getenv("DEEPTHIN_ROWS_STG") ? atoi(getenv("DEEPTHIN_ROWS_STG")) : 1;
  p.nd = std::max(2, std::min(want_nd, (int)(512 - (2 * p.pcols + 127) / 128 * 128) / (int)kNc));
  p.dcol0 = 512u - (uint32_t)p.nd * kNc;
  p.nstage = (want_stg == 2 && !p.softmax) ? 2 : 1;
  // wide bf16 epilogue (see the kernel), opt-in with DEEPTHIN_ROWS_WIDE=1: measured 28.96 vs
  // 28.50 us per config-3 hidden layer — halving the TMA store requests does not pay, the x
  // ring it shrinks (7 -> 5 stages) costs as much
  static const int want_wide = getenv("DEEPTHIN_ROWS_WIDE") ? atoi(getenv("DEEPTHIN_ROWS_WIDE")) : 0;
  static const int want_tma_y0 = getenv("DEEPTHIN_ROWS_TMA_Y") ? atoi(getenv("DEEPTHIN_ROWS_TMA_Y")) : 1;
  p.wide = (want_wide && want_tma_y0 && y_dtype == DT_BF16 && !p.softmax && p.nd == 2 &&
            !p.wait_flags && !p.post_flags && (g.r_dim * 2) % 16 == 0) ? 1 : 0;
  if (p.wide) p.nstage = 1;
  p.off_x = p.off_out + (p.wide ? (uint32_t)kEpi * 4096u
                                : (uint32_t)p.nstage * kEpi * 32u * 32u * (uint32_t)(y_dtype == DT_BF16 ? 2 : 4));
  if (p.softmax) {  // [4][128] column-warp partials, then 2 x cs x 128 cluster partials
    p.off_red = p.off_x;
    p.off_x += 4 * kTM * 8;
    p.off_sm = p.off_x;
    p.off_x += 2u * (uint32_t)p.cs * kTM * 8;
    p.off_x = (p.off_x + 1023) & ~1023u;
  }
  constexpr uint32_t kSmemMax = 227 * 1024, kTail = 512 + 1024;
  static const int want_xs = getenv("DEEPTHIN_ROWS_XS") ? atoi(getenv("DEEPTHIN_ROWS_XS")) : kXSMax;
  p.xs = (int)std::min<uint32_t>((uint32_t)std::max(2, std::min(want_xs, kXSMax)),
                                 (kSmemMax - kTail - p.off_x) / kXBytes);
  p.off_bar = p.off_x + (uint32_t)p.xs * kXBytes;
  const uint32_t smem_bytes = p.off_bar + kTail;

  __nv_bfloat16 *wf16 = reinterpret_cast<__nv_bfloat16 *>(ws);
  float *xf2p = reinterpret_cast<float *>(ws + rows_wf_bytes(g));
  // operands derived once per factor pair (dt_rows_prepare) or here, per call
  if (!prepared)
    if (int rc = tc_rows_prepare(g, wf, xf, bias, act, y_dtype, ws, st)) return rc;

  // The slab kernel (k_tc_slab.cu: no clusters, every SM a contiguous slab of rows) takes the
  // layer when s is a power of two and no per-tile chaining was requested
  // (DEEPTHIN_ROWS_SLAB=0: the clustered row-tile kernel below, A/B runs and tests)
  {
    const char *senv = getenv("DEEPTHIN_ROWS_SLAB");  // read per call (tests flip it)
    if ((senv ? atoi(senv) != 0 : false) && !p.wait_flags && !p.post_flags && tc_slab_ok(g, batch, p.softmax)) {
      if (int rc = tc_slab_forward(g, batch, x, wf16, xf2p, bias, p.bslot, act, act_arg, y, y_dtype, st))
        return rc;
      return want_sm && !p.softmax ? launch_row_softmax(batch, g.r_dim, y, y_dtype, st) : DT_OK;
    }
  }

  CUtensorMap tm_x, tm_wf, tm_xf2;
  if (int rc = encode_tensor_map_2d(&tm_x, DT_BF16, const_cast<void *>(x), (uint64_t)g.q,
                                    (uint64_t)batch, (uint64_t)g.q * 2, 64, kTM, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_wf, DT_BF16, wf16, (uint64_t)g.n, (uint64_t)(2 * g.rank),
                                    (uint64_t)g.n * 2, 64, (uint32_t)p.np, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_xf2, DT_F32, xf2p, (uint64_t)p.k2, (uint64_t)g.r_dim,
                                    (uint64_t)p.k2 * 4, 32, kNc, true))
    return rc;
  // TMA stores of the epilogue's 32 x 32 boxes (DEEPTHIN_ROWS_TMA_Y=0: st.global.v4, A/B runs)
  static const int want_tma_y = getenv("DEEPTHIN_ROWS_TMA_Y") ? atoi(getenv("DEEPTHIN_ROWS_TMA_Y")) : 1;
  CUtensorMap tm_y;
  memset(&tm_y, 0, sizeof(tm_y));
  p.tma_y = (want_tma_y || p.softmax) ? 1 : 0;  // the softmax epilogue stores through TMA
  if (p.tma_y)
    if (int rc = encode_tensor_map_2d_sw(&tm_y, y_dtype, y, (uint64_t)g.r_dim, (uint64_t)batch,
                                         (uint64_t)g.r_dim * (y_dtype == DT_BF16 ? 2 : 4),
                                         p.wide ? 64 : 32, 32,
                                         y_dtype == DT_BF16 && !p.wide ? (int)CU_TENSOR_MAP_SWIZZLE_64B
                                                                       : (int)CU_TENSOR_MAP_SWIZZLE_128B))
      return rc;
  RowsFn fn = y_dtype == DT_BF16 ? pick_act<DT_BF16>(act) : pick_act<DT_F32>(act);
  // the opt-in shared-memory size once per (device, kernel instance)
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kRowsThreads);
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
  // persistent: as many clusters as fit at once (each loops over row tiles)
  // (occupancy per (device, kernel instance, cluster size), queried once)
  static std::mutex occ_mu;
  static std::map<std::tuple<int, const void *, int>, int> occ;
  int max_cl = 0;
  {
    int dev = 0;
    DT_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(occ_mu);
    int &slot = occ[std::make_tuple(dev, reinterpret_cast<const void *>(fn), p.cs)];
    if (!slot) {
      cfg.gridDim = dim3((unsigned)(p.cs * 64));
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        n = g_nsm() / p.cs;
      }
      slot = n;
    }
    max_cl = slot;
  }
  const int ncl = std::max(1, std::min(p.n_tiles, max_cl));
  cfg.gridDim = dim3((unsigned)(ncl * p.cs));
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_ROWS_TRACE") != 0;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&p.trace, (size_t)ncl * p.cs * kTr * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, (size_t)ncl * p.cs * kTr * 8, st));
  }
  cudaEvent_t ev_b = nullptr, ev_a = nullptr;  // dt_profile_kernel_events
  profile_next(&ev_b, &ev_a, DT_PROF_ROWS);
  if (ev_b) DT_CUDA_CHECK(cudaEventRecord(ev_b, st));
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm_x, tm_wf, tm_xf2, tm_y, p));
  if (ev_a) DT_CUDA_CHECK(cudaEventRecord(ev_a, st));
  if (tracing) {  // every CTA's stamps, raw, to DEEPTHIN_ROWS_TRACE_FILE (scripts/rows_trace.py)
    const int nb = ncl * p.cs;
    std::vector<unsigned long long> h((size_t)nb * kTr);
    DT_CUDA_CHECK(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFree(p.trace);
    const char *fn = getenv("DEEPTHIN_ROWS_TRACE_FILE");
    if (FILE *f = fopen(fn ? fn : "rows_trace.bin", "wb")) {
      const int hdr[6] = {nb, kTr, p.cs, p.n_tiles, p.n_chunks, p.s};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (int rc = check_launch("tc_rows_reuse")) return rc;
  return want_sm && !p.softmax ? launch_row_softmax(batch, g.r_dim, y, y_dtype, st) : DT_OK;
}

}  // namespace dt
