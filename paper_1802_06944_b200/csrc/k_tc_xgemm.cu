// Any-major tcgen05 GEMM on CTA pairs — the contractions of the tensor-core training step and of
// the general-geometry backward (grad.py:63-95, train.py:86-117), which the reference runs as
// numpy matmuls over transposed views:
//
//   D[M x N] = sum_k A(m, k) * B(n, k)          (fp32 accumulate in TMEM)
//
// A is stored K-major (A[m * lda + k]) or MN-major (A[k * lda + m]); B likewise. Both major
// orders feed tcgen05 directly (instruction-descriptor bits 15/16): a transposed view costs
// nothing — no transpose kernel and no copy. Operands: tf32 (fp32 in memory, kind::tf32) or
// bf16 (kind::f16), TMA-staged with 128-byte swizzle.
//
// Tile: a cluster of two CTAs computes 256 rows (128 per CTA: TMEM lanes) x BN columns
// (BN in {64, 128, 256}; each CTA stages half of the B tile, cta_group::2 MMA M = 256). The leader
// CTA's single thread issues every MMA; commits multicast to both CTAs. Accumulators are
// double-buffered in TMEM (2 x BN columns) so the epilogue of unit u overlaps the MMAs of u + 1.
// Work units are (row block, column block, K split), persistent over the clusters. Split-K
// writes fixed-size partial slices that k_xg_reduce sums in split order: results never depend
// on timing or on the number of SMs (no float atomics).
//
// Epilogues (one per template instance):
//   XE_STORE   out = alpha * D (+ bias[n]), fp32, TMA-stored (split-K: the partial slice)
//   XE_MSE     g = scale * (D + bias[n] - target), TMA-stored; per-warp fp64 loss partials of
//              sum (D + bias - target)^2 and fixed-order per-CTA column sums of g (d_bias)
//              (grad.py:98-103 and :85 fused into the forward's last contraction)
//   XE_PAIRSUM out[m, k] = D[m, k] + D[m, k + BN/2]: the hi + lo halves of a bf16-split operand
//   XE_SPLITH  H (fp32, B x s*r) -> H2 (B*s x 2r bf16, [hi | lo] per row of the re-laid view)
//
// Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (leader CTA), warps 2-9 epilogue
// (TMEM lane quarter = warp % 4, column half = (warp - 2) / 4).

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <type_traits>

#include "act.cuh"
#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

constexpr int XEPI = 8;                       // epilogue warps
constexpr int XTHREADS = 64 + 32 * XEPI;
constexpr uint32_t XA_BYTES = 128 * 128;      // A half-tile stage: 128 rows x 128 B (16 KB)
constexpr uint32_t XSTG = 32 * 128;           // one 32 x 32 fp32 staging box (4 KB)
constexpr int XSMEM_MAX = 227 * 1024;

enum { XE_STORE = 0, XE_MSE = 1, XE_PAIRSUM = 2, XE_SPLITH = 3, XE_STORE_T = 4 };

struct XgParams {
  int M, N, BN, nhalf;        // nhalf = BN / 2 columns staged per CTA
  int n_mb, n_nb, splits, units, kb_total, kb_per;
  int a_mn, b_mn;             // 1: MN-major operand
  int b_wrap;                 // > 0: B's k-block index wraps modulo b_wrap (K-stacked hi/lo A)
  int S;
  uint32_t off_b, stage_bytes, off_stg, off_bar;
  int Mp;                     // rows per split slice of the partial buffer (multiple of 256)
  // epilogue
  float alpha;
  const float *bias;
  int ldo;
  float scale;
  double *loss_part;
  float *colsum_part;         // [2 * n_mb][N]
  __nv_bfloat16 *out16;       // XE_SPLITH
  int h_r, h_s;
  int pair_half;              // XE_PAIRSUM: out[:, k] = D[:, k] + D[:, k + pair_half]
  int ks_major;               // unit order: K split slowest (tiles of one split run together)
  int chain;                  // pipelined forward: let the next call's W regeneration start early
  float act_arg;              // XE_STORE_T activation argument
  void *out_t;                // XE_STORE_T: out[n][m] (pitch ldo), fp32 or bf16
  int N_true;                 // XE_STORE_T: rows of out (D columns) actually stored
  int tma_t;                  // XE_STORE_T, fp32 out: transposed through shared staging + TMA stores
  int dbg;                    // timing build only (DEEPTHIN_DBG_XG): 1 no y stores, 2 no MMAs, 4 no TMEM reads, 8 no dual-A loads
  int dual_kb;                // > 0: each stage also carries A at k-block kb + dual_kb (a second
                              // A half, e.g. W_lo beside W_hi) multiplied by the same B tile
};

// K-major: rows of 128 B (the k-block), 8-row swizzle atoms 1024 B apart (SWIZZLE_128B).
// MN-major: 128-byte chunks along M/N, each BKE K-rows x 128 B, chunk stride LBO = BKE * 128.
//   bf16: SWIZZLE_128B, 8-row atoms (SBO 1024); tf32: tcgen05 takes MN-major tf32 only in the
//   128B_BASE32B layout (32-byte swizzle atoms, 4-row groups: SBO 512), which TMA writes with
//   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t xdesc(uint32_t base, int mn, int k, int el) {
  if (!mn) return smem_desc(base + (uint32_t)k * 32u, 16, 1024, SL_SW128);
  const uint32_t bke = el ? 32u : 64u;
  const uint32_t step = el ? 1024u : 2048u;  // one MMA's K rows (8 tf32 / 16 bf16) x 128 B
  if (el) return smem_desc(base + (uint32_t)k * step, bke * 128u, 512, 1u /* 128B_BASE32B */);
  return smem_desc(base + (uint32_t)k * step, bke * 128u, 1024, SL_SW128);
}

// Stage one operand half-tile (rows = 128 for A, nhalf for B) of k-block kb. mn == 2: an
// MN-major operand through a 3-D map (one box covers every 128-byte chunk of the half-tile).
__device__ __forceinline__ void xload(uint8_t *dst, const CUtensorMap *tm, uint64_t *bar, int mn,
                                      int el, int row0, int rows, int kb) {
  const int bke = el ? 32 : 64;
  if (!mn) {
    tma_load_2d_pair(dst, tm, bar, kb * bke, row0);
  } else if (mn == 2) {
    const int ce = 128 / (el ? 4 : 2);
    tma_load_3d_pair(dst, tm, bar, 0, kb * bke, row0 / ce);
  } else {
    const int ce = 128 / (el ? 4 : 2);  // elements per 128-byte chunk along M/N
    for (int c = 0; c * ce < rows; ++c)
      tma_load_2d_pair(dst + c * (uint32_t)bke * 128u, tm, bar, row0 + c * ce, kb * bke);
  }
}

__device__ __forceinline__ uint32_t stg_off(int r, int c16) {  // SW128 32 x 128 B box
  return (uint32_t)r * 128u + ((uint32_t)(c16 ^ (r & 7)) << 4);
}

// the epilogue's "TMEM read" signal: relaxed (see mbar_arrive_relaxed)
__device__ __forceinline__ void arrive_leader_x(uint64_t *bar, uint32_t crank) {
  if (crank == 0)
    mbar_arrive_relaxed(bar);
  else
    mbar_arrive_remote_relaxed(bar, 0);
}

template <int EL, int EPI, int YDT = DT_F32, int ACT = DT_ACT_IDENTITY>
__global__ void __launch_bounds__(XTHREADS, 1)
    k_tc_xgemm(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
               const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ CUtensorMap tm_t,
               const XgParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *tload = tempty + 2;  // [XEPI][3] target boxes (XE_MSE)
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tload + 3 * XEPI);
  float *red = reinterpret_cast<float *>(smem + p.off_bar + 512);  // XE_MSE [2][4][256] colsums
  // (the shuffles make the warp index, the cluster rank and the TMEM base provably warp-uniform
  // for the compiler: the producer and issuer loops run on all 32 lanes with only the
  // asynchronous instructions predicated on lane 0, so their operands stay in uniform registers
  // instead of a per-instruction ELECT / R2UR waterfall — ~200 -> ~40 clocks per MMA issue,
  // measured on the row kernels; the issue rate, not the tensor pipe, paced these GEMMs)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const bool l0 = lane == 0;
  const uint32_t crank = blockIdx.x & 1u;  // rank in the cluster of 2 along x (uniform to the compiler)
  const bool leader = crank == 0;
  const int cid = (int)blockIdx.x / 2, ncl = (int)gridDim.x / 2;
  const int BN = p.BN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * XEPI); }
    for (int i = 0; i < 3 * XEPI; ++i) mbar_init(&tload[i], 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_a);
    tma_prefetch_desc(&tm_b);
    tma_prefetch_desc(&tm_o);
    if (EPI == XE_MSE) tma_prefetch_desc(&tm_t);
  }
  if (warp == 1) tmem_alloc_pair(tslot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tslot, 0);
  griddep_wait();  // operands may come from the previous kernel on the stream
  if (p.chain) griddep_launch_dependents();  // the next forward's W regeneration may start

  auto unit_of = [&](int u, int &mb, int &nb, int &ks) {
    int t;
    if (p.ks_major) {
      const int tiles = p.n_mb * p.n_nb;
      ks = u / tiles;
      t = u - ks * tiles;
    } else {
      ks = u % p.splits;
      t = u / p.splits;
    }
    nb = t % p.n_nb;
    mb = t / p.n_nb;
    // (integer division runs on the vector pipe: pass the results through a shuffle so the
    // compiler keeps treating everything derived from them as warp-uniform)
    mb = __shfl_sync(0xffffffffu, mb, 0);
    nb = __shfl_sync(0xffffffffu, nb, 0);
    ks = __shfl_sync(0xffffffffu, ks, 0);
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own A rows, own half of the B columns) -------
    {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t abytes = p.dual_kb > 0 ? 2u * XA_BYTES : XA_BYTES;
      const bool skip_dual = kTimingSwitches && (p.dbg & 8);  // traffic experiment: no A_lo loads
      const uint32_t bytes = 2u * ((skip_dual ? XA_BYTES : abytes) + (uint32_t)p.nhalf * 128u);
      for (int u = cid; u < p.units; u += ncl) {
        int mb, nb, ks;
        unit_of(u, mb, nb, ks);
        const int kb0 = ks * p.kb_per, kb1 = min(p.kb_total, kb0 + p.kb_per);
        const int m0 = mb * 256 + (int)crank * 128, n0 = nb * BN + (int)crank * p.nhalf;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *st = smem + stage * p.stage_bytes;
          const int kbb = p.b_wrap > 0 ? kb % p.b_wrap : kb;
          if (l0) {
            if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
            xload(st, &tm_a, &full[stage], p.a_mn, EL, m0, 128, kb);
            if (p.dual_kb > 0 && !skip_dual) xload(st + abytes - XA_BYTES, &tm_a, &full[stage], p.a_mn, EL, m0, 128,
                                     kb + p.dual_kb);
            xload(st + abytes, &tm_b, &full[stage], p.b_mn, EL, n0, p.nhalf, kbb);
          }
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader) {
      const uint32_t idesc = idesc_f32acc(256, (uint32_t)BN, EL ? 2 : 1) |
                             ((uint32_t)(p.a_mn != 0) << 15) | ((uint32_t)(p.b_mn != 0) << 16);
      const uint32_t s0 = smem_u32(smem);
      // descriptors: stage 0 / K step 0 once, then plain 64-bit additions in the start-address
      // field (16-byte units; no carry out of its 14 bits within shared memory)
      const uint32_t b_off = p.dual_kb > 0 ? 2u * XA_BYTES : XA_BYTES;
      const uint64_t dA0 = xdesc(s0, p.a_mn, 0, EL), dB0 = xdesc(s0 + b_off, p.b_mn, 0, EL);
      const uint32_t ksA = p.a_mn ? (EL ? 1024u : 2048u) >> 4 : 2u;
      const uint32_t ksB = p.b_mn ? (EL ? 1024u : 2048u) >> 4 : 2u;
      const uint32_t st16 = p.stage_bytes >> 4;
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (int u = cid; u < p.units; u += ncl) {
        int mb, nb, ks;
        unit_of(u, mb, nb, ks);
        const int kb0 = ks * p.kb_per, kb1 = min(p.kb_total, kb0 + p.kb_per);
        mbar_wait(&tempty[acc], aphase ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = dA0 + (uint64_t)((uint32_t)stage * st16);
          const uint64_t db = dB0 + (uint64_t)((uint32_t)stage * st16);
          const uint64_t da2 = da + (uint64_t)(XA_BYTES >> 4);
          const uint32_t acc0 = kb > kb0 ? 1u : 0u;
          if (l0 && !(kTimingSwitches && (p.dbg & 2))) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if constexpr (EL)
                mma_tf32_ss_pair(d, da + (uint64_t)(k * ksA), db + (uint64_t)(k * ksB), idesc, k > 0 ? 1u : acc0);
              else
                mma_bf16_ss_pair(d, da + (uint64_t)(k * ksA), db + (uint64_t)(k * ksB), idesc, k > 0 ? 1u : acc0);
            }
            if (p.dual_kb > 0) {  // the second A half against the same B stage
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if constexpr (EL) mma_tf32_ss_pair(d, da2 + (uint64_t)(k * ksA), db + (uint64_t)(k * ksB), idesc, 1u);
                else mma_bf16_ss_pair(d, da2 + (uint64_t)(k * ksA), db + (uint64_t)(k * ksB), idesc, 1u);
              }
            }
          }
          if (l0) mma_commit_pair(&empty[stage]);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        if (l0) mma_commit_pair(&tfull[acc]);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (both CTAs: 128 rows x BN columns each) ----------------
    const int e = warp - 2, q = warp & 3, h = e / 4;
    const uint32_t lane_t = (uint32_t)(32 * q) << 16;
    constexpr int NBUF = EPI == XE_MSE ? 3 : EPI == XE_STORE_T ? 1 : 2;  // staging boxes per warp
    const uint32_t stg0 = smem_u32(smem) + p.off_stg + (uint32_t)e * NBUF * XSTG;
    uint8_t *stg0p = smem + p.off_stg + e * NBUF * XSTG;
    const int nch = EPI == XE_PAIRSUM ? (p.pair_half + 31) / 32 : BN / 32;
    int acc = 0, jb = 0;  // jb: this warp's running chunk count (staging buffer = jb % NBUF)
    uint32_t aphase = 0;
    uint32_t tph = 0;     // XE_MSE: parity bit per staging buffer (bit b)
    // XE_MSE target prefetch: the warp's chunk sequence (unit, chunk) walked two chunks ahead of
    // the one being processed, across unit boundaries (the target does not depend on the MMAs)
    int lu = cid, lc = h, nload = 0;
    auto load_next = [&]() {
      if (lu >= p.units) return;
      int mb, nb, ks;
      unit_of(lu, mb, nb, ks);
      const int b = nload % NBUF;
      if (lane == 0) {
        mbar_arrive_expect_tx(&tload[NBUF * e + b], XSTG);
        tma_load_2d(stg0p + b * XSTG, &tm_t, &tload[NBUF * e + b], nb * BN + 32 * lc,
                    mb * 256 + (int)crank * 128 + 32 * q);
      }
      ++nload;
      lc += 2;
      if (lc >= nch) { lc = h; lu += ncl; }
    };
    if constexpr (EPI == XE_MSE) { load_next(); load_next(); }
    int par = 0;  // XE_MSE: column-sum exchange buffer parity (by unit)
    for (int u = cid; u < p.units; u += ncl) {
      int mb, nb, ks;
      unit_of(u, mb, nb, ks);
      const int row = mb * 256 + (int)crank * 128 + 32 * q + lane;  // this thread's D row
      const int r0 = mb * 256 + (int)crank * 128 + 32 * q;           // the warp's first row
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      double sq = 0.0;
      for (int c = h; c < nch; c += 2) {
        const int col0 = nb * BN + 32 * c;  // first D column of this chunk
        uint32_t v[32];
        if (kTimingSwitches && (p.dbg & 4)) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0u;
        } else
        tmem_ld_32x32b_x32(tbase + lane_t + (uint32_t)(acc * BN + 32 * c), v);
        if constexpr (EPI == XE_PAIRSUM) {
          uint32_t w[32];
          tmem_ld_32x32b_x32(tbase + lane_t + (uint32_t)(acc * BN + 32 * c + p.pair_half), w);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(w[i]));
        } else {
          tmem_ld_wait();
        }
        if constexpr (EPI == XE_STORE_T) {
          // out[n][m] = act(D[m][n] + bias[m]): lane = output column m, the chunk's 32 D
          // columns = 32 output rows; each store instruction writes 32 consecutive columns of
          // one output row (coalesced)
          using OutT = typename std::conditional<YDT == DT_BF16, __nv_bfloat16, float>::type;
          if constexpr (YDT == DT_F32) {
            if (p.tma_t) {
              // Transposed through shared memory: the chunk is staged as two 16 x 32 fp32 half
              // boxes (batch row i = one 128-byte line, this lane's output column at word `lane`,
              // 16-byte units XOR-swizzled by i & 7 as the SW128 tensor map expects: every
              // st.shared covers 32 distinct banks), each stored by ONE bulk tensor copy instead
              // of 16 st.global instructions through L1 (TMA clips the ragged edges of y). The
              // half boxes alternate, so a half is rewritten only after the store two back read it.
              const float bm = (p.bias && row < p.M) ? __ldg(p.bias + row) : 0.f;
#pragma unroll
              for (int hb = 0; hb < 2; ++hb) {
                if (lane == 0) bulk_wait_group_read<1>();
                __syncwarp();
                const uint32_t sb = stg0 + (uint32_t)hb * 2048u;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[16 * hb + i]) + bm, p.act_arg);
                  asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + (uint32_t)i * 128u +
                                                                 ((uint32_t)((lane >> 2) ^ (i & 7)) << 4) +
                                                                 (uint32_t)(lane & 3) * 4u),
                               "f"(o)
                               : "memory");
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  if (col0 + 16 * hb < p.N_true && r0 < p.M)
                    tma_store_2d(&tm_o, stg0p + hb * 2048, r0, col0 + 16 * hb);
                  bulk_commit_group();  // (an empty group keeps the wait above counting halves)
                }
              }
              continue;
            }
          }
          if (row < p.M && !(kTimingSwitches && (p.dbg & 1) && v[0] != 0x7fc12345u)) {
            const float bm = p.bias ? __ldg(p.bias + row) : 0.f;
            OutT *yp = reinterpret_cast<OutT *>(p.out_t) + (int64_t)col0 * p.ldo + row;
            const int nrow = min(32, p.N_true - col0);
            if (nrow >= 32) {
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[i]) + bm, p.act_arg);
                if constexpr (YDT == DT_BF16) yp[(int64_t)i * p.ldo] = __float2bfloat16_rn(o);
                else yp[(int64_t)i * p.ldo] = o;
              }
            } else {
              for (int i = 0; i < nrow; ++i) {
                const float o = act_out_bf16<YDT, ACT>(__uint_as_float(v[i]) + bm, p.act_arg);
                if constexpr (YDT == DT_BF16) yp[(int64_t)i * p.ldo] = __float2bfloat16_rn(o);
                else yp[(int64_t)i * p.ldo] = o;
              }
            }
          }
          continue;
        } else if constexpr (EPI == XE_SPLITH) {
          // H[row, col0 .. col0+31] -> H2 row (row * s + col0 / r), [hi | lo]
          if (row < p.M && (p.h_r & 31)) {  // a chunk may cross a segment: element stores
#pragma unroll 4
            for (int i = 0; i < 32; ++i) {
              const int cc = col0 + i;
              if (cc >= p.N) break;
              const int seg = cc / p.h_r, k = cc - seg * p.h_r;
              const float a = __uint_as_float(v[i]);
              const __nv_bfloat16 ha = __float2bfloat16_rn(a);
              __nv_bfloat16 *hp = p.out16 + ((int64_t)row * p.h_s + seg) * (2 * p.h_r) + k;
              hp[0] = ha;
              hp[p.h_r] = __float2bfloat16_rn(a - __bfloat162float(ha));
            }
          } else if (row < p.M) {
            const int seg = col0 / p.h_r, k0 = col0 % p.h_r;
            __nv_bfloat16 *hp = p.out16 + ((int64_t)row * p.h_s + seg) * (2 * p.h_r) + k0;
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float a = __uint_as_float(v[2 * i]), b = __uint_as_float(v[2 * i + 1]);
              const __nv_bfloat16 ha = __float2bfloat16_rn(a), hb = __float2bfloat16_rn(b);
              __nv_bfloat162 hh, ll;
              hh.x = ha; hh.y = hb;
              ll = __floats2bfloat162_rn(a - __bfloat162float(ha), b - __bfloat162float(hb));
              hi[i] = *reinterpret_cast<uint32_t *>(&hh);
              lo[i] = *reinterpret_cast<uint32_t *>(&ll);
            }
            uint4 *dh = reinterpret_cast<uint4 *>(hp), *dl = reinterpret_cast<uint4 *>(hp + p.h_r);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              dh[i] = make_uint4(hi[4 * i], hi[4 * i + 1], hi[4 * i + 2], hi[4 * i + 3]);
              dl[i] = make_uint4(lo[4 * i], lo[4 * i + 1], lo[4 * i + 2], lo[4 * i + 3]);
            }
          }
          continue;
        } else {
          const int b = jb % NBUF;
          ++jb;
          const uint32_t sbase = stg0 + (uint32_t)b * XSTG;
          uint8_t *sptr = stg0p + b * XSTG;
          if constexpr (EPI == XE_MSE) {  // this chunk's target box (loaded two chunks ago)
            mbar_wait(&tload[NBUF * e + b], (tph >> b) & 1u);
            tph ^= 1u << b;
          } else {  // the box's previous TMA store has read it
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
          }
          float bias_v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) bias_v[i] = 0.f;
          if (p.bias) {
#pragma unroll
            for (int i = 0; i < 32; ++i) bias_v[i] = (col0 + i < p.N) ? __ldg(p.bias + col0 + i) : 0.f;
          }
          float csq = 0.f;
          float go[32];  // XE_MSE: this chunk's g values (column sums below)
#pragma unroll
          for (int c16 = 0; c16 < 8; ++c16) {
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = 4 * c16 + j;
              const float z = __uint_as_float(v[i]);
              if constexpr (EPI == XE_MSE) {
                const float t = reinterpret_cast<const float *>(sptr + stg_off(lane, c16))[j];
                const float dz = (z + bias_v[i]) - t;
                const bool ok = row < p.M && col0 + i < p.N;
                csq = ok ? fmaf(dz, dz, csq) : csq;
                o[j] = ok ? p.scale * dz : 0.f;
                go[i] = o[j];
              } else {
                o[j] = fmaf(p.alpha, z, bias_v[i]);
              }
            }
            sts_v4(sbase + stg_off(lane, c16), __float_as_uint(o[0]), __float_as_uint(o[1]),
                   __float_as_uint(o[2]), __float_as_uint(o[3]));
          }
          if constexpr (EPI == XE_MSE) {
            sq += (double)csq;
            // column sums of g over this warp's 32 rows: a shuffle transpose-reduce (5 halving
            // rounds, fixed order) leaves column `lane`'s sum in lane `lane`
            float cs[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) cs[i] = go[i];
#pragma unroll
            for (int w = 16; w >= 1; w >>= 1) {
              const bool upper = (lane & w) != 0;
#pragma unroll
              for (int i = 0; i < w; ++i) {
                const float send = upper ? cs[i] : cs[i + w];
                const float keep = upper ? cs[i + w] : cs[i];
                cs[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
              }
            }
            red[(par * 4 + q) * 256 + 32 * c + lane] = cs[0];
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int ocol = EPI == XE_PAIRSUM ? 32 * c : col0;
            const int orow = r0 + (p.splits > 1 ? ks * p.Mp : 0);
            tma_store_2d(&tm_o, sptr, ocol, orow);
            bulk_commit_group();
          }
          if constexpr (EPI == XE_MSE) {
            // the store of the previous chunk has read its box: prefetch two chunks ahead into it
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
            load_next();
          }
        }
      }
      if constexpr (EPI == XE_MSE) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) p.loss_part[((int64_t)u * 2 + crank) * XEPI + e] = sq;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_leader_x(&tempty[acc], crank);
      if (++acc == 2) { acc = 0; aphase ^= 1; }
      if constexpr (EPI == XE_MSE) {
        // the CTA's column sums of the unit: four lane quarters added in quarter order
        named_bar_sync(1, 32 * XEPI);
        const int t = threadIdx.x - 64;
        if (t < BN && nb * BN + t < p.N)
          p.colsum_part[(int64_t)(mb * 2 + (int)crank) * p.N + nb * BN + t] =
              ((red[(par * 4 + 0) * 256 + t] + red[(par * 4 + 1) * 256 + t]) +
               red[(par * 4 + 2) * 256 + t]) + red[(par * 4 + 3) * 256 + t];
        par ^= 1;
      }
    }
    if (lane == 0) bulk_wait_group<0>();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

typedef void (*XgFn)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, XgParams);

template <int YDT>
XgFn pick_t(int act) {  // XE_STORE_T (bf16 operands: the general-path forward)
  switch (act) {
    case DT_ACT_RELU: return k_tc_xgemm<0, XE_STORE_T, YDT, DT_ACT_RELU>;
    case DT_ACT_SIGMOID: return k_tc_xgemm<0, XE_STORE_T, YDT, DT_ACT_SIGMOID>;
    case DT_ACT_TANH: return k_tc_xgemm<0, XE_STORE_T, YDT, DT_ACT_TANH>;
    case DT_ACT_CLIPPED_RELU: return k_tc_xgemm<0, XE_STORE_T, YDT, DT_ACT_CLIPPED_RELU>;
    default: return k_tc_xgemm<0, XE_STORE_T, YDT, DT_ACT_IDENTITY>;
  }
}

template <int EL>
XgFn pick_x(int epi) {
  switch (epi) {
    case XE_MSE: return k_tc_xgemm<EL, XE_MSE>;
    case XE_PAIRSUM: return k_tc_xgemm<EL, XE_PAIRSUM>;
    case XE_SPLITH: return k_tc_xgemm<EL, XE_SPLITH>;
    default: return k_tc_xgemm<EL, XE_STORE>;
  }
}

// out (or out^T) = sum over splits (fixed order) of the partial slices, optionally the hi + lo
// column halves added (pair_half > 0: columns [0, pair_half) + [pair_half, 2 pair_half)).
__global__ void k_xg_reduce(int splits, int M, int N, int Mp, const float *part, float *out,
                            int ldo, int transpose, int pair_half) {
  const int cols = pair_half > 0 ? pair_half : N;
  const int64_t total = (int64_t)M * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int m, n;
    if (transpose) {  // consecutive threads walk m: coalesced writes of out[n][m]
      n = (int)(i / M);
      m = (int)(i - (int64_t)n * M);
    } else {
      m = (int)(i / cols);
      n = (int)(i - (int64_t)m * cols);
    }
    float s = 0.f;
    for (int k = 0; k < splits; ++k) {
      const float *sl = part + ((int64_t)k * Mp + m) * N;
      s += sl[n];
      if (pair_half > 0) s += sl[n + pair_half];
    }
    if (transpose)
      out[(int64_t)n * ldo + m] = s;
    else
      out[(int64_t)m * ldo + n] = s;
  }
}

// column sums over the [rows][N] partials (d_bias from XE_MSE's per-CTA sums), two fixed-order
// levels: block (x, y) sums rows [y*kRowsPer, ...) of its columns into mid[y][n], then k_colsum_mid
// adds the mid rows in order
constexpr int kRowsPer = 32;
__global__ void k_colsum_rows(int rows, int N, const float *part, float *mid) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int r0 = blockIdx.y * kRowsPer, r1 = min(rows, r0 + kRowsPer);
  float s = 0.f;
  for (int r = r0; r < r1; ++r) s += part[(int64_t)r * N + n];
  mid[(int64_t)blockIdx.y * N + n] = s;
}
__global__ void k_colsum_mid(int chunks, int N, const float *mid, float *out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int c = 0; c < chunks; ++c) s += mid[(int64_t)c * N + n];
  out[n] = s;
}

// fixed-order fp64 sum of many partials: block b sums its contiguous slice (strided per thread,
// tree in shared memory), then one block adds the block sums in order
__global__ void __launch_bounds__(256) k_sum_f64_blocks(int64_t count, const double *part,
                                                        double *mid) {
  __shared__ double red[256];
  const int64_t per = (count + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(count, b0 + per);
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += 256) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = 128; h; h >>= 1) {
    if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) mid[blockIdx.x] = red[0];
}
__global__ void k_sum_f64_final(int n, const double *mid, double *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += mid[i];
    out[0] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------------------------
size_t xgemm_ws(const XGemm &g) {
  if (g.splits <= 1 && !g.reduce_transpose && g.reduce_pair_half <= 0 && !g.force_part) return 0;
  const int64_t Mp = (g.M + 255) / 256 * 256;
  return (size_t)g.splits * Mp * g.N * 4;
}

int xgemm_splits(int64_t M, int64_t N, int64_t K, int BN, int el, int nsm) {
  const int64_t tiles = ((M + 255) / 256) * ((N + BN - 1) / BN);
  const int64_t kb = (K + (el ? 31 : 63)) / (el ? 32 : 64);
  const int64_t ncl = nsm / 2;
  if (tiles >= ncl) return 1;
  // enough units for every cluster, several waves when that balances better, >= 8 k-blocks each
  int best = 1;
  double best_eff = (double)tiles / ncl;
  for (int s = 2; s <= 64 && kb / s >= 8; ++s) {
    const double units = (double)tiles * s;
    const double waves = std::ceil(units / ncl);
    const double eff = units / (waves * ncl) - 0.002 * s;  // partial-slice traffic
    if (eff > best_eff) { best_eff = eff; best = s; }
  }
  return best;
}

int xgemm(const XGemm &g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return DT_OK;
  const int el = g.el;
  const int esz = el ? 4 : 2, bke = el ? 32 : 64;
  int BN = g.BN;
  if (BN != 64 && BN != 128 && BN != 256) {
    set_error("xgemm: BN must be 64, 128 or 256");
    return DT_E_ARG;
  }
  const int nhalf = BN / 2;
  if (g.b_mn && nhalf * esz < 128) {
    set_error("xgemm: an MN-major B needs BN/2 * element size >= 128 bytes");
    return DT_E_ARG;
  }
  if (g.epi == XE_PAIRSUM && (g.N > BN || 2 * g.pair_half > g.N || g.pair_half <= 0 || g.splits > 1)) {
    set_error("xgemm: the pair-sum epilogue needs one column block (N <= BN), no split");
    return DT_E_ARG;
  }
  if (g.epi == XE_SPLITH && g.splits > 1) {
    set_error("xgemm: the H split epilogue takes no split");
    return DT_E_ARG;
  }
  int dev = 0, nsm = 148;
  DT_CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);

  XgParams p{};
  p.M = (int)g.M;
  p.N = (int)g.N;
  p.BN = BN;
  p.nhalf = nhalf;
  p.n_mb = (int)((g.M + 255) / 256);
  p.n_nb = (int)((g.N + BN - 1) / BN);
  p.kb_total = (int)((g.K + bke - 1) / bke);
  p.splits = std::max(1, std::min(g.splits, p.kb_total));
  p.kb_per = (p.kb_total + p.splits - 1) / p.splits;
  p.splits = (p.kb_total + p.kb_per - 1) / p.kb_per;  // no empty split
  p.units = p.n_mb * p.n_nb * p.splits;
  p.a_mn = g.a_mn;
  p.b_mn = g.b_mn;
  p.b_wrap = g.b_wrap_k > 0 ? (int)(g.b_wrap_k / bke) : 0;
  if (g.b_wrap_k > 0 && g.b_wrap_k % bke) {
    set_error("xgemm: the B wrap length must be a multiple of the k-block");
    return DT_E_ARG;
  }
  p.Mp = p.n_mb * 256;
  p.alpha = g.alpha;
  p.bias = g.bias;
  p.ldo = (int)g.ldo;
  p.scale = g.scale;
  p.loss_part = g.loss_part;
  p.colsum_part = g.colsum_part;
  p.out16 = g.out16;
  p.h_r = g.h_r;
  p.h_s = g.h_s;
  p.pair_half = g.pair_half;
  p.ks_major = g.ks_major;
  p.dual_kb = g.dual_k > 0 ? (int)(g.dual_k / bke) : 0;
  if (g.dual_k > 0 && (g.dual_k % bke || g.a_mn)) {
    set_error("xgemm: the dual-A offset must be whole k-blocks of a K-major A");
    return DT_E_ARG;
  }
  p.stage_bytes = (p.dual_kb > 0 ? 2u : 1u) * XA_BYTES + (uint32_t)nhalf * 128u;
  // XE_STORE_T with fp32 outputs stores through TMA when y's base and pitch allow a tensor map
  // (one 4 KB box per epilogue warp, used as two alternating 16-row halves)
  const bool tma_t = g.epi == XE_STORE_T && g.y_dtype == DT_F32 && g.ldo % 4 == 0 &&
                     (reinterpret_cast<uintptr_t>(g.out_t) & 15) == 0 &&
                     !DT_DBG_ENV("DEEPTHIN_DBG_XG_NOTMA");
  p.tma_t = tma_t ? 1 : 0;
  const uint32_t stg_bytes = g.epi == XE_SPLITH ? 0u
                             : g.epi == XE_STORE_T ? (tma_t ? (uint32_t)XEPI * XSTG : 0u)
                             : (uint32_t)XEPI * (g.epi == XE_MSE ? 3u : 2u) * XSTG;
  // barriers + TMEM slot (512 B), then the XE_MSE column-sum exchange [2][4][256] floats
  const uint32_t tail = 512 + (g.epi == XE_MSE ? 8192u : 0u);
  // A pipelined forward (chain) leaves room for one CTA of the next call's W regeneration
  // (k_regen_wt: 22 KB static + 1 KB reserved) beside this kernel on every SM, so that grid
  // runs under this GEMM instead of after it.
  const uint32_t smem_cap = g.chain ? XSMEM_MAX - 26 * 1024 : XSMEM_MAX;
  p.S = (int)std::min<uint32_t>(8, (smem_cap - stg_bytes - tail - 1024) / p.stage_bytes);
  if (DT_DBG_ENV("DEEPTHIN_DBG_XG_S") > 0) p.S = DT_DBG_ENV("DEEPTHIN_DBG_XG_S");
  p.off_stg = (uint32_t)p.S * p.stage_bytes;
  p.off_bar = p.off_stg + stg_bytes;
  const uint32_t smem_bytes = p.off_bar + tail + 1024;  // + the in-kernel 1024-B alignment
  if (p.S < 2) {
    set_error("xgemm: shared memory too small");
    return DT_E_UNSUPPORTED;
  }

  CUtensorMap tm_a, tm_b, tm_o, tm_t;
  const int tdt = el ? DT_F32 : DT_BF16;
  void *A = const_cast<void *>(g.A), *B = const_cast<void *>(g.B);
  // A: K-major [M][lda] box (bke, 128); MN-major [K][lda] box (128 B of M, bke)
  const int mn_sw = el ? (int)CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : (int)CU_TENSOR_MAP_SWIZZLE_128B;
  // MN-major operands whose extent is whole 128-byte chunks load through a 3-D map: one TMA per
  // half-tile instead of one per chunk (measured: the 2-D form made MN-major tf32 GEMMs 20-30 %
  // slower than K-major ones)
  const int ce = 128 / esz;
  const bool a3 = g.a_mn && g.M % ce == 0 && (g.lda * esz) % 16 == 0;
  const bool b3 = g.b_mn && g.N % ce == 0 && (g.ldb * esz) % 16 == 0 && nhalf % ce == 0;
  if (a3) p.a_mn = 2;
  if (b3) p.b_mn = 2;
  if (int rc = a3 ? encode_tensor_map_mn3d(&tm_a, tdt, A, (uint64_t)g.M, (uint64_t)g.K,
                                           (uint64_t)g.lda * esz, bke, 128 / ce, mn_sw)
               : g.a_mn ? encode_tensor_map_2d_sw(&tm_a, tdt, A, (uint64_t)g.M, (uint64_t)g.K,
                                                (uint64_t)g.lda * esz, 128 / esz, bke, mn_sw)
                      : encode_tensor_map_2d(&tm_a, tdt, A, (uint64_t)(g.K + g.dual_k), (uint64_t)g.M,
                                             (uint64_t)g.lda * esz, bke, 128, true))
    return rc;
  // rows of B along K: the wrap length, or the stored extent when shorter (zero fill past it)
  const uint64_t kb_rows = g.b_wrap_k > 0 ? (uint64_t)(g.b_rows > 0 ? std::min(g.b_rows, g.b_wrap_k)
                                                                   : g.b_wrap_k)
                                          : (uint64_t)(g.b_rows > 0 ? std::min(g.b_rows, g.K) : g.K);
  if (int rc = b3 ? encode_tensor_map_mn3d(&tm_b, tdt, B, (uint64_t)g.N, kb_rows,
                                           (uint64_t)g.ldb * esz, bke, (uint32_t)(nhalf / ce), mn_sw)
               : g.b_mn ? encode_tensor_map_2d_sw(&tm_b, tdt, B, (uint64_t)g.N, kb_rows,
                                                (uint64_t)g.ldb * esz, 128 / esz, bke, mn_sw)
                      : encode_tensor_map_2d(&tm_b, tdt, B, kb_rows, (uint64_t)g.N,
                                             (uint64_t)g.ldb * esz, bke, (uint32_t)nhalf, true))
    return rc;
  float *out = g.out;
  int64_t out_rows = g.M, out_cols = g.epi == XE_PAIRSUM ? g.pair_half : g.N, ldo = g.ldo;
  // partial slices (then the fixed-order reduce) for split-K, and for a transposed or
  // column-paired result
  const bool use_part = p.splits > 1 || g.reduce_transpose || g.reduce_pair_half > 0 ||
                        g.force_part;
  if (use_part && g.epi != XE_STORE) {
    set_error("xgemm: split / transposed / paired results need the store epilogue");
    return DT_E_ARG;
  }
  if (use_part) {
    if (!g.part) {
      set_error("xgemm: split-K needs a partial buffer (xgemm_ws bytes)");
      return DT_E_ARG;
    }
    out = g.part;
    out_rows = (int64_t)p.splits * p.Mp;
    out_cols = g.N;
    ldo = g.N;
    p.ldo = (int)g.N;
  }
  p.chain = g.chain;
  p.dbg = DT_DBG_ENV("DEEPTHIN_DBG_XG");
  p.act_arg = g.act_arg;
  p.out_t = g.out_t;
  p.N_true = (int)g.N;
  if (g.epi != XE_SPLITH && g.epi != XE_STORE_T) {
    if (int rc = encode_tensor_map_2d(&tm_o, DT_F32, out, (uint64_t)out_cols, (uint64_t)out_rows,
                                      (uint64_t)ldo * 4, 32, 32, true))
      return rc;
  } else if (tma_t) {  // y[batch][r_dim]: boxes of 32 output columns x 16 batch rows
    if (int rc = encode_tensor_map_2d(&tm_o, DT_F32, g.out_t, (uint64_t)g.M, (uint64_t)g.N,
                                      (uint64_t)g.ldo * 4, 32, 16, true))
      return rc;
  } else {
    tm_o = tm_a;  // unused
  }
  if (g.epi == XE_MSE) {
    if (int rc = encode_tensor_map_2d(&tm_t, DT_F32, const_cast<float *>(g.target), (uint64_t)g.N,
                                      (uint64_t)g.M, (uint64_t)g.ldt * 4, 32, 32, true))
      return rc;
  } else {
    tm_t = tm_a;  // unused
  }
  if (g.epi == XE_MSE && g.loss_part)
    DT_CUDA_CHECK(cudaMemsetAsync(g.loss_part, 0, (size_t)p.units * 2 * XEPI * 8, st));

  XgFn fn;
  if (g.epi == XE_STORE_T) {
    if (el) {
      set_error("xgemm: the transposed-store epilogue takes bf16 operands");
      return DT_E_ARG;
    }
    fn = g.y_dtype == DT_BF16 ? pick_t<DT_BF16>(g.act) : pick_t<DT_F32>(g.act);
  } else {
    fn = el ? pick_x<1>(g.epi) : pick_x<0>(g.epi);
  }
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  const int ncl = std::max(1, std::min(p.units, nsm / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * ncl));
  cfg.blockDim = dim3(XTHREADS);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm_a, tm_b, tm_o, tm_t, p));
  if (int rc = check_launch("tc_xgemm")) return rc;
  if (g.n_loss_part) *g.n_loss_part = (int64_t)p.units * 2 * XEPI;

  if (use_part) {
    const int pair = g.reduce_pair_half;
    const int64_t total = g.M * (pair > 0 ? pair : g.N);
    k_xg_reduce<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8 * nsm), 256, 0, st>>>(
        p.splits, (int)g.M, (int)g.N, p.Mp, g.part, g.out, (int)g.ldo, g.reduce_transpose ? 1 : 0,
        pair);
    if (int rc = check_launch("xg_reduce")) return rc;
  }
  return DT_OK;
}

size_t xgemm_reduce_scratch(int rows, int64_t N) {
  return (size_t)((rows + kRowsPer - 1) / kRowsPer) * N * 4 + 64 * 8;
}

int xgemm_colsum(int rows, int64_t N, const float *part, float *out, void *scratch, cudaStream_t st) {
  const int chunks = (rows + kRowsPer - 1) / kRowsPer;
  float *mid = reinterpret_cast<float *>(scratch);
  k_colsum_rows<<<dim3((unsigned)((N + 255) / 256), (unsigned)chunks), 256, 0, st>>>(rows, (int)N,
                                                                                   part, mid);
  if (int rc = check_launch("colsum_rows")) return rc;
  k_colsum_mid<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(chunks, (int)N, mid, out);
  return check_launch("colsum_mid");
}

int xgemm_sum_f64(int64_t count, const double *part, double *out, void *scratch, cudaStream_t st) {
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(64, (count + 2047) / 2048));
  double *mid = reinterpret_cast<double *>(scratch);
  k_sum_f64_blocks<<<nb, 256, 0, st>>>(count, part, mid);
  if (int rc = check_launch("sum_f64_blocks")) return rc;
  k_sum_f64_final<<<1, 32, 0, st>>>(nb, mid, out);
  return check_launch("sum_f64_final");
}

}  // namespace dt
