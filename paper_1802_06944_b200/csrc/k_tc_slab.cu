// Row-slab tensor-core forward for reuse geometries (n_f | q, s = q / n_f a power of two): the
// factored DeepThin layer in ONE persistent kernel without clusters. Every CTA owns a contiguous
// slab of batch rows (batch / #SMs, rounded to the phase-A unit), reads those rows of x once and
// writes those rows of y once: all SMs stream, no P exchange between CTAs, no tail round.
//
// Reference: kernel.py:1-16 / 99-164 (the reuse identity: every output column reads s = q/n
// whole rows of I = xf @ wf, so each distinct run dot x_seg . wf[k] is computed once) and
// kernel.py:296-320 (layer_forward = act(x W + b)).
//
//   phase A:  x viewed as x' (batch*s x n): P'[b*s + seg, k] = sum_t x'[b*s + seg, t] wf[k, t]
//             — one UMMA of M = 128 x' rows covers 128/s batch rows with ALL their segments
//             (bf16 x bf16 -> fp32 in TMEM; wf as bf16 hi | lo in the two N halves)
//   re-lay:   TMEM lane (b*s + seg) -> row b, K slots [seg*rp, seg*rp + rank) of the tf32 A
//             operand of phase B (128-byte swizzled K-major rows in shared memory)
//   phase B:  y[b, j] = act(sum_kk A2[b, kk] XF2p[j, kk])   (kind::tf32, bias in a K pad slot)
//             per group of up to 64 batch rows, 128 output columns per D buffer, XF2p chunks
//             streamed from L2. A group's rows sit in TMEM lanes 32 q + (0..15), q = 0..3 (the
//             re-lay chooses the A2 row): every epilogue warp reads its quarter's 16 live lanes
//             with the 16-lane tcgen05.ld shape, so all 32 threads hold live values (the
//             epilogue is MUFU-bound: one tanh per output) although the UMMA runs M = 128.
//             Groups of 64 let a slab's first stores overlap its later loads.
//   epilogue: D (TMEM) -> activation -> bf16/fp32 -> swizzled staging -> TMA store (16 x 32
//             boxes); the fused row softmax (two passes, the contraction recomputed) needs no
//             exchange: a CTA holds whole rows.
//
// Warp roles (768 threads, one CTA per SM):
//   warp 0  TMA producer of x' k-blocks (128 x' rows x 64 bf16, SW128)
//   warp 1  TMA producer of XF2p chunks (128 output columns x 32 fp32, SW128)
//   warp 2  TMEM allocator + single-thread tcgen05.mma issuer of phase A (P ring of 8 units)
//   warp 3  single-thread tcgen05.mma issuer of phase B
//   warps 4-7   P re-lay (one per TMEM lane quarter)
//   warps 8-23  epilogue (four per lane quarter, each 32 of a chunk's 128 columns)
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "act.cuh"
#include "dt_internal.h"
#include "rows_common.cuh"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;
using namespace rowsdev;

constexpr int kGM = 64;            // batch rows per phase-B group (16 live lanes per TMEM quarter)
constexpr int kMM = 128;           // UMMA M of phase B (= A2 rows = TMEM lanes)
constexpr int kNc = 128;           // output columns per D chunk (UMMA N of phase B)
constexpr int kXSMax = 8;          // x ring depth cap
constexpr int kBSMax = 4;          // XF2p chunk ring depth cap
constexpr int kPS = 8;             // P ring: phase-A units in TMEM
constexpr int kPW = 4;             // re-lay warps
constexpr int kEpi = 16;           // epilogue warps
constexpr int kSlabThreads = 32 * (4 + kPW + kEpi);
constexpr uint32_t kXBytes = 128 * 128;   // 128 x' rows x 64 bf16
constexpr uint32_t kBBytes = kNc * 128;   // 128 columns x 32 fp32
constexpr uint32_t kA2Bytes = kMM * 128;  // 128 rows x 32 fp32
constexpr int kTr = 64;                   // trace slots per CTA

struct SlabParams {
  int64_t batch;
  int r_dim, s, ls, nkb, np, rank, rp, k2, n_chunks;
  int ur;       // batch rows per phase-A unit (128 / s)
  int slab;     // batch rows per CTA (a multiple of max(ur, 16))
  int xs, bs, nd;
  int nstage;   // output staging boxes per epilogue warp (TMA stores in flight)
  int dbg;      // timing build only (DEEPTHIN_DBG_SLAB): 1 no TMA store, 2 no staging, 3 no act
  uint32_t dcol0;
  int bslot;    // K slot carrying the bias (A2 = 1 there), -1: the epilogue adds it
  int softmax;
  const float *bias;
  float arg;
  uint32_t off_a2, off_wf, off_b, off_out, off_red, off_x, off_bar;
  unsigned long long *trace;
};

__device__ __forceinline__ void strace(const SlabParams &p, int slot) {
  if (p.trace && slot < kTr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[blockIdx.x * kTr + slot] = t;
  }
}

__device__ __forceinline__ void st_shared_b32(uint32_t addr, uint32_t a) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

// this warp's 16 x 32 outputs in the 16x256b register layout (o[4i], o[4i+1]: row lane/4,
// columns 8i + 2(lane%4) + {0,1}; o[4i+2], o[4i+3]: row 8 + lane/4) into its swizzled staging
// box (the TMA SW64 / SW128 pattern: 16-byte chunk ch of row r at ch ^ (r >> 1 & 3) / ch ^ (r & 7))
template <int E>
__device__ __forceinline__ void stage_16x32(uint32_t out_s, int lane, const float (&o)[16]) {
  const int r = lane >> 2, cp = lane & 3;
  if constexpr (E == 2) {  // rows of 64 bytes; (r + 8) >> 1 & 3 == r >> 1 & 3
    const uint32_t lo = out_s + (uint32_t)r * 64u + (uint32_t)cp * 4u, hi = lo + 8u * 64u;
    const int sw = (r >> 1) & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      st_shared_b32(lo + ((uint32_t)(i ^ sw) << 4), pack_bf16(o[4 * i], o[4 * i + 1]));
      st_shared_b32(hi + ((uint32_t)(i ^ sw) << 4), pack_bf16(o[4 * i + 2], o[4 * i + 3]));
    }
  } else {  // rows of 128 bytes; (r + 8) & 7 == r
    const uint32_t lo = out_s + (uint32_t)r * 128u + (uint32_t)(cp & 1) * 8u, hi = lo + 8u * 128u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t ch = (uint32_t)((2 * i + (cp >> 1)) ^ r) << 4;
      st_shared_v2(lo + ch, __float_as_uint(o[4 * i]), __float_as_uint(o[4 * i + 1]));
      st_shared_v2(hi + ch, __float_as_uint(o[4 * i + 2]), __float_as_uint(o[4 * i + 3]));
    }
  }
}

template <int YDT, int ACT>
__global__ void __launch_bounds__(kSlabThreads, 1)
    k_tc_rows_slab(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_wf,
                   const __grid_constant__ CUtensorMap tm_xf2, const __grid_constant__ CUtensorMap tm_y,
                   const SlabParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *x_full = bars, *x_empty = x_full + kXSMax;
  uint64_t *b_full = x_empty + kXSMax, *b_empty = b_full + kBSMax;
  uint64_t *d_full = b_empty + kBSMax, *d_empty = d_full + 4;
  uint64_t *p_full = d_empty + 4, *p_free = p_full + kPS;
  uint64_t *a2_full = p_free + kPS, *a2_free = a2_full + 2;
  uint64_t *wf_full = a2_free + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(wf_full + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // this CTA's slab: rows [row_begin, row_begin + rows), in groups of kGM, each group in units
  // of ur rows
  const int64_t row_begin = (int64_t)blockIdx.x * p.slab;
  const int rows = (int)min((int64_t)p.slab, p.batch - row_begin);
  const int n_groups = (rows + kGM - 1) / kGM;
  // Every CTA streams every XF2p chunk: CTA i starts at chunk i mod n_chunks, so that at any
  // time the CTAs read n_chunks different chunks (all of them on the same 128 lines at once
  // serialise on a few L2 slices: measured 0.53 us per chunk with nothing else running). The
  // softmax passes keep the natural order: their sums run in chunk order, which must not
  // depend on the CTA a row falls in.
  const int rot = p.softmax ? 0 : (int)(blockIdx.x % (unsigned)p.n_chunks);

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.xs; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < p.bs; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 4; ++i) { mbar_init(&d_full[i], 1); mbar_init(&d_empty[i], kEpi); }
    for (int i = 0; i < kPS; ++i) { mbar_init(&p_full[i], 1); mbar_init(&p_free[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&a2_full[i], 1); mbar_init(&a2_free[i], 1); }
    mbar_init(wf_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wf);
    tma_prefetch_desc(&tm_xf2);
    tma_prefetch_desc(&tm_y);
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) strace(p, 0);
  // x is the previous layer's output; factors / bias may come from a prep kernel or an SGD step
  griddep_wait();
  griddep_launch_dependents();
  if (threadIdx.x == 0) strace(p, 1);

  if (warp == 0) {
    // ---------------- x' producer ----------------
    if (lane == 0) {
      uint8_t *wf_s = smem + p.off_wf;
      mbar_arrive_expect_tx(wf_full, (uint32_t)(p.nkb * p.np * 128));
      for (int kb = 0; kb < p.nkb; ++kb)
        tma_load_2d(wf_s + kb * p.np * 128, &tm_wf, wf_full, kb * 64, 0);
      int st = 0;
      uint32_t ph = 0;
      for (int g = 0; g < n_groups; ++g) {
        const int g_rows = min(kGM, rows - g * kGM);
        const int g_units = (g_rows + p.ur - 1) / p.ur;
        for (int u = 0; u < g_units; ++u) {
          // x' rows of the unit: (first batch row) * s .. + 128 (past the batch: zero-filled)
          const int32_t r0 = (int32_t)((row_begin + g * kGM + u * p.ur) << p.ls);
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&x_empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&x_full[st], kXBytes);
            tma_load_2d(smem + p.off_x + st * kXBytes, &tm_x, &x_full[st], kb * 64, r0);
            if (++st == p.xs) { st = 0; ph ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- XF2p chunk producer (every chunk once per group and pass) ----------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int g = 0; g < n_groups; ++g)
        for (int pass = 0; pass < (p.softmax ? 2 : 1); ++pass)
          for (int ci = 0; ci < p.n_chunks; ++ci) {
            const int c = ci + rot < p.n_chunks ? ci + rot : ci + rot - p.n_chunks;
            mbar_wait(&b_empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&b_full[st], kBBytes);
            tma_load_2d(smem + p.off_b + st * kBBytes, &tm_xf2, &b_full[st], 0, c * kNc);
            if (++st == p.bs) { st = 0; ph ^= 1; }
          }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ---------------- phase-A MMA issuer: P[unit] = x' unit . [wf_hi | wf_lo]^T ----------------
    if (lane == 0) {
      const uint32_t s0 = smem_u32(smem);
      const uint32_t wf_s = s0 + p.off_wf;
      const uint32_t idA = idesc_f32acc(128, (uint32_t)p.np, 1);
      mbar_wait(wf_full, 0);
      int xs = 0;
      uint32_t xph = 0, seq = 0;
      for (int g = 0; g < n_groups; ++g) {
        const int g_rows = min(kGM, rows - g * kGM);
        const int g_units = (g_rows + p.ur - 1) / p.ur;
        for (int u = 0; u < g_units; ++u, ++seq) {
          const uint32_t slot = seq % kPS;
          mbar_wait(&p_free[slot], ((seq / kPS) & 1u) ^ 1u);  // the re-lay warps read unit seq-8
          tc_fence_after();
          const uint32_t d = tbase + slot * (uint32_t)p.np;
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&x_full[xs], xph);
            if (seq == 0 && kb == 0) strace(p, 2);
            tc_fence_after();
            const uint32_t a = s0 + p.off_x + (uint32_t)xs * kXBytes;
            const uint32_t b = wf_s + (uint32_t)(kb * p.np * 128);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16_ss(d, smem_desc(a + k * 32, 16, 1024, SL_SW128),
                          smem_desc(b + k * 32, 16, 1024, SL_SW128), idA, (kb | k) != 0);
            mma_commit(&x_empty[xs]);
            if (++xs == p.xs) { xs = 0; xph ^= 1; }
          }
          mma_commit(&p_full[slot]);
          if (u == g_units - 1) strace(p, 3 + 8 * min(g, 6));
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ---------------- phase-B MMA issuer: D = A2[group] . XF2p chunk^T (tf32) ----------------
    if (lane == 0) {
      const uint32_t s0 = smem_u32(smem);
      const uint32_t idB = idesc_f32acc(kMM, kNc, 2);
      int bs = 0, db = 0;
      uint32_t bph = 0, dph = 0;
      for (int g = 0; g < n_groups; ++g) {
        const int gb = g & 1;
        mbar_wait(&a2_full[gb], (uint32_t)(g >> 1) & 1u);
        strace(p, 4 + 8 * min(g, 6));
        tc_fence_after();
        const uint32_t a2_s = s0 + p.off_a2 + (uint32_t)gb * kA2Bytes;
        for (int pass = 0; pass < (p.softmax ? 2 : 1); ++pass)
          for (int c = 0; c < p.n_chunks; ++c) {
            mbar_wait(&b_full[bs], bph);
            mbar_wait(&d_empty[db], dph ^ 1);
            tc_fence_after();
            const uint32_t d = tbase + p.dcol0 + (uint32_t)(db * kNc);
            const uint32_t b = s0 + p.off_b + (uint32_t)bs * kBBytes;
            for (int k = 0; k < p.k2 / 8; ++k)
              mma_tf32_ss(d, smem_desc(a2_s + k * 32, 16, 1024, SL_SW128),
                          smem_desc(b + k * 32, 16, 1024, SL_SW128), idB, k != 0);
            mma_commit(&b_empty[bs]);
            if (++bs == p.bs) { bs = 0; bph ^= 1; }
            mma_commit(&d_full[db]);
            if (++db == p.nd) { db = 0; dph ^= 1; }
          }
        mma_commit(&a2_free[gb]);  // this group's reads of A2[gb] are done when these complete
      }
    }
    __syncwarp();
  } else if (warp < 4 + kPW) {
    // ---------------- P re-lay: TMEM lane (b*s + seg) -> A2 row b, K slots of seg ----------------
    const int sp = warp & 3, lrow = 32 * sp + lane;  // x' row of the unit = TMEM lane
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    const uint32_t a2_local = smem_u32(smem) + p.off_a2;
    const int seg = lrow & (p.s - 1), bq = lrow >> p.ls;
    const int cpr = p.rp / 4;  // 16-byte chunks per segment
    // K padding of the tf32 operand (never overwritten): zero, 1.0 in a bias slot past s*rp
    for (int b = 0; b < 2; ++b)
      for (int kk = p.s * p.rp; kk < p.k2; kk += 4)
        st_shared_v4(a2_local + (uint32_t)b * kA2Bytes + (uint32_t)lrow * 128u +
                         ((uint32_t)((kk >> 2) ^ (lrow & 7)) << 4),
                     kk == p.bslot ? 0x3f800000u : 0u, 0u, 0u, 0u);
    uint32_t seq = 0;
    for (int g = 0; g < n_groups; ++g) {
      const int gb = g & 1;
      const int g_rows = min(kGM, rows - g * kGM);
      const int g_units = (g_rows + p.ur - 1) / p.ur;
      mbar_wait(&a2_free[gb], ((uint32_t)(g >> 1) & 1u) ^ 1u);  // phase B of group g-2 finished
      const uint32_t a2b = a2_local + (uint32_t)gb * kA2Bytes;
      for (int u = 0; u < g_units; ++u, ++seq) {
        const uint32_t slot = seq % kPS;
        mbar_wait(&p_full[slot], (seq / kPS) & 1u);
        tc_fence_after();
        // columns [0, rank) hold x' . wf_hi, [rank, 2 rank) x' . wf_lo: two loads, the second
        // offset by rank columns, so P = hi + lo pairs up register by register
        const uint32_t pcol = tbase + lane_t + slot * (uint32_t)p.np;
        uint32_t vh[32], vl[32];
        tmem_ld_32x32b_x32(pcol, vh);
        tmem_ld_32x32b_x32(pcol + (uint32_t)p.rank, vl);
        tmem_ld_wait();
        // batch row u*ur + bq of the group -> A2 row (= TMEM lane) 32 (r / 16) + r % 16
        const int grow = u * p.ur + bq;
        const int row = 32 * (grow >> 4) + (grow & 15);
        const uint32_t rbase = a2b + (uint32_t)row * 128u;
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
            const int ch = seg * cpr + (k0 >> 2);
            st_shared_v4(rbase + ((uint32_t)(ch ^ (row & 7)) << 4), w[0], w[1], w[2], w[3]);
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();  // visible to the phase-B MMAs (async proxy)
        named_bar_sync(1, 32 * kPW);
        if (warp == 4 && lane == 0) {
          mbar_arrive(&p_free[slot]);
          if (u == g_units - 1) mbar_arrive(&a2_full[gb]);
        }
      }
    }
  } else {
    // ---------------- epilogue: 16 warps, four per TMEM lane quarter ----------------
    // quarter sp holds group rows 16 sp .. 16 sp + 15 in its lanes 0..15; warp (sp, qc) takes
    // columns 32 qc .. 32 qc + 31 of every 128-column chunk in the 16x256b register layout:
    // this thread has rows ra = lane/4 and ra + 8, columns 8i + 2(lane%4) + {0,1}, i = 0..3
    const int sp = warp & 3;
    const int e = warp - 4 - kPW;      // 0..15
    const int qc = e / 4;
    const int ra = lane >> 2, cp = lane & 3;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    constexpr int E = YDT == DT_BF16 ? 2 : 4;
    constexpr int RB = 32 * E;         // bytes per row of this warp's 32 columns (64 or 128)
    const uint32_t out_s0 = s0 + p.off_out + (uint32_t)(e * p.nstage) * (16u * RB);
    int sb = 0;
    const int64_t slab_end = row_begin + rows;
    const float l2e = 1.4426950408889634f;
    int db = 0;
    uint32_t dph = 0;
    for (int g = 0; g < n_groups; ++g) {
      const int64_t row0 = row_begin + g * kGM + 16 * sp;
      // this quarter's 16 rows lie inside the slab (slabs end on multiples of 16; the batch end
      // is clipped by TMA) or past it (no store)
      const bool live = row0 < slab_end;
      float Ma = 0.f, Mb = 0.f, inva = 1.f, invb = 1.f;
      if (p.softmax) {
        // pass 1: per row, the online (max, sum 2^((z - max) log2 e)) over this warp's columns of
        // every chunk (the four threads of a row combined by shuffles), then the four column
        // warps combined in a fixed order (deterministic)
        float2 *red = reinterpret_cast<float2 *>(smem + p.off_red) + (g & 1) * 4 * kGM;  // [4][64]
        float ma = -INFINITY, la = 0.f, mb = -INFINITY, lb = 0.f;
        for (int c = 0; c < p.n_chunks; ++c) {
          mbar_wait(&d_full[db], dph);
          tc_fence_after();
          uint32_t v[16];
          tmem_ld_16x256b_x4(tbase + lane_t + p.dcol0 + (uint32_t)(db * kNc + 32 * qc), v);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[db]);
          if (++db == p.nd) { db = 0; dph ^= 1; }
          const int col0 = c * kNc + 32 * qc;
          if (col0 >= p.r_dim) continue;  // (uniform over the warp)
          float ca = -INFINITY, cb = -INFINITY;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (col0 + 8 * i + 2 * cp < p.r_dim) {  // r_dim is even: the pair is in or out
              ca = fmaxf(ca, fmaxf(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1])));
              cb = fmaxf(cb, fmaxf(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3])));
            }
          ca = fmaxf(ca, __shfl_xor_sync(0xffffffffu, ca, 1));
          ca = fmaxf(ca, __shfl_xor_sync(0xffffffffu, ca, 2));
          cb = fmaxf(cb, __shfl_xor_sync(0xffffffffu, cb, 1));
          cb = fmaxf(cb, __shfl_xor_sync(0xffffffffu, cb, 2));
          const float na = fmaxf(ma, ca), nb = fmaxf(mb, cb);
          float sa = 0.f, sb = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (col0 + 8 * i + 2 * cp < p.r_dim) {
              sa += ex2_approx((__uint_as_float(v[4 * i]) - na) * l2e) +
                    ex2_approx((__uint_as_float(v[4 * i + 1]) - na) * l2e);
              sb += ex2_approx((__uint_as_float(v[4 * i + 2]) - nb) * l2e) +
                    ex2_approx((__uint_as_float(v[4 * i + 3]) - nb) * l2e);
            }
          sa += __shfl_xor_sync(0xffffffffu, sa, 1);
          sa += __shfl_xor_sync(0xffffffffu, sa, 2);
          sb += __shfl_xor_sync(0xffffffffu, sb, 1);
          sb += __shfl_xor_sync(0xffffffffu, sb, 2);
          la = (ma > -INFINITY ? la * ex2_approx((ma - na) * l2e) : 0.f) + sa;
          lb = (mb > -INFINITY ? lb * ex2_approx((mb - nb) * l2e) : 0.f) + sb;
          ma = na;
          mb = nb;
        }
        if (cp == 0) {
          red[qc * kGM + 16 * sp + ra] = make_float2(ma, la);
          red[qc * kGM + 16 * sp + ra + 8] = make_float2(mb, lb);
        }
        named_bar_sync(2, 32 * kEpi);
        float La = 0.f, Lb = 0.f;
        Ma = Mb = -INFINITY;
        for (int k = 0; k < 4; ++k) {
          const float2 qa = red[k * kGM + 16 * sp + ra], qb = red[k * kGM + 16 * sp + ra + 8];
          if (qa.x > -INFINITY) {
            const float nm = fmaxf(Ma, qa.x);
            La = La * exp2f((Ma - nm) * l2e) + qa.y * exp2f((qa.x - nm) * l2e);
            Ma = nm;
          }
          if (qb.x > -INFINITY) {
            const float nm = fmaxf(Mb, qb.x);
            Lb = Lb * exp2f((Mb - nm) * l2e) + qb.y * exp2f((qb.x - nm) * l2e);
            Mb = nm;
          }
        }
        inva = 1.f / La;
        invb = 1.f / Lb;
      }
      // (softmax: pass 2 over the recomputed chunks)
      for (int ci = 0; ci < p.n_chunks; ++ci) {
        const int c = ci + rot < p.n_chunks ? ci + rot : ci + rot - p.n_chunks;
        mbar_wait(&d_full[db], dph);
        if (e == 0 && ci == 0) strace(p, 5 + 8 * min(g, 6));
        tc_fence_after();
        const int col0 = c * kNc + 32 * qc;
        uint32_t v[16];
        tmem_ld_16x256b_x4(tbase + lane_t + p.dcol0 + (uint32_t)(db * kNc + 32 * qc), v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[db]);
        if (++db == p.nd) { db = 0; dph ^= 1; }
        if (col0 >= p.r_dim || !live) continue;
        if (kTimingSwitches && p.dbg >= 3) continue;
        float o[16];
        if (p.softmax) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            o[4 * i] = ex2_approx((__uint_as_float(v[4 * i]) - Ma) * l2e) * inva;
            o[4 * i + 1] = ex2_approx((__uint_as_float(v[4 * i + 1]) - Ma) * l2e) * inva;
            o[4 * i + 2] = ex2_approx((__uint_as_float(v[4 * i + 2]) - Mb) * l2e) * invb;
            o[4 * i + 3] = ex2_approx((__uint_as_float(v[4 * i + 3]) - Mb) * l2e) * invb;
          }
        } else if (p.bias && p.bslot < 0) {
          constexpr float bsc = (YDT == DT_BF16 && ACT == DT_ACT_SIGMOID) ? 0.5f : 1.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int col = col0 + 8 * i + 2 * cp;
            const float b0 = col < p.r_dim ? bsc * __ldg(p.bias + col) : 0.f;
            const float b1 = col + 1 < p.r_dim ? bsc * __ldg(p.bias + col + 1) : 0.f;
            o[4 * i] = act_out<YDT, ACT>(__uint_as_float(v[4 * i]) + b0, p.arg);
            o[4 * i + 1] = act_out<YDT, ACT>(__uint_as_float(v[4 * i + 1]) + b1, p.arg);
            o[4 * i + 2] = act_out<YDT, ACT>(__uint_as_float(v[4 * i + 2]) + b0, p.arg);
            o[4 * i + 3] = act_out<YDT, ACT>(__uint_as_float(v[4 * i + 3]) + b1, p.arg);
          }
        } else {  // bias folded into the tf32 contraction (or absent)
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]), p.arg);
        }
        if (kTimingSwitches && p.dbg >= 2) {
          if (o[0] == 1234.5f) strace(p, 63);
          continue;
        }
        // the staging box's previous store (nstage stores ago) has read it
        const uint32_t out_s = out_s0 + (uint32_t)sb * (16u * RB);
        if (++sb == p.nstage) sb = 0;
        if (lane == 0) {
          if (p.nstage == 4) bulk_wait_group_read<3>();
          else if (p.nstage == 2) bulk_wait_group_read<1>();
          else bulk_wait_group_read<0>();
        }
        __syncwarp();
        stage_16x32<E>(out_s, lane, o);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(kTimingSwitches && p.dbg >= 1)) {
          tma_store_2d(&tm_y, smem + (out_s - s0), col0, (int32_t)row0);
          bulk_commit_group();
        }
      }
      if (e == 0) strace(p, 6 + 8 * min(g, 6));
    }
    if (lane == 0) bulk_wait_group<0>();  // staging read + y written before exit
    if (e == 0) strace(p, 62);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

using SlabFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, SlabParams);

template <int YDT>
SlabFn pick_act(int act) {
  switch (act) {
    case DT_ACT_RELU: return k_tc_rows_slab<YDT, DT_ACT_RELU>;
    case DT_ACT_SIGMOID: return k_tc_rows_slab<YDT, DT_ACT_SIGMOID>;
    case DT_ACT_TANH: return k_tc_rows_slab<YDT, DT_ACT_TANH>;
    case DT_ACT_CLIPPED_RELU: return k_tc_rows_slab<YDT, DT_ACT_CLIPPED_RELU>;
    default: return k_tc_rows_slab<YDT, DT_ACT_IDENTITY>;
  }
}

int slab_nsm() {
  static int nsm = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return nsm;
}

}  // namespace

// Geometries the slab kernel takes among those tc_rows_ok accepts: s = 2, 4 or 8 (a unit of
// 128 x' rows holds 64 / 32 / 16 whole batch rows, a group of 64 whole units), batch * s within
// the tensor map's 32-bit coordinates.
bool tc_slab_ok(const Geo &g, int64_t batch) {
  if (g.s < 2 || g.s > 8 || (g.s & (g.s - 1)) != 0) return false;  // units of 16 / 32 / 64 rows
  if (batch * g.s >= (int64_t)1 << 31) return false;
  return true;
}

int tc_slab_forward(const Geo &g, int64_t batch, const void *x, const void *wf16, const void *xf2p,
                    const float *bias, int bslot, int act, float act_arg, int softmax, void *y,
                    int y_dtype, cudaStream_t st) {
  SlabParams p{};
  p.batch = batch;
  p.r_dim = (int)g.r_dim;
  p.s = (int)g.s;
  p.ls = 0;
  while ((1 << p.ls) < p.s) ++p.ls;
  p.nkb = (int)(g.n / 64);
  p.rank = (int)g.rank;
  p.np = (int)((2 * g.rank + 15) / 16 * 16);
  p.rp = (int)((g.rank + 3) / 4 * 4);
  p.k2 = (int)((g.s * p.rp + 7) / 8 * 8);
  p.n_chunks = (int)((g.r_dim + kNc - 1) / kNc);
  p.ur = 128 / p.s;
  p.bias = bias;
  p.bslot = bslot;
  p.arg = act_arg;
  p.softmax = softmax;
  p.dbg = DT_DBG_ENV("DEEPTHIN_DBG_SLAB");
  // slab: the batch split evenly over the SMs, rounded up to whole units and to the 16-row
  // store box (DEEPTHIN_SLAB_CTAS: A/B runs with fewer CTAs)
  static const int want_ctas = getenv("DEEPTHIN_SLAB_CTAS") ? atoi(getenv("DEEPTHIN_SLAB_CTAS")) : 0;
  const int nsm = want_ctas > 0 ? std::min(want_ctas, slab_nsm()) : slab_nsm();
  const int gran = std::max(p.ur, 16);
  const int64_t per = (batch + nsm - 1) / nsm;
  p.slab = (int)((per + gran - 1) / gran * gran);
  const int ncta = (int)((batch + p.slab - 1) / p.slab);
  // TMEM: P ring of kPS units in columns [0, kPS * np), nd D buffers of 128 columns at the top
  p.nd = std::min(3, (512 - (kPS * p.np + 127) / 128 * 128) / kNc);
  p.dcol0 = 512u - (uint32_t)p.nd * kNc;
  // shared memory: A2 x 2 | wf | XF2p ring | output staging | softmax partials | x ring | barriers
  const int E = y_dtype == DT_BF16 ? 2 : 4;
  const uint32_t wf_bytes = (uint32_t)(p.nkb * p.np * 128);
  static const int want_bs = getenv("DEEPTHIN_SLAB_BS") ? atoi(getenv("DEEPTHIN_SLAB_BS")) : 0;
  p.bs = want_bs > 0 ? std::max(2, std::min(want_bs, kBSMax)) : 3;
  p.off_a2 = 0;
  p.off_wf = 2 * kA2Bytes;
  p.off_b = (p.off_wf + wf_bytes + 1023) & ~1023u;
  p.off_out = p.off_b + (uint32_t)p.bs * kBBytes;
  static const int want_stg = getenv("DEEPTHIN_SLAB_STG") ? atoi(getenv("DEEPTHIN_SLAB_STG")) : 2;
  p.nstage = want_stg >= 4 ? 4 : want_stg >= 2 ? 2 : 1;
  p.off_red = p.off_out + (uint32_t)(kEpi * p.nstage) * 16u * 32u * (uint32_t)E;
  p.off_x = p.off_red + (softmax ? 2u * 4u * kGM * 8u : 0u);
  p.off_x = (p.off_x + 1023) & ~1023u;
  constexpr uint32_t kSmemMax = 227 * 1024, kTail = 512 + 1024;
  static const int want_xs = getenv("DEEPTHIN_SLAB_XS") ? atoi(getenv("DEEPTHIN_SLAB_XS")) : kXSMax;
  if (kSmemMax - kTail < p.off_x + 2 * kXBytes) {
    set_error("row-slab kernel: operands do not fit shared memory");
    return DT_E_UNSUPPORTED;
  }
  p.xs = (int)std::min<uint32_t>((uint32_t)std::max(2, std::min(want_xs, kXSMax)),
                                 (kSmemMax - kTail - p.off_x) / kXBytes);
  p.off_bar = p.off_x + (uint32_t)p.xs * kXBytes;
  const uint32_t smem_bytes = p.off_bar + kTail;

  CUtensorMap tm_x, tm_wf, tm_xf2, tm_y;
  // x viewed (batch * s) x n: every 128 x' rows are 128 / s batch rows with all their segments
  if (int rc = encode_tensor_map_2d(&tm_x, DT_BF16, const_cast<void *>(x), (uint64_t)g.n,
                                    (uint64_t)(batch * g.s), (uint64_t)g.n * 2, 64, 128, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_wf, DT_BF16, const_cast<void *>(wf16), (uint64_t)g.n,
                                    (uint64_t)(2 * g.rank), (uint64_t)g.n * 2, 64, (uint32_t)p.np, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_xf2, DT_F32, const_cast<void *>(xf2p), (uint64_t)p.k2,
                                    (uint64_t)g.r_dim, (uint64_t)p.k2 * 4, 32, kNc, true))
    return rc;
  const int sw = y_dtype == DT_BF16 ? (int)CU_TENSOR_MAP_SWIZZLE_64B : (int)CU_TENSOR_MAP_SWIZZLE_128B;
  if (int rc = encode_tensor_map_2d_sw(&tm_y, y_dtype, y, (uint64_t)g.r_dim, (uint64_t)batch,
                                       (uint64_t)g.r_dim * E, 32, 16, sw))
    return rc;
  SlabFn fn = y_dtype == DT_BF16 ? pick_act<DT_BF16>(act) : pick_act<DT_F32>(act);
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ncta);
  cfg.blockDim = dim3(kSlabThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_ROWS_TRACE") != 0;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&p.trace, (size_t)ncta * kTr * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(p.trace, 0, (size_t)ncta * kTr * 8, st));
  }
  cudaEvent_t ev_b = nullptr, ev_a = nullptr;  // dt_profile_kernel_events
  profile_next(&ev_b, &ev_a, DT_PROF_ROWS);
  if (ev_b) DT_CUDA_CHECK(cudaEventRecord(ev_b, st));
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm_x, tm_wf, tm_xf2, tm_y, p));
  if (ev_a) DT_CUDA_CHECK(cudaEventRecord(ev_a, st));
  if (tracing) {  // every CTA's stamps, raw, to DEEPTHIN_ROWS_TRACE_FILE (scripts/rows_trace.py)
    std::vector<unsigned long long> h((size_t)ncta * kTr);
    DT_CUDA_CHECK(cudaMemcpyAsync(h.data(), p.trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFree(p.trace);
    const char *fname = getenv("DEEPTHIN_ROWS_TRACE_FILE");
    if (FILE *f = fopen(fname ? fname : "rows_trace.bin", "wb")) {
      const int hdr[6] = {ncta, kTr, 1, p.slab, p.n_chunks, p.s};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  return check_launch("tc_rows_slab");
}

}  // namespace dt
