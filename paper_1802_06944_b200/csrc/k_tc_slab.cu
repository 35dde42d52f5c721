// Row-slab tensor-core forward for reuse geometries (n_f | q, s = q / n_f in {2, 4, 8}): the
// factored DeepThin layer in ONE persistent kernel without clusters. Every CTA owns a contiguous
// slab of batch rows (batch / #SMs, rounded to the phase-A unit), reads those rows of x once and
// writes those rows of y once: all SMs stream, no P exchange between CTAs, no tail round.
// OPT-IN (DEEPTHIN_ROWS_SLAB=1): on config 3 it measures 30.5 us per hidden layer against
// 28.2 us for the clustered row-tile kernel (k_tc_rows.cu) — its transposed epilogue costs more
// instructions per output than the exchange it removes. Bit-identical outputs
// (test_slab_kernel_bits_equal_cluster_kernel). Its traces are where this round's two
// library-wide findings came from: the cost of bounded mbarrier wait loops (sm100_ptx.cuh
// mbar_wait) and of issuing tcgen05 / TMA instructions from inside `if (lane == 0)` (below).
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
//   phase B:  TRANSPOSED, output columns on the UMMA M axis (= TMEM lanes), batch rows on N:
//             D^T[j, b] = sum_kk XF2p[j, kk] A2[b, kk]   (kind::tf32, bias in a K pad slot)
//             per group of up to 64 batch rows (N = 64) and chunk of 128 output columns, XF2p
//             chunks streamed from L2. With the columns on the lanes every lane and every
//             thread is live whatever the group's row count, so slabs split into small groups
//             and a group's stores overlap the next group's loads. (Rows on the lanes —
//             measured — need 128-row groups to keep lanes, TMEM reads and MUFU busy: one group
//             per slab, all loads before all stores; 64-row groups read through the 16-lane
//             tcgen05.ld shape halve the TMEM read efficiency.)
//   epilogue: D^T (TMEM; thread = output column, registers = 2 x 16 batch rows) -> activation
//             -> bf16/fp32 -> transposed (lane-pair shuffle + byte permute) into a swizzled
//             32 x 32 staging box -> TMA store. The row softmax is not fused here (per-row
//             statistics would cross lanes): softmax layers stay on the clustered kernel.
//
// Warp roles (768 threads, one CTA per SM):
//   warp 0      TMA producer of x' k-blocks (128 x' rows x 64 bf16, SW128)
//   warp 2      TMEM allocator + tcgen05.mma issuer of phase A (P ring of 8 units)
//   warps 1, 3  phase-B issuers, one per team (team t = chunks t, t + 2, ... of every group):
//               XF2p chunk loads (3 slots, 3 chunks ahead: an L2 -> shared chunk load takes
//               ~1 us) and the chunk's MMAs nd - 1 chunks ahead into the team's D ring; one
//               named barrier per chunk joins the issuer and the team's eight epilogue warps
//   warps 4-7   P re-lay (one per TMEM lane quarter)
//   warps 8-23  epilogue, 8 warps per team: quarter (warp % 4) = 32 of a chunk's 128 output
//               columns, ((warp - 8) / 4) % 2 = 32 of the group's 64 rows
// All producer / issuer loops run warp-convergent with the asynchronous instructions predicated
// on lane 0 (see the comment at their head).
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

constexpr int kGM = 64;            // batch rows per phase-B group (UMMA N = TMEM columns per D buffer)
constexpr int kNc = 128;           // output columns per D chunk (UMMA M of phase B = TMEM lanes)
constexpr int kTeams = 2;          // independent phase-B pipelines (issuer + 8 epilogue warps each)
constexpr int kNDMax = 3;          // D buffers in TMEM per team (kGM columns each): 3 when the P ring
                                   // leaves room (np = 16), else 2
constexpr int kXSMax = 8;          // x ring depth cap
constexpr int kBSMax = 4;          // XF2p chunk ring depth cap (per team)
constexpr uint32_t kBS = 3;        // XF2p slots per team
constexpr int kPS = 8;             // P ring: phase-A units in TMEM
constexpr int kPW = 4;             // re-lay warps
constexpr int kEpi = 16;           // epilogue warps
constexpr int kSlabThreads = 32 * (4 + kPW + kEpi);
constexpr uint32_t kXBytes = 128 * 128;   // 128 x' rows x 64 bf16
constexpr uint32_t kBBytes = kNc * 128;   // 128 columns x 32 fp32
constexpr uint32_t kA2Bytes = kGM * 128;  // 64 rows x 32 fp32
constexpr int kTr = 64;                   // trace slots per CTA

struct SlabParams {
  int64_t batch;
  int r_dim, s, ls, nkb, np, rank, rp, k2, n_chunks;
  int ur;       // batch rows per phase-A unit (128 / s)
  int slab;     // batch rows per CTA (a multiple of max(ur, 16))
  int xs, bs, nd;
  int nstage;   // output staging boxes per epilogue warp (TMA stores in flight)
  int dbg;      // timing build only (DEEPTHIN_DBG_SLAB): >= 1 no TMA store, >= 2 no staging, >= 3
                // no activation, >= 4 no TMEM reads (wrong outputs: a ladder for the traces)
  uint32_t dcol0;
  int bslot;    // K slot carrying the bias (A2 = 1 there), -1: the epilogue adds it
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

// this warp's 16 x 32 outputs, o[i] = row i of output column `lane`, transposed into its
// swizzled row-major staging box (the TMA SW64 / SW128 pattern: 16-byte chunk ch of row r at
// ch ^ (r >> 1 & 3) / ch ^ (r & 7)). bf16: lane pairs exchange so that the even lane holds
// columns (lane, lane + 1) of the even rows and the odd lane those of the odd rows — one 4-byte
// store per two outputs, 128 contiguous bytes per instruction (rows r, r + 1 are adjacent).
template <int E>
__device__ __forceinline__ void stage_t16x32(uint32_t out_s, int lane, const float *o) {
  if constexpr (E == 2) {
    // rows (i, i + 1) of this column packed, exchanged with the partner lane, and one byte
    // permute picks (own, partner) low halves (even lane: row i) or (partner, own) high halves
    // (odd lane: row i + 1): four instructions per two outputs
    const int odd = lane & 1;
    const uint32_t sel = odd ? 0x3276u : 0x5410u;
    const uint32_t base = out_s + (uint32_t)odd * 64u + (uint32_t)((lane >> 1) & 3) * 4u;
    const int ch = lane >> 3;  // 16-byte chunk of columns lane - odd, lane - odd + 1
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      const uint32_t w = pack_bf16(o[i], o[i + 1]);
      const uint32_t pw = __shfl_xor_sync(0xffffffffu, w, 1);
      // even row of the pair is i; this lane stores row i + odd (same swizzle)
      st_shared_b32(base + (uint32_t)i * 64u + ((uint32_t)(ch ^ ((i >> 1) & 3)) << 4),
                    __byte_perm(w, pw, sel));
    }
  } else {
    const uint32_t base = out_s + (uint32_t)(lane & 3) * 4u;
    const int ch = lane >> 2;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      st_shared_b32(base + (uint32_t)i * 128u + ((uint32_t)(ch ^ (i & 7)) << 4), __float_as_uint(o[i]));
  }
}

template <int YDT, int ACT>
__global__ void __launch_bounds__(kSlabThreads, 1)
    k_tc_rows_slab(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_wf,
                   const __grid_constant__ CUtensorMap tm_xf2, const __grid_constant__ CUtensorMap tm_y,
                   const __grid_constant__ CUtensorMap tm_y16, const SlabParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *x_full = bars, *x_empty = x_full + kXSMax;
  uint64_t *b_full = x_empty + kXSMax, *b_empty = b_full + kTeams * kBSMax;  // [team][slot]
  uint64_t *d_full = b_empty + kTeams * kBSMax, *d_empty = d_full + kTeams * kNDMax;  // [team][buffer]
  uint64_t *p_full = d_empty + kTeams * kNDMax, *p_free = p_full + kPS;
  uint64_t *a2_full = p_free + kPS, *a2_free = a2_full + 2;
  uint64_t *wf_full = a2_free + 2;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(wf_full + 1);
  // (the shuffle makes the warp index — and everything derived from it — provably warp-uniform
  // for the compiler: uniform registers instead of per-lane waterfalls in the issuer loops)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;

  // this CTA's slab: rows [row_begin, row_begin + rows), in groups of kGM, each group in units
  // of ur rows
  const int64_t row_begin = (int64_t)blockIdx.x * p.slab;
  const int rows = (int)min((int64_t)p.slab, p.batch - row_begin);
  const int n_groups = (rows + kGM - 1) / kGM;
  // Every CTA streams every XF2p chunk: CTA i starts at chunk i mod n_chunks, so that at any
  // time the CTAs read n_chunks different chunks (all of them on the same 128 lines at once
  // would hit the same few L2 slices).
  const int rot = (int)(blockIdx.x % (unsigned)p.n_chunks);

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.xs; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < kTeams * kBSMax; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < kTeams * kNDMax; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], kEpi / kTeams);
    }
    for (int i = 0; i < kPS; ++i) { mbar_init(&p_full[i], 1); mbar_init(&p_free[i], 1); }
    for (int i = 0; i < 2; ++i) {  // a2_free: one arrive per team that has chunks
      mbar_init(&a2_full[i], 1);
      mbar_init(&a2_free[i], (uint32_t)min(kTeams, p.n_chunks));
    }
    mbar_init(wf_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wf);
    tma_prefetch_desc(&tm_xf2);
    tma_prefetch_desc(&tm_y);
    tma_prefetch_desc(&tm_y16);
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

  // The role warps below run their loops on ALL 32 lanes (uniform control flow, uniform ring
  // positions and addresses) and only predicate the asynchronous instructions on lane 0. With
  // the whole loop inside `if (lane == 0)` the compiler treats every operand as lane-varying and
  // wraps each UTCHMMA / UTMALDG in a waterfall (ELECT, five R2UR.BROADCAST, branch): ~200
  // clocks per MMA issue, which paced phase A at 1.7 us per 64 KB of x and phase B at ~0.7 us
  // per chunk. (Warp index and TMEM base pass through a shuffle for the same reason.)
  const bool l0 = lane == 0;
  const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
  if (warp == 0) {
    // ---------------- x' producer ----------------
    const uint32_t s0 = smem_u32(smem);
    if (l0) {
      mbar_arrive_expect_tx(wf_full, (uint32_t)(p.nkb * p.np * 128));
      for (int kb = 0; kb < p.nkb; ++kb)
        tma_load_2d_s(s0 + p.off_wf + (uint32_t)(kb * p.np * 128), &tm_wf, smem_u32(wf_full), kb * 64, 0);
    }
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
          if (l0) {
            mbar_arrive_expect_tx(&x_full[st], kXBytes);
            tma_load_2d_s(s0 + p.off_x + (uint32_t)st * kXBytes, &tm_x, smem_u32(&x_full[st]), kb * 64, r0);
          }
          if (++st == p.xs) { st = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ---------------- phase-A MMA issuer: P[unit] = x' unit . [wf_hi | wf_lo]^T ----------------
    const uint32_t s0 = smem_u32(smem);
    const uint32_t idA = idesc_f32acc(128, (uint32_t)p.np, 1);
    const uint64_t descX0 = smem_desc(s0 + p.off_x, 16, 1024, SL_SW128);
    const uint64_t descW0 = smem_desc(s0 + p.off_wf, 16, 1024, SL_SW128);
    const uint32_t wstep = (uint32_t)(p.np * 128) >> 4;  // descriptor units per wf k-block
    mbar_wait(wf_full, 0);
    int xs = 0;
    uint32_t xph = 0, slot = 0, sph = 0;
    bool first = true;
    for (int g = 0; g < n_groups; ++g) {
      const int g_rows = min(kGM, rows - g * kGM);
      const int g_units = (g_rows + p.ur - 1) / p.ur;
      for (int u = 0; u < g_units; ++u) {
        mbar_wait(&p_free[slot], sph ^ 1u);  // the re-lay warps read the unit 8 units back
        tc_fence_after();
        const uint32_t d = tb + slot * (uint32_t)p.np;
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&x_full[xs], xph);
          if (first && l0) strace(p, 2);
          first = false;
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
        if (l0) {
          mma_commit(&p_full[slot]);
          if (u == g_units - 1) strace(p, 3 + 8 * min(g, 6));
        }
        if (++slot == kPS) { slot = 0; sph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- phase-B issuers (warp 1: team 0, warp 3: team 1) ----------------
    // Team t = chunks t, t + 2, ... of every group, eight epilogue warps and this warp's lane 0,
    // which loads the team's XF2p chunks (kBS slots, kBS chunks ahead: an L2 -> shared chunk
    // load takes ~1 us here) and issues the chunk's MMAs nd - 1 chunks ahead into the team's D
    // ring. One named barrier per chunk joins the nine warps: past it, every epilogue warp has
    // read the D buffer the issuer overwrites next. The loop is single-thread scalar code and
    // was the bottleneck (~2400 clocks per chunk with descriptors rebuilt per MMA, divisions for
    // ring positions, ...): everything is kept incremental and the descriptors precomputed.
    const int t = warp >> 1;
    const int cpt = t < p.n_chunks ? (p.n_chunks - t + kTeams - 1) / kTeams : 0;  // chunks per group
    const int K = n_groups * cpt;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t nd = (uint32_t)p.nd;
    const int ahead = p.nd - 1;
    const int nk = p.k2 / 8;
    const uint32_t idB = idesc_f32acc(kNc, kGM, 2);
    uint64_t *bf = b_full + t * kBSMax, *df = d_full + t * kNDMax;
    const uint64_t descA0 = smem_desc(s0 + p.off_b + (uint32_t)(t * kBS) * kBBytes, 16, 1024, SL_SW128);
    const uint64_t descB0 = smem_desc(s0 + p.off_a2, 16, 1024, SL_SW128);
    const uint32_t dbase = tb + p.dcol0 + (uint32_t)t * nd * (uint32_t)kGM;
    const uint32_t b_s0 = s0 + p.off_b + (uint32_t)(t * kBS) * kBBytes;
    // ring positions: loads (l_*), MMA issue (i_*), completion waits (w_*)
    uint32_t l_slot = 0, i_slot = 0, i_par = 0, i_d = 0, w_d = 0, w_par = 0;
    int l_j = 0, l_n = 0;
    auto load_next = [&]() {  // XF2p chunk of the next element of the team's sequence
      const int ci = t + l_j * kTeams;
      const int c = ci + rot < p.n_chunks ? ci + rot : ci + rot - p.n_chunks;
      if (l0) {
        mbar_arrive_expect_tx(&bf[l_slot], kBBytes);
        tma_load_2d_s(b_s0 + l_slot * kBBytes, &tm_xf2, smem_u32(&bf[l_slot]), 0, c * kNc);
      }
      if (++l_slot == kBS) l_slot = 0;
      if (++l_j == cpt) l_j = 0;
      ++l_n;
    };
    auto issue_next = [&](uint64_t descB) {  // the MMAs of the next element
      mbar_wait(&bf[i_slot], i_par);
      tc_fence_after();
      const uint32_t d = dbase + i_d * (uint32_t)kGM;
      const uint64_t a = descA0 + (uint64_t)(i_slot * (kBBytes >> 4));
      if (l0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (kk < nk) mma_tf32_ss(d, a + (uint64_t)(2 * kk), descB + (uint64_t)(2 * kk), idB, kk != 0);
        mma_commit(&df[i_d]);
      }
      if (++i_slot == kBS) { i_slot = 0; i_par ^= 1; }
      if (++i_d == nd) i_d = 0;
    };
    for (int i = 0; i < (int)kBS && i < K; ++i) load_next();
    for (int g = 0; g < n_groups; ++g) {
      const int gb = g & 1;
      const uint64_t descB = descB0 + (uint64_t)(gb * (int)(kA2Bytes >> 4));
      for (int j = 0; j < cpt; ++j) {
        named_bar_sync(2 + t, 32 * (kEpi / kTeams + 1));
        if (j == 0) {  // first chunk of a group: its A2 has to be complete (nothing issued early)
          mbar_wait(&a2_full[gb], (uint32_t)(g >> 1) & 1u);
          if (t == 0 && l0) strace(p, 4 + 8 * min(g, 6));
          for (int a = 0; a < ahead && a < cpt; ++a) issue_next(descB);
        }
        if (j + ahead < cpt) issue_next(descB);
        // the MMAs of this chunk are complete: its XF2p slot is free (the element kBS further
        // goes there) and, after the group's last chunk, so is A2[gb] as far as this team goes
        mbar_wait(&df[w_d], w_par);
        if (++w_d == nd) { w_d = 0; w_par ^= 1; }
        if (l_n < K) load_next();
        if (j + 1 == cpt && l0) mbar_arrive(&a2_free[gb]);
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
    if (lrow < kGM)
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
        const int row = u * p.ur + bq;  // batch row within the group = A2 row
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
    // ---------------- epilogue: 2 teams of 8 warps ----------------
    // Team t reads the chunks its issuer multiplies (t, t + 2, ... of every group). Within a team
    // quarter sp = output columns 32 sp .. 32 sp + 31 of the chunk (lane = column), h = rows
    // 32 h .. 32 h + 31 of the group (32 TMEM columns).
    const int sp = warp & 3;
    const int e = warp - 4 - kPW;      // 0..15
    const int t = e >> 3, h = (e >> 2) & 1;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    constexpr int E = YDT == DT_BF16 ? 2 : 4;
    constexpr int RB = 32 * E;         // bytes per row of this warp's 32 columns (64 or 128)
    const uint32_t out_s0 = s0 + p.off_out + (uint32_t)(e * p.nstage) * (32u * RB);
    int sb = 0;
    const int64_t slab_end = row_begin + rows;
    const int cpt = t < p.n_chunks ? (p.n_chunks - t + kTeams - 1) / kTeams : 0;  // chunks per group
    uint64_t *df = d_full + t * kNDMax;
    const uint32_t dcol = p.dcol0 + (uint32_t)(t * p.nd * kGM + 32 * h);
    uint32_t w_d = 0, w_par = 0;  // position in the team's D ring
    for (int g = 0; g < n_groups; ++g) {
      const int64_t row0 = row_begin + g * kGM + 32 * h;
      // rows of this warp inside the slab: all 32 (or the batch end, which TMA clips) -> the
      // 32-row box; 16 -> the 16-row box (slabs end on multiples of 16); none -> nothing to do
      const int live = (int)min((int64_t)32, slab_end - row0);
      const CUtensorMap *tmy = (live >= 32 || slab_end == p.batch) ? &tm_y : &tm_y16;
      for (int j = 0; j < cpt; ++j) {
        // (joins the team's issuer: every warp has read the D buffer it overwrites next)
        named_bar_sync(2 + t, 32 * (kEpi / kTeams + 1));
        const int ci = t + j * kTeams;
        const int c = ci + rot < p.n_chunks ? ci + rot : ci + rot - p.n_chunks;
        mbar_wait(&df[w_d], w_par);
        const uint32_t dc = dcol + w_d * (uint32_t)kGM;
        if (++w_d == (uint32_t)p.nd) { w_d = 0; w_par ^= 1; }
        if (e == 0 && j == 0) strace(p, 5 + 8 * min(g, 6));
        tc_fence_after();
        const int col0 = c * kNc + 32 * sp;
        const bool work = live > 0 && col0 < p.r_dim && !(kTimingSwitches && p.dbg >= 4);
        // the staging box's previous store (nstage stores ago) has read it
        const uint32_t out_s = out_s0 + (uint32_t)sb * (32u * RB);
        if (work) {
          if (++sb == p.nstage) sb = 0;
          if (lane == 0) {
            if (p.nstage == 2) bulk_wait_group_read<1>();
            else bulk_wait_group_read<0>();
          }
          __syncwarp();
        }
        // two halves of 16 rows (16 live registers each)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t v[16];
          if (work) {
            tmem_ld_32x32b_x16(tbase + lane_t + dc + (uint32_t)(16 * hh), v);
            tmem_ld_wait();
          }
          if (hh == 1) tc_fence_before();  // both halves read (the team barrier follows)
          if (!work || (kTimingSwitches && p.dbg >= 3)) continue;
          float o[16];
          if (p.bias && p.bslot < 0) {
            constexpr float bsc = (YDT == DT_BF16 && ACT == DT_ACT_SIGMOID) ? 0.5f : 1.f;
            const float bj = col0 + lane < p.r_dim ? bsc * __ldg(p.bias + col0 + lane) : 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]) + bj, p.arg);
          } else {  // bias folded into the tf32 contraction (or absent)
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = act_out<YDT, ACT>(__uint_as_float(v[i]), p.arg);
          }
          if (kTimingSwitches && p.dbg >= 2) {
            if (o[0] == 1234.5f) strace(p, 63);
            continue;
          }
          stage_t16x32<E>(out_s + (uint32_t)hh * (16u * RB), lane, o);
        }
        if (!work || (kTimingSwitches && p.dbg >= 2)) continue;
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(kTimingSwitches && p.dbg >= 1)) {
          tma_store_2d(tmy, smem + (out_s - s0), col0, (int32_t)row0);
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

using SlabFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, SlabParams);

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
bool tc_slab_ok(const Geo &g, int64_t batch, int softmax) {
  if (softmax) return false;  // per-row statistics would cross lanes: the clustered kernel fuses it
  if (g.s < 2 || g.s > 8 || (g.s & (g.s - 1)) != 0) return false;  // units of 16 / 32 / 64 rows
  if (batch * g.s >= (int64_t)1 << 31) return false;
  return true;
}

int tc_slab_forward(const Geo &g, int64_t batch, const void *x, const void *wf16, const void *xf2p,
                    const float *bias, int bslot, int act, float act_arg, void *y, int y_dtype,
                    cudaStream_t st) {
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
  p.dbg = DT_DBG_ENV("DEEPTHIN_DBG_SLAB");
  // slab: the batch split evenly over the SMs, rounded up to whole units and to the 16-row
  // store box (DEEPTHIN_SLAB_CTAS: A/B runs with fewer CTAs)
  static const int want_ctas = getenv("DEEPTHIN_SLAB_CTAS") ? atoi(getenv("DEEPTHIN_SLAB_CTAS")) : 0;
  const int nsm = want_ctas > 0 ? std::min(want_ctas, slab_nsm()) : slab_nsm();
  const int gran = std::max(p.ur, 16);
  const int64_t per = (batch + nsm - 1) / nsm;
  p.slab = (int)((per + gran - 1) / gran * gran);
  const int ncta = (int)((batch + p.slab - 1) / p.slab);
  // TMEM: P ring of kPS units in columns [0, kPS * np), kTeams x kND D buffers of kGM columns
  // at the top
  p.nd = std::min(kNDMax, (512 - (kPS * p.np + 63) / 64 * 64) / (kTeams * kGM));
  p.dcol0 = 512u - (uint32_t)(kTeams * p.nd * kGM);
  // shared memory: A2 x 2 | wf | XF2p ring | output staging | softmax partials | x ring | barriers
  const int E = y_dtype == DT_BF16 ? 2 : 4;
  const uint32_t wf_bytes = (uint32_t)(p.nkb * p.np * 128);
  static const int want_bs = getenv("DEEPTHIN_SLAB_BS") ? atoi(getenv("DEEPTHIN_SLAB_BS")) : 0;
  (void)want_bs;
  p.bs = 3;  // per team (kBS in the kernel)
  p.off_a2 = 0;
  p.off_wf = 2 * kA2Bytes;
  p.off_b = (p.off_wf + wf_bytes + 1023) & ~1023u;
  p.off_out = p.off_b + (uint32_t)(kTeams * p.bs) * kBBytes;
  static const int want_stg = getenv("DEEPTHIN_SLAB_STG") ? atoi(getenv("DEEPTHIN_SLAB_STG")) : 1;
  p.nstage = want_stg >= 2 ? 2 : 1;
  p.off_red = p.off_out + (uint32_t)(kEpi * p.nstage) * 32u * 32u * (uint32_t)E;
  p.off_x = (p.off_red + 1023) & ~1023u;
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

  CUtensorMap tm_x, tm_wf, tm_xf2, tm_y, tm_y16;
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
                                       (uint64_t)g.r_dim * E, 32, 32, sw))
    return rc;
  if (int rc = encode_tensor_map_2d_sw(&tm_y16, y_dtype, y, (uint64_t)g.r_dim, (uint64_t)batch,
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
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm_x, tm_wf, tm_xf2, tm_y, tm_y16, p));
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
