// General-path (straddling rows) forward on tcgen05 tensor cores — kernel K3.
//
// y = act(x @ W + bias) where W (q x r_dim) is the DeepThin re-layout of
// I = xf @ wf (factor.py:87-93) and, on this path, n does not divide q, so an
// output column's q weights start at phase (j*q) mod n and straddle aux rows
// (kernel.py:1-16). W is never materialised in HBM:
//
//  * Persistent CTAs walk a contiguous range of (column block, batch tile) work
//    items, column-block-major, so a CTA regenerates its W block once and reuses
//    it (resident in shared memory) for every batch tile it owns.
//  * Regeneration runs on the tensor cores: the aux rows a_lo..a_hi covering
//    the block's flat range [j0*q, (j0+128)*q) are small MMAs
//    I_rows(128 x n) = xf_rows(128 x rank) @ wf(rank x n) into TMEM; the
//    epilogue warps read them back (tcgen05.ld), round to bf16 and scatter every
//    element f -> (jj, i) = divmod(f - j0*q, q) into the 128B-swizzled K-major
//    operand layout (16-byte stores when q and n are multiples of 8). The
//    discarded tail (f >= q*r_dim) is never produced.
//  * Main loop: D[j, b] (TMEM, fp32) += W_blk[j, :] . x[b, :] with
//    tcgen05.mma.cta_group::1.kind::f16, M = 128 output columns, N = 128 batch
//    rows, A = the resident W block, B = TMA-staged x tiles (S-stage mbarrier
//    ring). Accumulators are double-buffered in TMEM so the epilogue of tile t
//    overlaps the MMAs of tile t+1.
//  * Epilogue: lanes are output columns, TMEM columns are batch rows, so each
//    warp store instruction writes 32 consecutive outputs of one batch row
//    (coalesced), fused with bias + activation. Output dtype and activation are
//    template parameters: the epilogue stays a few hundred instructions (the
//    runtime-switch version thrashed the instruction cache).
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-5 regeneration + epilogue.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "act.cuh"
#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

// warps 0-1: TMA producer / MMA issuer; warps 2..: regeneration + epilogue, kParts warps per
// TMEM lane quarter (warp % 4) splitting the columns between them (part = (warp - 2) / 4).
#ifndef DT_TC_PARTS
#define DT_TC_PARTS 3
#endif
constexpr int kParts = DT_TC_PARTS;
constexpr int kEpiThreads = 128 * kParts;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int BMW = 128;   // W rows (output columns) per block == UMMA M
constexpr int BNB = 256;   // batch rows per tile == UMMA N (N=256 runs the MMA at ~88% of
                           // peak; N=128 is shared-memory-bound at ~60%, measured)
constexpr int KATOM = 64;  // bf16 elements per 128-byte swizzle row
constexpr uint32_t kXStage = BNB * 128;   // bytes per x stage (128 rows x 64 bf16)
constexpr uint32_t kWKBlk = BMW * 128;    // bytes per W k-block
constexpr uint32_t kTmemCols = 512;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kTraceSlots = 48;

struct TcParams {
  int64_t batch;
  int q, r_dim, rank, m, n, ldy;
  int KB, S, S_ded, RK, Nc, n_chunks, n_cb, n_bt, items, per_cta;
  int a_res;  // passes of xf rows resident at once (all, or 1 = streamed per pass)
  int csize;  // cluster size: CTAs sharing (multicasting) each x tile
  const uint8_t *xf_pk, *wf_pk;  // regeneration operands, pre-packed (dt_pack_factors)
  const float *bias;
  void *y;
  float arg;
  uint32_t off_w, off_x, off_ar, off_br, off_bar;
  uint32_t w_sbo;  // W block 8-row-group stride (no-swizzle K-major layout)
  unsigned long long *trace;  // DEEPTHIN_TC_TRACE: per-CTA globaltimer stamps, else null
  int dbg_serial;             // DEEPTHIN_REGEN_SERIAL: no regen MMA / read-back overlap
  int dbg_regen;              // DEEPTHIN_DBG_REGEN: 1 skip scatter, 2 skip TMEM loads (timing only)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// slots: 0 start, 1 setup done, 2..5 regen begin/end (x2), 6..13 epilogue tile done,
// 14..21 MMA tile committed, 22 producer done, 23 end
__device__ __forceinline__ void trace(const TcParams &p, int slot) {
  if (p.trace && slot < kTraceSlots) p.trace[(size_t)blockIdx.x * kTraceSlots + slot] = gtimer();
}

// Byte offset of W-block element (jj, i) in the no-swizzle K-major core-matrix layout:
// [8-row group][K core of 8][8 rows x 16 B]. The regeneration scatter writes 16-byte units
// whose rows advance ~q/n per thread; here the bank group of a unit is jj & 7, so a warp's
// stores spread over all banks (the 128B-swizzled layout put every lane on one chunk when
// n = 0 mod 64, a 32-way conflict). sbo = 8-row-group stride = (K extent / 8) * 128.
__device__ __forceinline__ uint32_t w_off(uint32_t jj, uint32_t i, uint32_t sbo) {
  return (jj >> 3) * sbo + (i >> 3) * 128u + (jj & 7u) * 16u + (i & 7u) * 2u;
}

// No-swizzle K-major ("interleave") layout of the small regeneration operands:
// 8-row x 16-byte core matrices, K-adjacent cores 128 B apart (LBO), 8-row groups SBO apart.
__device__ __forceinline__ uint32_t core_off(uint32_t row, uint32_t k, uint32_t sbo) {
  return (row >> 3) * sbo + (k >> 3) * 128u + (row & 7u) * 16u + (k & 7u) * 2u;
}

__device__ __forceinline__ void sts_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t *>(&h);
}

// Scatter one tcgen05.ld group (32 consecutive aux columns of one aux row) into the W block.
// (jj, i) = position of the group's first element (jj may be negative: skipped).
// MODE 2: q, n multiples of 8 (16-byte stores); 1: both even (4-byte); 0: scalar.
template <int MODE>
__device__ __forceinline__ void scatter32(const uint32_t (&v)[32], uint32_t w_s, uint32_t sbo,
                                          int jj, int i, int q, int cvalid, int jrows) {
  // predicated stores (no per-store branch / reconvergence barrier)
  if constexpr (MODE == 2) {
    // 16-byte units (i % 8 == 0). A 32-element group wraps to the next W row at most once
    // (q >= 32): units t < wrap stay in row jj (128 B apart in the core-matrix layout), the
    // rest continue in row jj+1 from column i + 8*t - q. Every unit's address and predicate
    // is computed independently (no serial chain across units).
    const int wrap = (q - i + 7) >> 3;  // units left in row jj
    const uint32_t a0 = w_s + w_off((uint32_t)jj, (uint32_t)i, sbo);
    const uint32_t a1 = w_s + w_off((uint32_t)(jj + 1), (uint32_t)(i + 8 * wrap - q), sbo);
    const bool r0 = (uint32_t)jj < (uint32_t)jrows, r1 = (uint32_t)(jj + 1) < (uint32_t)jrows;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool second = t >= wrap;
      const uint32_t addr = second ? a1 + 128u * (uint32_t)(t - wrap) : a0 + 128u * (uint32_t)t;
      const uint32_t ok = (8 * t < cvalid) & (second ? r1 : r0);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"
          "@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}" ::"r"(addr),
          "r"(pack_bf16(v[8 * t], v[8 * t + 1])), "r"(pack_bf16(v[8 * t + 2], v[8 * t + 3])),
          "r"(pack_bf16(v[8 * t + 4], v[8 * t + 5])), "r"(pack_bf16(v[8 * t + 6], v[8 * t + 7])),
          "r"(ok));
    }
  } else if constexpr (MODE == 1) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const uint32_t ok = (2 * t < cvalid) & (jj >= 0) & (jj < jrows);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t}" ::"r"(
              w_s + w_off(jj, i, sbo)),
          "r"(pack_bf16(v[2 * t], v[2 * t + 1])), "r"(ok));
      i += 2;
      const bool wrap = i >= q;
      i -= wrap ? q : 0;
      jj += wrap;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      if (t < cvalid && jj >= 0 && jj < jrows) {
        __nv_bfloat16 h = __float2bfloat16_rn(__uint_as_float(v[t]));
        sts_u16(w_s + w_off(jj, i, sbo), *reinterpret_cast<uint16_t *>(&h));
      }
      if (++i == q) { i = 0; ++jj; }
    }
  }
}

struct BlockRows {
  int jrows, a_lo, a_hi, a_first, n_pass;
  int64_t fbeg;
};
__device__ __forceinline__ BlockRows block_rows(const TcParams &p, int cb) {
  BlockRows b;
  const int j0 = cb * BMW;
  b.jrows = min(BMW, p.r_dim - j0);
  b.fbeg = (int64_t)j0 * p.q;
  const int64_t fend = (int64_t)(j0 + b.jrows) * p.q;
  b.a_lo = (int)(b.fbeg / p.n);
  b.a_hi = (int)min((int64_t)p.m - 1, (fend - 1) / p.n);
  b.a_first = b.a_lo & ~7;
  b.n_pass = (b.a_hi - b.a_first) / 128 + 1;
  return b;
}

// Request the regeneration operands of column block cb (one thread): every pass of xf rows
// as one contiguous bulk copy; all of wf^T only when not already resident.
__device__ __forceinline__ void regen_request(const TcParams &p, int cb, uint8_t *ar, uint8_t *br,
                                              uint64_t *obar, bool need_b) {
  const BlockRows b = block_rows(p, cb);
  const uint32_t sbo = (uint32_t)(p.RK / 8) * 128u;
  const uint32_t a_bytes = (uint32_t)min(b.n_pass, p.a_res) * 16u * sbo;
  const uint32_t b_bytes = (uint32_t)p.n_chunks * (uint32_t)(p.Nc / 8) * sbo;
  mbar_arrive_expect_tx(obar, a_bytes + (need_b ? b_bytes : 0u));
  bulk_load(ar, p.xf_pk + (size_t)(b.a_first >> 3) * sbo, a_bytes, obar);
  if (need_b) bulk_load(br, p.wf_pk, b_bytes, obar);
}

// How many regeneration steps TMEM holds at once: the first `slots` steps' MMAs are issued
// up front and each read-back frees a slot for step s + slots, so MMA -> commit -> mbarrier
// round trips overlap the read-backs. A streamed pass of xf rows (very skinny n) must first
// replace the resident one: one step at a time.
__device__ __forceinline__ int regen_slots(const TcParams &p, const BlockRows &b) {
  const int n_steps = b.n_pass * p.n_chunks;
  const bool stream = p.a_res < b.n_pass;
  return (stream || p.dbg_serial) ? 1 : min(4, min(n_steps, 512 / p.Nc));
}

// Regeneration MMAs of column block cb — issued by the MMA warp's elected lane (issuing
// tcgen05 from a lane of a divergent epilogue warp measured ~5x slower).
// Steps (pass, chunk): pass = 128 aux rows from a_first + 128*pass, chunk = Nc aux columns.
// rbar[slot]: MMA -> read-back ("step done"); rfree[slot]: read-back -> MMA ("slot free").
__device__ void regen_issue(const TcParams &p, int cb, uint8_t *ar, uint8_t *br, uint64_t *rbar,
                            uint64_t *rfree, uint32_t &fphase, uint64_t *obar, uint32_t &ophase,
                            uint32_t tbase) {
  const BlockRows b = block_rows(p, cb);
  const int n_steps = b.n_pass * p.n_chunks;
  const bool stream = p.a_res < b.n_pass;
  const int slots = regen_slots(p, b);
  const uint32_t sbo = (uint32_t)(p.RK / 8) * 128u;
  const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)p.Nc);
  const uint32_t ar_s = smem_u32(ar), br_s = smem_u32(br);
  mbar_wait(obar, ophase);  // operands landed (regen_request)
  ophase ^= 1;
  trace(p, 24);
  for (int s = 0; s < n_steps; ++s) {
    const int slot = s % slots, pass = s / p.n_chunks, chunk = s % p.n_chunks;
    if (s >= slots) {  // the read-back of step s - slots has released this TMEM slot
      mbar_wait(&rfree[slot], (fphase >> slot) & 1u);
      fphase ^= 1u << slot;
    }
    if (stream && s > 0 && chunk == 0) {  // replace the resident pass of xf rows
      const uint32_t bytes = 16u * sbo;
      mbar_arrive_expect_tx(obar, bytes);
      bulk_load(ar, p.xf_pk + (size_t)((b.a_first >> 3) + 16 * pass) * sbo, bytes, obar);
      mbar_wait(obar, ophase);
      ophase ^= 1;
    }
    tc_fence_after();
    const uint32_t a_s = ar_s + (stream ? 0u : (uint32_t)pass * 16u * sbo);
    const uint32_t b_s = br_s + (uint32_t)chunk * (uint32_t)(p.Nc / 8) * sbo;
    for (int kk = 0; kk < p.RK / 16; ++kk) {
      uint64_t ad = smem_desc(a_s + kk * 256u, 128u, sbo, SL_NONE);
      uint64_t bd = smem_desc(b_s + kk * 256u, 128u, sbo, SL_NONE);
      mma_bf16_ss(tbase + (uint32_t)(slot * p.Nc), ad, bd, idesc, kk > 0);
    }
    mma_commit(&rbar[slot]);  // one mbarrier per TMEM slot: one phase in flight each
    if (s == slots - 1) trace(p, 39);
  }
}

// Read back the regeneration steps of column block cb (the epilogue warps): TMEM -> bf16 ->
// scatter of every element f -> (jj, i) = divmod(f - j0*q, q) into the W block.
template <int MODE>
__device__ void regen_readout(const TcParams &p, int cb, uint32_t w_s, uint64_t *rbar,
                              uint32_t &rphase, uint64_t *rfree, uint32_t tbase, int et, int wq,
                              int part, int lane) {
  const BlockRows b = block_rows(p, cb);
  const int q = p.q, n = p.n;
  const int n_steps = b.n_pass * p.n_chunks;
  const int slots = regen_slots(p, b);
  const int L = 32 * wq + lane;  // TMEM lane (= aux row offset within the pass)
  for (int s = 0; s < n_steps; ++s) {
    const int pass = s / p.n_chunks, chunk = s % p.n_chunks;
    const int c0 = chunk * p.Nc;
    const int cols = min(p.Nc, n - c0);
    const int slot = s % slots;
    mbar_wait(&rbar[slot], (rphase >> slot) & 1u);  // one parity bit per slot
    rphase ^= 1u << slot;
    if (et == 0 && s < 4) trace(p, 25 + s);
    tc_fence_after();
    const int a = b.a_first + 128 * pass + L;
    const int a_warp = b.a_first + 128 * pass + 32 * wq;  // this warp's rows: a_warp .. +31
    const uint32_t tcol = tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(slot * p.Nc);
    if (a_warp <= b.a_hi && a_warp + 31 >= b.a_lo && (!kTimingSwitches || p.dbg_regen != 3)) {  // skip all-invalid warps
      // this warp's column groups: part, part + kParts, ... (32 columns each)
      const int f0 = (int)((int64_t)a * n + c0 + 32 * part - b.fbeg);
      int jj = f0 >= 0 ? f0 / q : -((-f0 + q - 1) / q);
      int i = f0 - jj * q;
      const bool row_ok = a >= b.a_lo && a <= b.a_hi;
      int g = 0;
      for (int col0 = 32 * part; col0 < p.Nc; col0 += 32 * kParts, ++g) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tcol + (uint32_t)col0, v);
        tmem_ld_wait();
        if (p.trace && et == 0 && s == 0 && g < 3) {
          asm volatile("" ::"r"(v[0] ^ v[31]));
          trace(p, 32 + 2 * g);
        }
        if (row_ok && col0 < cols && (!kTimingSwitches || p.dbg_regen != 1))
          scatter32<MODE>(v, w_s, p.w_sbo, jj, i, q, cols - col0, b.jrows);
        if (p.trace && et == 0 && s == 0 && g < 3) trace(p, 33 + 2 * g);
        i += 32 * kParts;
        while (i >= q) { i -= q; ++jj; }
      }
    }
    if (et == 0 && s == 0) trace(p, 31);
    tc_fence_before();
    named_bar_sync(1, kEpiThreads);
    if (et == 0 && s == 0) trace(p, 38);
    if (et == 0 && s + slots < n_steps) mbar_arrive(&rfree[slot]);  // slot reusable
  }
}

template <int YDT, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_general(const __grid_constant__ CUtensorMap tm_x, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *wblk = smem + p.off_w;
  uint8_t *xst = smem + p.off_x;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *bready = tempty + 2, *rbar = bready + 1, *rfree = rbar + 4, *obar = rfree + 4;
  uint64_t *cregen = obar + 1;  // "every CTA of my cluster finished regenerating this block"
  uint32_t *tslot = reinterpret_cast<uint32_t *>(cregen + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // Clusters of p.csize CTAs own consecutive column blocks and walk the same batch tiles:
  // each CTA TMA-loads 1/csize of every x stage and multicasts it to the whole cluster.
  // Work items are cluster items (column-block group, batch tile).
  const uint32_t crank = p.csize > 1 ? cluster_ctarank() : 0u;
  const uint16_t cmask = (uint16_t)((1u << p.csize) - 1u);
  const int cid = blockIdx.x / p.csize;
  const int item_beg = cid * p.per_cta;
  const int item_end = min(p.items, item_beg + p.per_cta);
  auto cb_of = [&](int it) { return (it / p.n_bt) * p.csize + (int)crank; };

  if (threadIdx.x == 0) {
    trace(p, 0);
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], p.csize); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], kEpiThreads); }
    mbar_init(bready, 1);
    for (int s = 0; s < 4; ++s) { mbar_init(&rbar[s], 1); mbar_init(&rfree[s], 1); }
    mbar_init(obar, 1);
    mbar_init(cregen, p.csize);
    fence_mbar_init();
    // the first block's regeneration operands start streaming in before anything else
    if (item_beg < item_end)
      regen_request(p, cb_of(item_beg), smem + p.off_ar, smem + p.off_br, obar, true);
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_x);
  if (warp == 1) tmem_alloc(tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  if (p.csize > 1) cluster_sync();  // peers' barriers are initialised before any multicast
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) trace(p, 1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0, cur_cb = -1, n_cbs = 0;
      uint32_t phase = 0;
      bool regen_pending = false;
      const uint32_t slice_rows = BNB / p.csize, slice_bytes = kXStage / p.csize;
      for (int it = item_beg; it < item_end; ++it) {
        const int32_t b0 = (it % p.n_bt) * BNB;
        if (cb_of(it) != cur_cb) {
          cur_cb = cb_of(it);
          ++n_cbs;
          regen_pending = true;
        }
        for (int kb = 0; kb < p.KB; ++kb) {
          if ((stage >= p.S_ded || (kTimingSwitches && p.dbg_regen == 4)) && regen_pending) {
            // this stage aliases the regeneration operands of every CTA it multicasts into
            mbar_wait_sleepy(cregen, (uint32_t)(n_cbs - 1) & 1u);
            regen_pending = false;
          }
          mbar_wait(&empty[stage], phase ^ 1);  // consumed by every CTA of the cluster
          mbar_arrive_expect_tx(&full[stage], kXStage);
          if (p.csize == 1)
            tma_load_2d(xst + (size_t)stage * kXStage, &tm_x, &full[stage], kb * KATOM, b0);
          else
            tma_load_2d_mc(xst + (size_t)stage * kXStage + crank * slice_bytes, &tm_x,
                           &full[stage], kb * KATOM, b0 + (int32_t)(crank * slice_rows), cmask);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
      }
      trace(p, 22);
    }
    __syncwarp();  // lanes 1-31 wait here: no lane reaches the aligned barriers below early
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(BMW, BNB);
      const uint32_t w_s = smem_u32(wblk), x_s = smem_u32(xst);
      int stage = 0, acc = 0, cur_cb = -1;
      uint32_t phase = 0, acc_phase = 0, bphase = 0, fphase = 0, ophase = 0;
      uint8_t *ar = smem + p.off_ar, *br = smem + p.off_br;
      for (int it = item_beg; it < item_end; ++it) {
        const int cb = cb_of(it);
        if (cb != cur_cb) {
          // regenerate this block's W on the tensor cores, then wait for the read-back
          regen_issue(p, cb, ar, br, rbar, rfree, fphase, obar, ophase, tbase);
          mbar_wait_sleepy(bready, bphase);
          bphase ^= 1;
          cur_cb = cb;
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * BNB);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < KATOM / 16; ++k) {
            // A = W block, no-swizzle K-major: a 16-wide K step is 2 core columns (256 B)
            uint64_t ad = smem_desc(w_s + (uint32_t)(kb * 4 + k) * 256u, 128u, p.w_sbo, SL_NONE);
            uint64_t bd = smem_desc(x_s + stage * kXStage + k * 32, 16, 1024, SL_SW128);
            mma_bf16_ss(d, ad, bd, idesc, (kb | k) != 0);
          }
          if (p.csize == 1)
            mma_commit(&empty[stage]);
          else  // every producer of the cluster multicasts into this stage
            mma_commit_mc(&empty[stage], cmask);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        trace(p, 14 + min(7, it - item_beg));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();  // reconverge before tcgen05.dealloc (.sync.aligned)
  } else {
    // ---------------- regeneration + epilogue (warps 2-9) ----------------
    const int et = threadIdx.x - 64;
    const int wq = warp & 3;
    const int part = (warp - 2) / 4;
    const int jl = 32 * wq + lane;  // output column within the block (TMEM lane)
    const uint32_t w_s = smem_u32(wblk);
    uint8_t *ar = smem + p.off_ar, *br = smem + p.off_br;
    // one-time zeroing of the W K-padding [q, KB*64)
    if (et < BMW)
      for (int i = p.q; i < p.KB * KATOM; ++i) sts_u16(w_s + w_off(et, i, p.w_sbo), 0);
    const int mode = (p.q % 8 == 0 && p.n % 8 == 0 && p.q >= 32)
                         ? 2
                         : ((p.q % 2 == 0 && p.n % 2 == 0) ? 1 : 0);
    uint32_t rphase = 0, acc_phase = 0;
    int acc = 0, cur_cb = -1, n_regen = 0;
    float bias_j = 0.f;
    for (int it = item_beg; it < item_end; ++it) {
      const int cb = cb_of(it), bt = it % p.n_bt;
      const int j = cb * BMW + jl;
      if (cb != cur_cb) {
        if (et == 0 && n_regen < 2) trace(p, 2 + 2 * n_regen);
        if (et == 0 && n_regen > 0) regen_request(p, cb, ar, br, obar, false);
        if (mode == 2)
          regen_readout<2>(p, cb, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        else if (mode == 1)
          regen_readout<1>(p, cb, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        else
          regen_readout<0>(p, cb, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          mbar_arrive(bready);
          // every cluster CTA may now multicast x into the stages aliasing my operands
          if (p.csize == 1)
            mbar_arrive(cregen);
          else
            for (int r = 0; r < p.csize; ++r) mbar_arrive_remote(cregen, (uint32_t)r);
        }
        if (et == 0 && n_regen < 2) trace(p, 3 + 2 * n_regen);
        ++n_regen;
        cur_cb = cb;
        bias_j = (p.bias && j < p.r_dim) ? p.bias[j] : 0.f;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int b0 = bt * BNB;
      const bool jok = j < p.r_dim;
      const int nrows = (int)min((int64_t)BNB, p.batch - b0);
      using OutT = typename std::conditional<YDT == DT_BF16, __nv_bfloat16, float>::type;
      for (int c32 = part; c32 < BNB / 32; c32 += kParts) {  // this part's 32-row groups
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(acc * BNB + c32 * 32), v);
        tmem_ld_wait();
        if (jok) {
          OutT *yp = reinterpret_cast<OutT *>(p.y) + (int64_t)(b0 + 32 * c32) * p.ldy + j;
          const int rmax = nrows - c32 * 32;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            if (r < rmax) {
              const float o = act_fast<ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
              if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
            }
            yp += p.ldy;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (et == 0) trace(p, 6 + min(7, it - item_beg));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace(p, 23);
  if (p.csize > 1) cluster_sync();  // no CTA leaves while peers may still signal / multicast to it
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kTmemCols);
  }
}

// =============================================================================================
// CTA-pair variant (tcgen05 cta_group::2). A cluster of two CTAs owns two consecutive column
// blocks (M = 256 output columns, 128 per CTA, each CTA regenerating its own W block) and
// 256-row batch tiles of which each CTA TMA-loads 128 rows: per-SM x traffic halves and the
// 2-SM MMA (256 x 256 x 16) runs at the full per-SM rate, with seven 16 KB x stages in flight.
// The leader (cluster rank 0) issues every MMA — regeneration (M = 256: both CTAs' aux rows
// against wf^T, whose N rows are split across the pair) and main loop — and its commits
// multicast to both CTAs. Peer -> leader signals (operands landed, slot free, block
// regenerated, accumulator drained) are remote mbarrier arrivals.
// =============================================================================================

__device__ __forceinline__ void arrive_leader(uint64_t *bar, uint32_t crank) {
  if (crank == 0)
    mbar_arrive(bar);
  else
    mbar_arrive_remote(bar, 0);
}

// Steps of a pair regeneration: the pair's passes cover both CTAs' aux rows.
__device__ __forceinline__ int pair_passes(const TcParams &p, int cb_leader) {
  return max(block_rows(p, cb_leader).n_pass, block_rows(p, cb_leader + 1).n_pass);
}

// Own xf rows (every pass) and this CTA's half of each wf^T chunk (rows [crank*Nc/2, +Nc/2)).
__device__ __forceinline__ void regen_request_pair(const TcParams &p, int cb, uint32_t crank,
                                                   uint8_t *ar, uint8_t *br, uint64_t *obar,
                                                   bool need_b) {
  const BlockRows b = block_rows(p, cb);
  const uint32_t sbo = (uint32_t)(p.RK / 8) * 128u;
  const uint32_t a_bytes = (uint32_t)pair_passes(p, cb - (int)crank) * 16u * sbo;
  const uint32_t half = (uint32_t)(p.Nc / 16) * sbo;  // Nc/2 rows of one chunk
  mbar_arrive_expect_tx(obar, a_bytes + (need_b ? half * (uint32_t)p.n_chunks : 0u));
  bulk_load(ar, p.xf_pk + (size_t)(b.a_first >> 3) * sbo, a_bytes, obar);
  if (need_b)
    for (int ch = 0; ch < p.n_chunks; ++ch)
      bulk_load(br + ch * half, p.wf_pk + (size_t)ch * 2u * half + crank * half, half, obar);
}

template <int MODE>
__device__ void regen_readout_pair(const TcParams &p, int cb, uint32_t crank, uint32_t w_s,
                                   uint64_t *rbar, uint32_t &rphase, uint64_t *rfree,
                                   uint32_t tbase, int et, int wq, int part, int lane) {
  const BlockRows b = block_rows(p, cb);
  const int q = p.q, n = p.n;
  const int n_steps = pair_passes(p, cb - (int)crank) * p.n_chunks;
  const int slots = min(4, min(n_steps, 512 / p.Nc));
  const int L = 32 * wq + lane;
  for (int s = 0; s < n_steps; ++s) {
    const int pass = s / p.n_chunks, chunk = s % p.n_chunks;
    const int c0 = chunk * p.Nc;
    const int cols = min(p.Nc, n - c0);
    const int slot = s % slots;
    mbar_wait(&rbar[slot], (rphase >> slot) & 1u);
    rphase ^= 1u << slot;
    if (et == 0 && s < 4) trace(p, 25 + s);
    tc_fence_after();
    const int a = b.a_first + 128 * pass + L;
    const int a_warp = b.a_first + 128 * pass + 32 * wq;
    const uint32_t tcol = tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(slot * p.Nc);
    if (a_warp <= b.a_hi && a_warp + 31 >= b.a_lo) {
      const int f0 = (int)((int64_t)a * n + c0 + 32 * part - b.fbeg);
      int jj = f0 >= 0 ? f0 / q : -((-f0 + q - 1) / q);
      int i = f0 - jj * q;
      const bool row_ok = a >= b.a_lo && a <= b.a_hi;
      for (int col0 = 32 * part; col0 < p.Nc; col0 += 32 * kParts) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tcol + (uint32_t)col0, v);
        tmem_ld_wait();
        if (row_ok && col0 < cols)
          scatter32<MODE>(v, w_s, p.w_sbo, jj, i, q, cols - col0, b.jrows);
        i += 32 * kParts;
        while (i >= q) { i -= q; ++jj; }
      }
    }
    tc_fence_before();
    named_bar_sync(1, kEpiThreads);
    if (et == 0 && s + slots < n_steps) arrive_leader(&rfree[slot], crank);
  }
}

template <int YDT, int ACT>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_general_pair(const __grid_constant__ CUtensorMap tm_x, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *wblk = smem + p.off_w;
  uint8_t *xst = smem + p.off_x;
  uint8_t *ar = smem + p.off_ar, *br = smem + p.off_br;
  const uint32_t stage_bytes = kXStage / 2;  // this CTA's 128 of the tile's 256 rows
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *bready = tempty + 2, *rbar = bready + 1, *rfree = rbar + 4, *obar = rfree + 4;
  uint64_t *cregen = obar + 1, *pobar = cregen + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(pobar + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int item_beg = (blockIdx.x / 2) * p.per_cta;
  const int item_end = min(p.items, item_beg + p.per_cta);
  auto cb_of = [&](int it) { return (it / p.n_bt) * 2 + (int)crank; };

  if (threadIdx.x == 0) {
    trace(p, 0);
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 2); }
    mbar_init(bready, 2);
    for (int s = 0; s < 4; ++s) { mbar_init(&rbar[s], 1); mbar_init(&rfree[s], 2); }
    mbar_init(obar, 1);
    mbar_init(cregen, 1);
    mbar_init(pobar, 1);
    fence_mbar_init();
    if (item_beg < item_end) regen_request_pair(p, cb_of(item_beg), crank, ar, br, obar, true);
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_x);
  if (warp == 1) tmem_alloc_pair(tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) trace(p, 1);

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs: own 128 rows of each tile) ----------------
    if (lane == 0) {
      int stage = 0, cur_cb = -1, n_cbs = 0;
      uint32_t phase = 0;
      bool regen_pending = false;
      for (int it = item_beg; it < item_end; ++it) {
        const int32_t b0 = (it % p.n_bt) * BNB + (int32_t)crank * (BNB / 2);
        if (cb_of(it) != cur_cb) {
          cur_cb = cb_of(it);
          ++n_cbs;
          regen_pending = true;
        }
        for (int kb = 0; kb < p.KB; ++kb) {
          if (stage >= p.S_ded && regen_pending) {  // stage aliases my regeneration operands
            mbar_wait_sleepy(cregen, (uint32_t)(n_cbs - 1) & 1u);
            regen_pending = false;
          }
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);  // both halves
          tma_load_2d_pair(xst + (size_t)stage * stage_bytes, &tm_x, &full[stage], kb * KATOM, b0);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
      }
      trace(p, 22);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer (leader only; 2-SM MMAs) ----------------
      const uint32_t idesc = idesc_bf16_f32(2 * BMW, BNB);
      const uint32_t idesc_r = idesc_bf16_f32(2 * BMW, (uint32_t)p.Nc);
      const uint32_t w_s = smem_u32(wblk), x_s = smem_u32(xst);
      const uint32_t ar_s = smem_u32(ar), br_s = smem_u32(br);
      const uint32_t sbo = (uint32_t)(p.RK / 8) * 128u;
      const uint32_t half = (uint32_t)(p.Nc / 16) * sbo;
      int stage = 0, acc = 0, cur_cb = -1;
      uint32_t phase = 0, acc_phase = 0, bphase = 0, fphase = 0, ophase = 0;
      for (int it = item_beg; it < item_end; ++it) {
        const int cb = cb_of(it);
        if (cb != cur_cb) {
          // regeneration of both W blocks: own operands + the peer's (relayed)
          mbar_wait(obar, ophase);
          mbar_wait(pobar, ophase);
          ophase ^= 1;
          trace(p, 24);
          const int n_steps = pair_passes(p, cb) * p.n_chunks;
          const int slots = min(4, min(n_steps, 512 / p.Nc));
          for (int s = 0; s < n_steps; ++s) {
            const int slot = s % slots, pass = s / p.n_chunks, chunk = s % p.n_chunks;
            if (s >= slots) {
              mbar_wait(&rfree[slot], (fphase >> slot) & 1u);
              fphase ^= 1u << slot;
            }
            tc_fence_after();
            for (int kk = 0; kk < p.RK / 16; ++kk) {
              uint64_t ad = smem_desc(ar_s + (uint32_t)pass * 16u * sbo + kk * 256u, 128u, sbo, SL_NONE);
              uint64_t bd = smem_desc(br_s + (uint32_t)chunk * half + kk * 256u, 128u, sbo, SL_NONE);
              mma_bf16_ss_pair(tbase + (uint32_t)(slot * p.Nc), ad, bd, idesc_r, kk > 0);
            }
            mma_commit_pair(&rbar[slot]);
          }
          mbar_wait_sleepy(bready, bphase);  // both CTAs' W blocks are in shared memory
          bphase ^= 1;
          cur_cb = cb;
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(acc * BNB);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < KATOM / 16; ++k) {
            uint64_t ad = smem_desc(w_s + (uint32_t)(kb * 4 + k) * 256u, 128u, p.w_sbo, SL_NONE);
            uint64_t bd = smem_desc(x_s + stage * stage_bytes + k * 32, 16, 1024, SL_SW128);
            mma_bf16_ss_pair(d, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit_pair(&empty[stage]);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc]);
        trace(p, 14 + min(7, it - item_beg));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    } else if (lane == 0) {
      // peer: relay "my regeneration operands landed" to the leader, once per block
      int cur_cb = -1;
      uint32_t ophase = 0;
      for (int it = item_beg; it < item_end; ++it) {
        if (cb_of(it) == cur_cb) continue;
        cur_cb = cb_of(it);
        mbar_wait_sleepy(obar, ophase);
        ophase ^= 1;
        mbar_arrive_remote(pobar, 0);
      }
    }
    __syncwarp();
  } else {
    // ---------------- regeneration read-back + epilogue (both CTAs) ----------------
    const int et = threadIdx.x - 64;
    const int wq = warp & 3;
    const int part = (warp - 2) / 4;
    const int jl = 32 * wq + lane;
    const uint32_t w_s = smem_u32(wblk);
    if (et < BMW)
      for (int i = p.q; i < p.KB * KATOM; ++i) sts_u16(w_s + w_off(et, i, p.w_sbo), 0);
    const int mode = (p.q % 8 == 0 && p.n % 8 == 0 && p.q >= 32)
                         ? 2
                         : ((p.q % 2 == 0 && p.n % 2 == 0) ? 1 : 0);
    uint32_t rphase = 0, acc_phase = 0;
    int acc = 0, cur_cb = -1, n_regen = 0;
    float bias_j = 0.f;
    for (int it = item_beg; it < item_end; ++it) {
      const int cb = cb_of(it), bt = it % p.n_bt;
      const int j = cb * BMW + jl;
      if (cb != cur_cb) {
        if (et == 0 && n_regen < 2) trace(p, 2 + 2 * n_regen);
        if (et == 0 && n_regen > 0) regen_request_pair(p, cb, crank, ar, br, obar, false);
        if (mode == 2)
          regen_readout_pair<2>(p, cb, crank, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        else if (mode == 1)
          regen_readout_pair<1>(p, cb, crank, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        else
          regen_readout_pair<0>(p, cb, crank, w_s, rbar, rphase, rfree, tbase, et, wq, part, lane);
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) {
          arrive_leader(bready, crank);  // the leader's MMAs read both W blocks
          mbar_arrive(cregen);           // my producer may fill the aliased stages
        }
        if (et == 0 && n_regen < 2) trace(p, 3 + 2 * n_regen);
        ++n_regen;
        cur_cb = cb;
        bias_j = (p.bias && j < p.r_dim) ? p.bias[j] : 0.f;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int b0 = bt * BNB;
      const bool jok = j < p.r_dim;
      const int nrows = (int)min((int64_t)BNB, p.batch - b0);
      using OutT = typename std::conditional<YDT == DT_BF16, __nv_bfloat16, float>::type;
      for (int c32 = part; c32 < BNB / 32; c32 += kParts) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(acc * BNB + c32 * 32), v);
        tmem_ld_wait();
        if (jok) {
          OutT *yp = reinterpret_cast<OutT *>(p.y) + (int64_t)(b0 + 32 * c32) * p.ldy + j;
          const int rmax = nrows - c32 * 32;
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            if (r < rmax) {
              const float o = act_fast<ACT>(__uint_as_float(v[r]) + bias_j, p.arg);
              if constexpr (YDT == DT_BF16) *yp = __float2bfloat16_rn(o); else *yp = o;
            }
            yp += p.ldy;
          }
        }
      }
      tc_fence_before();
      named_bar_sync(1, kEpiThreads);  // every TMEM read of this accumulator has completed
      if (et == 0) arrive_leader(&tempty[acc], crank);
      if (et == 0) trace(p, 6 + min(7, it - item_beg));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace(p, 23);
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, kTmemCols);
  }
}

// x (fp32 or bf16, row stride q) -> bf16 with row stride ldx (zero padded). One thread per 8
// output elements (one 16-byte store); two 16-byte fp32 loads when the source row is aligned.
__global__ void k_pack_x(int64_t batch, int64_t q, int64_t ldx, const void *x, int x_dtype,
                         __nv_bfloat16 *out) {
  const int64_t per_row = ldx / 8;  // ldx is a multiple of 8
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * per_row) return;
  const int64_t b = idx / per_row, i0 = (idx - b * per_row) * 8;
  float v[8];
  const bool vec = x_dtype == DT_F32 && i0 + 8 <= q && ((q & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (vec) {
    const float4 *src = reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(x) + b * q + i0);
    const float4 a = __ldg(src), c = __ldg(src + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t i = i0 + e;
      v[e] = i >= q ? 0.f
             : x_dtype == DT_BF16
                 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(x)[b * q + i])
                 : reinterpret_cast<const float *>(x)[b * q + i];
    }
  }
  uint32_t w[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    __nv_bfloat162 t = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
    w[h] = *reinterpret_cast<uint32_t *>(&t);
  }
  *reinterpret_cast<uint4 *>(out + b * ldx + i0) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Pack bf16 factors into the regeneration operands' core-matrix layout (zero padded):
//   xf_pk: rows 0 .. xrows-1 (xrows = round_up(m, 8) + 128) x RK,
//   wf_pk: wf^T, rows c = 0 .. n_chunks*Nc - 1 x RK.
__global__ void k_pack_general(int m, int n, int rank, int RK, int xrows, int wrows,
                               const __nv_bfloat16 *xf, const __nv_bfloat16 *wf, uint8_t *xf_pk,
                               uint8_t *wf_pk) {
  const uint32_t sbo = (uint32_t)(RK / 8) * 128u;
  const int64_t nx = (int64_t)xrows * RK, nw = (int64_t)wrows * RK;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < nx + nw;
       idx += (int64_t)gridDim.x * blockDim.x) {
    if (idx < nx) {
      const int row = (int)(idx / RK), k = (int)(idx % RK);
      const __nv_bfloat16 v = (row < m && k < rank) ? xf[(int64_t)row * rank + k] : __float2bfloat16(0.f);
      *reinterpret_cast<__nv_bfloat16 *>(xf_pk + core_off(row, k, sbo)) = v;
    } else {
      const int64_t e = idx - nx;
      const int c = (int)(e / RK), k = (int)(e % RK);
      const __nv_bfloat16 v = (c < n && k < rank) ? wf[(int64_t)k * n + c] : __float2bfloat16(0.f);
      *reinterpret_cast<__nv_bfloat16 *>(wf_pk + core_off(c, k, sbo)) = v;
    }
  }
}

// ---- host ------------------------------------------------------------------------------
typedef CUresult (*PFN_encode_tiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                     const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                     const cuuint32_t *, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion,
                                     CUtensorMapFloatOOBfill);

PFN_encode_tiled encode_fn() {
  static PFN_encode_tiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encode_tiled>(ptr);
  });
  return fn;
}

struct Layout {
  int KB, S, S_ded, RK, Nc, n_chunks, n_pass, a_res;
  uint32_t off_w, off_x, off_ar, off_br, off_bar, total;
};

// pair: the cta_group::2 kernel (16 KB x stages = this CTA's half of a 256-row tile; half of
// each wf^T chunk; all passes resident — no streamed fallback).
bool make_layout(const Geo &g, Layout *L, bool pair = false) {
  const uint32_t kStage = pair ? kXStage / 2 : kXStage;
  L->KB = (int)((g.q + KATOM - 1) / KATOM);
  L->RK = (int)((g.rank + 15) / 16 * 16);
  L->n_chunks = (int)((g.n + 255) / 256);
  L->Nc = (int)(((g.n + L->n_chunks - 1) / L->n_chunks + 31) / 32 * 32);
  // aux rows one W block touches (+ the 8-row alignment of the first pass)
  const int64_t span = (BMW * g.q + g.n - 1) / g.n + 1 + 7;
  L->n_pass = (int)((span + 127) / 128);
  if (L->RK > 64) return false;
  const uint32_t w = (uint32_t)L->KB * kWKBlk;
  const uint32_t fixed = w + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  // Preferred: all of a block's regeneration operands resident (every pass of xf rows, all
  // of wf). Fallback for very skinny n (many passes): one pass of xf rows, streamed.
  for (int a_res : {L->n_pass, 1}) {
    if (pair && a_res != L->n_pass) break;
    const uint32_t arb = (uint32_t)a_res * 128u * L->RK * 2;
    const uint32_t brb = (uint32_t)L->n_chunks * L->Nc * L->RK * 2 / (pair ? 2 : 1);
    // The regeneration operands are only live while a W block is regenerated, so they
    // alias the last x stages; the producer fills those stages only after that block's regen.
    int S = 0;
    for (int s = 8; s >= 2; --s)
      if (fixed + (uint32_t)s * kStage <= (uint32_t)kSmemBudget) { S = s; break; }
    if (S == 0) return false;
    const uint32_t xbytes = (uint32_t)S * kStage;
    const uint32_t ops = (arb + brb + 1023) / 1024 * 1024;
    L->off_w = 0;
    L->off_x = w;
    if (ops > xbytes) {  // operands larger than the stage area: place them after it
      if (fixed + xbytes + ops > (uint32_t)kSmemBudget) continue;
      L->off_ar = L->off_x + xbytes;
    } else {
      L->off_ar = L->off_x + xbytes - ops;
    }
    L->S = S;
    L->S_ded = (int)std::min<uint32_t>((uint32_t)S, (L->off_ar - L->off_x) / kStage);
    if (L->S_ded < 1) continue;
    L->a_res = a_res;
    L->off_br = L->off_ar + arb;
    L->off_bar = std::max(L->off_x + xbytes, L->off_br + brb);
    L->off_bar = (L->off_bar + 15) / 16 * 16;
    L->total = L->off_bar + 512 + 1024;
    if (L->total <= (uint32_t)kSmemBudget) return true;
  }
  return false;
}

typedef void (*KernelFn)(CUtensorMap, TcParams);

template <int YDT>
KernelFn pick_act(int act) {
  switch (act) {
    case DT_ACT_RELU: return k_tc_general<YDT, DT_ACT_RELU>;
    case DT_ACT_SIGMOID: return k_tc_general<YDT, DT_ACT_SIGMOID>;
    case DT_ACT_TANH: return k_tc_general<YDT, DT_ACT_TANH>;
    case DT_ACT_CLIPPED_RELU: return k_tc_general<YDT, DT_ACT_CLIPPED_RELU>;
    default: return k_tc_general<YDT, DT_ACT_IDENTITY>;
  }
}

template <int YDT>
KernelFn pick_act_pair(int act) {
  switch (act) {
    case DT_ACT_RELU: return k_tc_general_pair<YDT, DT_ACT_RELU>;
    case DT_ACT_SIGMOID: return k_tc_general_pair<YDT, DT_ACT_SIGMOID>;
    case DT_ACT_TANH: return k_tc_general_pair<YDT, DT_ACT_TANH>;
    case DT_ACT_CLIPPED_RELU: return k_tc_general_pair<YDT, DT_ACT_CLIPPED_RELU>;
    default: return k_tc_general_pair<YDT, DT_ACT_IDENTITY>;
  }
}

void print_trace(const std::vector<unsigned long long> &h, int grid, const TcParams &p) {
  unsigned long long t0 = ~0ull, t1 = 0;
  for (int c = 0; c < grid; ++c) {
    t0 = std::min(t0, h[(size_t)c * kTraceSlots]);
    // the last stamp of any role (slot 23 is taken right after a BAR.SYNC.DEFER_BLOCKING and
    // can precede the epilogue's final stores)
    for (int s = 0; s < kTraceSlots; ++s) t1 = std::max(t1, h[(size_t)c * kTraceSlots + s]);
  }
  fprintf(stderr, "[tc trace] grid %d per_cta %d S %d (dedicated %d) KB %d span %.2f us\n", grid,
          p.per_cta, p.S, p.S_ded, p.KB, (t1 - t0) / 1e3);
  for (int c = 0; c < grid; c += std::max(1, grid / 6)) {
    const unsigned long long *r = &h[(size_t)c * kTraceSlots];
    auto rel = [&](int s) { return r[s] ? (double)(r[s] - t0) / 1e3 : -1.0; };
    fprintf(stderr, "  cta %3d: start %.2f setup %.2f regen [%.2f..%.2f] epi", c, rel(0), rel(1),
            rel(2), rel(3));
    for (int k = 0; k < 8; ++k)
      if (r[6 + k]) fprintf(stderr, " %.2f", rel(6 + k));
    fprintf(stderr, " | mma");
    for (int k = 0; k < 8; ++k)
      if (r[14 + k]) fprintf(stderr, " %.2f", rel(14 + k));
    fprintf(stderr,
            " | prod %.2f end %.2f | regen ops %.2f steps %.2f %.2f %.2f %.2f | ld0 %.2f..%.2f "
            "step0 end %.2f\n",
            rel(22), rel(23), rel(24), rel(25), rel(26), rel(27), rel(28), rel(29), rel(30),
            rel(31));
    fprintf(stderr,
            "        step0 (thread 64): ld0 %.3f sc0 %.3f ld1 %.3f sc1 %.3f ld2 %.3f sc2 %.3f "
            "pre-bar %.3f post-bar %.3f | regen MMAs issued %.3f\n",
            rel(32), rel(33), rel(34), rel(35), rel(36), rel(37), rel(31), rel(38), rel(39));
  }
}

}  // namespace

static int check_layout(const Geo &g, Layout *L) {
  if (!make_layout(g, L)) {
    set_error("tcgen05 general path: q=" + std::to_string(g.q) + ", rank=" +
              std::to_string(g.rank) + " does not fit the resident-W-block kernel "
              "(needs ceil(q/64)*16 KB + stages <= 227 KB and rank <= 64)");
    return DT_E_UNSUPPORTED;
  }
  if (g.m * g.n > INT32_MAX || g.q * g.r_dim > INT32_MAX) {
    set_error("tcgen05 general path: m*n must fit in 32 bits");
    return DT_E_UNSUPPORTED;
  }
  return DT_OK;
}

static int packed_x_rows(const Geo &g, const Layout &L) {
  return (int)(((g.m + 7) / 8) * 8 + 128 * L.n_pass);
}
static size_t packed_x_bytes(const Geo &g, const Layout &L) {
  return (size_t)packed_x_rows(g, L) * L.RK * 2;
}

size_t tc_general_packed_bytes(const Geo &g) {
  Layout L;
  if (!make_layout(g, &L)) return 0;
  return (packed_x_bytes(g, L) + 255) / 256 * 256 + (size_t)L.n_chunks * L.Nc * L.RK * 2;
}

int tc_general_pack(const Geo &g, const uint16_t *xf_bf16, const uint16_t *wf_bf16, void *packed,
                    cudaStream_t st) {
  Layout L;
  if (int rc = check_layout(g, &L)) return rc;
  const int xrows = packed_x_rows(g, L);
  const int wrows = L.n_chunks * L.Nc;
  uint8_t *xpk = reinterpret_cast<uint8_t *>(packed);
  uint8_t *wpk = xpk + (packed_x_bytes(g, L) + 255) / 256 * 256;
  const int64_t tot = (int64_t)(xrows + wrows) * L.RK;
  const unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 4096);
  k_pack_general<<<blocks, 256, 0, st>>>((int)g.m, (int)g.n, (int)g.rank, L.RK, xrows, wrows,
                                         reinterpret_cast<const __nv_bfloat16 *>(xf_bf16),
                                         reinterpret_cast<const __nv_bfloat16 *>(wf_bf16), xpk, wpk);
  return check_launch("pack_general");
}

size_t tc_general_ws(const Geo &g, int64_t batch) {
  int64_t ldx = (g.q + 7) / 8 * 8;
  return (size_t)batch * ldx * 2 + 256 + tc_general_packed_bytes(g) + 256;
}

int tc_general_forward(const Geo &g, int64_t batch, const void *x, int x_dtype,
                       const uint16_t *xf_bf16, const uint16_t *wf_bf16, const void *packed,
                       const float *bias, int act, float act_arg, void *y, int y_dtype, char *ws,
                       size_t ws_bytes, cudaStream_t st) {
  Layout L;
  if (int rc = check_layout(g, &L)) return rc;
  if (batch == 0) return DT_OK;
  PFN_encode_tiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return DT_E_CUDA;
  }
  if (ws_bytes < tc_general_ws(g, batch) - (packed ? tc_general_packed_bytes(g) + 256 : 0)) {
    set_error("forward workspace too small: need " + std::to_string(tc_general_ws(g, batch)));
    return DT_E_ARG;
  }
  if (!packed) {  // pack the regeneration operands into the workspace tail for this call
    char *pk = ws + ((size_t)batch * ((g.q + 7) / 8 * 8) * 2 + 256 + 255) / 256 * 256;
    if (int rc = tc_general_pack(g, xf_bf16, wf_bf16, pk, st)) return rc;
    packed = pk;
  }
  // TMA needs a bf16 x whose row pitch is a multiple of 16 bytes.
  const void *xt = x;
  int64_t ldx = g.q;
  if (x_dtype != DT_BF16 || (g.q % 8) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
    ldx = (g.q + 7) / 8 * 8;
    int64_t tot = batch * ldx;
    k_pack_x<<<(unsigned)((tot / 8 + 255) / 256), 256, 0, st>>>(batch, g.q, ldx, x, x_dtype,
                                                                 reinterpret_cast<__nv_bfloat16 *>(ws));
    if (int rc = check_launch("pack_x")) return rc;
    xt = ws;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)g.q, (cuuint64_t)batch};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
  // Cluster size: consecutive column blocks share every x tile through TMA multicast, so L2
  // serves each x tile once per cluster instead of once per CTA (DEEPTHIN_TC_CLUSTER
  // overrides; needs n_cb % csize == 0).
  const int n_cb = (int)((g.r_dim + BMW - 1) / BMW);
  // Preferred: the CTA-pair (cta_group::2) kernel when column blocks pair up and every
  // regeneration pass fits (DEEPTHIN_TC_PAIR=0 disables).
  static const int want_pair = getenv("DEEPTHIN_TC_PAIR") ? atoi(getenv("DEEPTHIN_TC_PAIR")) : 1;
  Layout LP;
  const bool pair = want_pair && n_cb % 2 == 0 && make_layout(g, &LP, true);
  if (pair) L = LP;
  static const int want_cluster =
      getenv("DEEPTHIN_TC_CLUSTER") ? atoi(getenv("DEEPTHIN_TC_CLUSTER")) : 1;
  int csize = 1;
  if (pair) {
    csize = 2;
  } else {
    for (int c : {4, 2})
      if (c <= want_cluster && n_cb % c == 0) { csize = c; break; }
  }
  cuuint32_t box[2] = {KATOM, (cuuint32_t)(BNB / csize)};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(xt), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(x) failed: " + std::to_string((int)cr));
    return DT_E_CUDA;
  }
  TcParams p{};
  p.batch = batch;
  p.q = (int)g.q; p.r_dim = (int)g.r_dim; p.rank = (int)g.rank; p.m = (int)g.m; p.n = (int)g.n;
  p.ldy = (int)g.r_dim;
  p.KB = L.KB; p.S = L.S; p.S_ded = L.S_ded; p.RK = L.RK; p.Nc = L.Nc; p.n_chunks = L.n_chunks;
  p.a_res = L.a_res;
  p.n_cb = n_cb;
  p.n_bt = (int)((batch + BNB - 1) / BNB);
  p.csize = csize;
  p.items = (n_cb / csize) * p.n_bt;  // cluster items: (column-block group, batch tile)
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int clusters = nsm / csize;
  p.per_cta = (p.items + clusters - 1) / clusters;  // items per cluster
  const int grid = ((p.items + p.per_cta - 1) / p.per_cta) * csize;
  p.xf_pk = reinterpret_cast<const uint8_t *>(packed);
  p.wf_pk = p.xf_pk + (packed_x_bytes(g, L) + 255) / 256 * 256;
  p.bias = bias;
  p.y = y;
  p.arg = act_arg;
  static const int dbg_serial = DT_DBG_ENV("DEEPTHIN_REGEN_SERIAL");
  p.dbg_serial = dbg_serial;
  static const int dbg_regen = DT_DBG_ENV("DEEPTHIN_DBG_REGEN");
  p.dbg_regen = dbg_regen;
  p.off_w = L.off_w; p.off_x = L.off_x; p.off_ar = L.off_ar; p.off_br = L.off_br;
  p.off_bar = L.off_bar;
  p.w_sbo = (uint32_t)L.KB * (KATOM / 8) * 128u;
  const int eact = act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act;
  KernelFn fn = pair ? (y_dtype == DT_BF16 ? pick_act_pair<DT_BF16>(eact) : pick_act_pair<DT_F32>(eact))
                     : (y_dtype == DT_BF16 ? pick_act<DT_BF16>(eact) : pick_act<DT_F32>(eact));
  DT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));

  // Debug: DEEPTHIN_TC_TRACE=1 records per-CTA globaltimer stamps and prints a phase summary.
  static const bool tracing = DT_DBG_ENV("DEEPTHIN_TC_TRACE") != 0;
  unsigned long long *tbuf = nullptr;
  if (tracing) {
    DT_CUDA_CHECK(cudaMalloc(&tbuf, (size_t)grid * kTraceSlots * 8));
    DT_CUDA_CHECK(cudaMemsetAsync(tbuf, 0, (size_t)grid * kTraceSlots * 8, st));
    p.trace = tbuf;
  }
  if (csize == 1) {
    fn<<<grid, kThreads, L.total, st>>>(tm, p);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm, p));
  }
  if (int rc = check_launch("tc_general")) return rc;
  if (tracing) {
    std::vector<unsigned long long> h((size_t)grid * kTraceSlots);
    DT_CUDA_CHECK(cudaStreamSynchronize(st));
    DT_CUDA_CHECK(cudaMemcpy(h.data(), tbuf, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(tbuf);
    print_trace(h, grid, p);
  }
  if (act == DT_ACT_SOFTMAX) return launch_row_softmax(batch, g.r_dim, y, y_dtype, st);
  return DT_OK;
}

int launch_pack_x(int64_t batch, int64_t q, int64_t ldx, const void *x, int x_dtype, void *out,
                  cudaStream_t st) {
  const int64_t tot = batch * ldx;
  if (tot == 0) return DT_OK;
  if (ldx % 8 != 0) {
    set_error("pack_x: ldx must be a multiple of 8");
    return DT_E_ARG;
  }
  k_pack_x<<<(unsigned)((tot / 8 + 255) / 256), 256, 0, st>>>(batch, q, ldx, x, x_dtype,
                                                               reinterpret_cast<__nv_bfloat16 *>(out));
  return check_launch("pack_x");
}

int encode_tensor_map_2d(CUtensorMap *tm, int dtype, void *base, uint64_t inner, uint64_t outer,
                         uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                         bool swizzle128) {
  return encode_tensor_map_2d_sw(tm, dtype, base, inner, outer, pitch_bytes, box_inner, box_outer,
                                 swizzle128 ? (int)CU_TENSOR_MAP_SWIZZLE_128B
                                            : (int)CU_TENSOR_MAP_SWIZZLE_NONE);
}

int encode_tensor_map_2d_sw(CUtensorMap *tm, int dtype, void *base, uint64_t inner, uint64_t outer,
                            uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                            int swizzle) {
  PFN_encode_tiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return DT_E_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(tm, dtype == DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    (CUtensorMapSwizzle)swizzle,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
    return DT_E_CUDA;
  }
  return DT_OK;
}

// 3-D map for an MN-major operand: dims (elements of one 128-byte chunk along M/N, K rows,
// chunks along M/N), so ONE box of (chunk, bk, nchunks) lands in shared memory as the UMMA
// canonical MN-major layout [chunk][K row][128 B] (instead of one 2-D box per chunk).
int encode_tensor_map_mn3d(CUtensorMap *tm, int dtype, void *base, uint64_t mn, uint64_t k,
                           uint64_t pitch_bytes, uint32_t bk, uint32_t nchunks, int swizzle) {
  PFN_encode_tiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return DT_E_CUDA;
  }
  const uint64_t esz = dtype == DT_BF16 ? 2 : 4, ce = 128 / esz;
  cuuint64_t dims[3] = {(cuuint64_t)ce, (cuuint64_t)k, (cuuint64_t)(mn / ce)};
  cuuint64_t strides[2] = {(cuuint64_t)pitch_bytes, (cuuint64_t)128};
  cuuint32_t box[3] = {(cuuint32_t)ce, bk, nchunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(tm, dtype == DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    (CUtensorMapSwizzle)swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)cr));
    return DT_E_CUDA;
  }
  return DT_OK;
}

}  // namespace dt
