// Straddling-row (general) layers of low rank as the reference's memoized runs, on tcgen05.
//
// Reference: kernel.py:99-164 (_Layout / _combine_block: every output column j of a general
// geometry reads v[j*q : (j+1)*q], which crosses aux rows of I = xf @ wf in a few "runs"; a run
// is a (x offset, wf offset, length) triple, and the distinct runs over all phases are few —
// config 3's 440 -> 2048 layer (n_f 320, period 8) has 18). The reference computes each distinct
// run dot once per row and combines them with xf (rank 1 only, kernel.py:238-240); restated for
// rank r by superposition:
//
//   P'[b, t*r + k] = sum_i x[b, i] * Wrun_t[k, i]        Wrun_t[k, i] = wf[k, c0_t + i - i0_t]
//                                                        on the run's x range, 0 elsewhere
//   y[b, j] = act( sum_{runs t of phase(j), order o} sum_k xf[a0(j) + o, k] * P'[b, t*r + k] + b_j )
//
// i.e. ONE dense contraction x @ Wrunsᵀ (K = q, N = nruns * r, bf16 hi + lo of wf: two column
// halves added in fp32) and one tiny one P' @ XFfullᵀ (K = nruns * r + the bias slot, tf32) whose
// B rows are zero outside each column's own runs. No W — dense or tiled — ever exists: 2*B*q*N'
// + 2*B*r_dim*K2 flops (config-3 L0: 1.6 GFLOP) instead of 2*B*q*r_dim (29.5 GFLOP), and the
// kernel streams x once and y once (HBM-bound).
//
// One CTA per 128-row tile (persistent), warp roles as k_tc_rows.cu: 0 x + Wruns producer,
// 1 XFfull chunk producer, 2 TMEM owner + MMA issuer, 3-6 P -> tf32 operand, 7-22 epilogue
// (bf16 outputs through swizzled staging, whole-line stores).

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <numeric>
#include <tuple>
#include <vector>

#include "act.cuh"
#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

constexpr int uTM = 128, uNc = 128, uPW = 4, uEpi = 16;
constexpr int uThreads = 32 * (3 + uPW + uEpi);
constexpr int uXS = 2;              // x + Wruns stage ring
constexpr int uBS = 2;              // XFfull chunk ring
constexpr int uMaxRuns = 32, uMaxPeriod = 64, uMaxOrd = 4;
constexpr uint32_t uDCol = 256;

struct RunTable {
  int nruns, period, nord;
  int i0[uMaxRuns], c0[uMaxRuns], len[uMaxRuns];
  signed char prun[uMaxPeriod][uMaxOrd];  // run id of (phase, order), -1 none
};

struct RunsParams {
  int64_t batch;
  int q, r_dim, n_tiles, nkb, npc, np, k2, ka, bslot, n_chunks;
  void *y;
  float arg;
  uint32_t stage_bytes, off_x, off_a2, off_b, off_out, off_bar;
};

__device__ __forceinline__ uint32_t a2u_off(int row, int kk) {  // as k_tc_rows.cu a2n_off
  return (uint32_t)(kk >> 2) * 2048u + (uint32_t)(row >> 3) * 128u + (uint32_t)(row & 7) * 16u +
         (uint32_t)(kk & 3) * 4u;
}
__device__ __forceinline__ uint32_t pk_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}
template <int ACT>
__device__ __forceinline__ float act_runs(float z, float arg) {
  // bf16 outputs: a sigmoid layer's operands are pre-scaled by 1/2 -> one MUFU op
  if constexpr (ACT == DT_ACT_SIGMOID) return fmaf(0.5f, tanh_approx(z), 0.5f);
  return act_out_bf16<DT_BF16, ACT>(z, arg);
}

template <int ACT>
__global__ void __launch_bounds__(uThreads, 1)
    k_tc_runs(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
              const __grid_constant__ CUtensorMap tm_xf, const RunsParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *x_full = bars, *x_empty = bars + uXS;
  uint64_t *b_full = x_empty + uXS, *b_empty = b_full + uBS;
  uint64_t *d_full = b_empty + uBS, *d_empty = d_full + 2;
  uint64_t *p_full = d_empty + 2, *a2_full = p_full + 2, *a2_free = a2_full + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(a2_free + 1);
  // (warp index and TMEM base through a shuffle: provably warp-uniform for the compiler, so the
  // producer / issuer loops — run on all 32 lanes, only the asynchronous instructions predicated
  // on lane 0 — keep their operands in uniform registers: no per-MMA ELECT / R2UR waterfall)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0), lane = threadIdx.x % 32;
  const bool l0 = lane == 0;
  const int ntl = (int)blockIdx.x < p.n_tiles
                      ? (p.n_tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const uint32_t bbytes = (uint32_t)p.ka * uNc * 128u;

  if (threadIdx.x == 0) {
    for (int i = 0; i < uXS; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 1); }
    for (int i = 0; i < uBS; ++i) { mbar_init(&b_full[i], 1); mbar_init(&b_empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], uEpi);
      mbar_init(&p_full[i], 1);
    }
    mbar_init(a2_full, uPW);
    mbar_init(a2_free, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_xf);
  }
  if (warp == 2) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = __shfl_sync(0xffffffffu, *tslot, 0);
  griddep_wait();  // x is the previous layer's output; the operands come from the prep kernel
  griddep_launch_dependents();
  const uint32_t s0 = smem_u32(smem);

  if (warp == 0) {
    // ---------------- x + Wruns producer: per tile, nkb stages of (x k-block, Wruns k-block) ----
    {
      int st = 0;
      uint32_t ph = 0;
      const uint32_t wbytes = (uint32_t)p.np * 128u;
      for (int i = 0; i < ntl; ++i) {
        const int t = (int)blockIdx.x + i * (int)gridDim.x;
        for (int kb = 0; kb < p.nkb; ++kb) {
          mbar_wait(&x_empty[st], ph ^ 1);
          const uint32_t sb = s0 + p.off_x + (uint32_t)st * p.stage_bytes;
          if (l0) {
            mbar_arrive_expect_tx(&x_full[st], (uint32_t)(uTM * 128) + wbytes);
            tma_load_2d_s(sb, &tm_x, smem_u32(&x_full[st]), kb * 64, t * uTM);
            tma_load_2d_s(sb + uTM * 128, &tm_w, smem_u32(&x_full[st]), kb * 64, 0);
          }
          if (++st == uXS) { st = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- XFfull chunk producer ----------------
    {
      int st = 0;
      uint32_t ph = 0;
      for (int i = 0; i < ntl; ++i)
        for (int c = 0; c < p.n_chunks; ++c) {
          mbar_wait(&b_empty[st], ph ^ 1);
          if (l0) {
            mbar_arrive_expect_tx(&b_full[st], bbytes);
            for (int a = 0; a < p.ka; ++a)
              tma_load_2d_s(s0 + p.off_b + (uint32_t)st * bbytes + (uint32_t)(a * uNc * 128), &tm_xf,
                            smem_u32(&b_full[st]), a * 32, c * uNc);
          }
          if (++st == uBS) { st = 0; ph ^= 1; }
        }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ---------------- MMA issuer ----------------
    {
      const uint32_t idA = idesc_f32acc(uTM, (uint32_t)p.np, 1);
      const uint32_t idB = idesc_f32acc(uTM, uNc, 2);
      // descriptors once, then 64-bit additions in the start-address field (16-byte units)
      const uint64_t dX0 = smem_desc(s0 + p.off_x, 16, 1024, SL_SW128);
      const uint64_t dA20 = smem_desc(s0 + p.off_a2, 2048, 128, SL_NONE);
      const uint64_t dB0 = smem_desc(s0 + p.off_b, 16, 1024, SL_SW128);
      const uint32_t st16 = p.stage_bytes >> 4, bb16 = bbytes >> 4;
      const int nk8 = p.k2 / 8;
      int xs = 0, bs = 0, db = 0;
      uint32_t xph = 0, bph = 0, dph = 0;
      for (int i = 0; i <= ntl; ++i) {
        if (i < ntl) {  // phase A of tile i into P[i & 1]: x . [Wruns_hi; Wruns_lo]^T
          const uint32_t d = tbase + (uint32_t)((i & 1) * p.np);
          for (int kb = 0; kb < p.nkb; ++kb) {
            mbar_wait(&x_full[xs], xph);
            tc_fence_after();
            const uint64_t a = dX0 + (uint64_t)((uint32_t)xs * st16);
            const uint64_t b = a + (uint64_t)((uTM * 128) >> 4);
            if (l0) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(d, a + (uint64_t)(2 * k), b + (uint64_t)(2 * k), idA, (kb | k) != 0);
              mma_commit(&x_empty[xs]);
            }
            if (++xs == uXS) { xs = 0; xph ^= 1; }
          }
          if (l0) mma_commit(&p_full[i & 1]);
        }
        if (i >= 1) {  // phase B of tile i-1: A2 (tf32 P') against every XFfull chunk
          mbar_wait(a2_full, (uint32_t)(i - 1) & 1u);
          tc_fence_after();
          for (int c = 0; c < p.n_chunks; ++c) {
            mbar_wait(&b_full[bs], bph);
            mbar_wait(&d_empty[db], dph ^ 1);
            tc_fence_after();
            const uint32_t d = tbase + uDCol + (uint32_t)(db * uNc);
            const uint64_t b = dB0 + (uint64_t)((uint32_t)bs * bb16);
            if (l0) {
              for (int k8 = 0; k8 < nk8; ++k8)  // A2: 4 KB per K step; XFfull: 32 B, next atom every 4
                mma_tf32_ss(d, dA20 + (uint64_t)(256 * k8),
                            b + (uint64_t)((uint32_t)(k8 >> 2) * ((uNc * 128u) >> 4) + (uint32_t)(k8 & 3) * 2u),
                            idB, k8 != 0);
              mma_commit(&b_empty[bs]);
              mma_commit(&d_full[db]);
            }
            if (++bs == uBS) { bs = 0; bph ^= 1; }
            if (++db == 2) { db = 0; dph ^= 1; }
          }
          if (l0) mma_commit(a2_free);  // the P warps may overwrite A2 with the next tile's P'
        }
      }
    }
    __syncwarp();
  } else if (warp < 3 + uPW) {
    // ---------------- P' (TMEM, hi | lo column halves) -> tf32 A operand ----------------
    const int sp = warp & 3, row = 32 * sp + lane;
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    const uint32_t a2 = s0 + p.off_a2;
    for (int i = 0; i < ntl; ++i) {
      mbar_wait(&p_full[i & 1], (uint32_t)(i >> 1) & 1u);
      tc_fence_after();
      if (i > 0) mbar_wait(a2_free, (uint32_t)(i - 1) & 1u);  // phase B of tile i-1 read A2
      const uint32_t pcol = tbase + lane_t + (uint32_t)((i & 1) * p.np);
      for (int g = 0; g < p.k2; g += 32) {  // 32 K values per pass: hi at g, lo at g + npc
        uint32_t vh[32], vl[32];
        tmem_ld_32x32b_x32(pcol + (uint32_t)g, vh);
        tmem_ld_32x32b_x32(pcol + (uint32_t)(g + p.npc), vl);
        tmem_ld_wait();
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
          if (g + k0 < p.k2) {
            uint32_t w[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
              const int kk = g + k0 + q4;
              w[q4] = kk < p.npc ? __float_as_uint(__uint_as_float(vh[k0 + q4]) +
                                                   __uint_as_float(vl[k0 + q4]))
                      : kk == p.bslot ? 0x3f800000u : 0u;  // 1.0 in the bias slot
            }
            sts_v4(a2 + a2u_off(row, g + k0), w[0], w[1], w[2], w[3]);
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(a2_full);
    }
  } else {
    // ---------------- epilogue (bf16 out): 16 warps, four per TMEM lane quarter ----------------
    const int sp = warp & 3;
    const int e = warp - 3 - uPW;
    const int qc = e / 4;
    const uint32_t lane_t = (uint32_t)(32 * sp) << 16;
    constexpr int RB = 64, LPR = 4, RPI = 8, SWM = 3;
    const uint32_t out_s = s0 + p.off_out + (uint32_t)e * (32u * RB);
    int db = 0;
    uint32_t dph = 0;
    for (int i = 0; i < ntl; ++i) {
      const int t = (int)blockIdx.x + i * (int)gridDim.x;
      const int64_t row0 = (int64_t)t * uTM + 32 * sp;
      for (int c = 0; c < p.n_chunks; ++c) {
        mbar_wait(&d_full[db], dph);
        tc_fence_after();
        const int col0 = c * uNc + 32 * qc;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + lane_t + uDCol + (uint32_t)(db * uNc + 32 * qc), v);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&d_empty[db]);
        if (++db == 2) { db = 0; dph ^= 1; }
        if (col0 >= p.r_dim) continue;
        float o[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) o[k] = act_runs<ACT>(__uint_as_float(v[k]), p.arg);
        const uint32_t rb = out_s + (uint32_t)lane * RB;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const float *f = o + ch * 8;
          const int sw = (lane >> 1) & SWM;
          sts_v4(rb + ((uint32_t)(ch ^ sw) << 4), pk_bf16(f[0], f[1]), pk_bf16(f[2], f[3]),
                 pk_bf16(f[4], f[5]), pk_bf16(f[6], f[7]));
        }
        __syncwarp();
        const int ch = lane % LPR;
        const int cb = col0 + ch * 8;
#pragma unroll
        for (int r8 = 0; r8 < 32 / RPI; ++r8) {
          const int r = RPI * r8 + lane / LPR;
          const int sw = (r >> 1) & SWM;
          uint32_t w0, w1, w2, w3;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                       : "r"(out_s + (uint32_t)r * RB + ((uint32_t)(ch ^ sw) << 4)));
          if (row0 + r < p.batch && cb < p.r_dim)
            *reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(p.y) + (row0 + r) * p.r_dim +
                                       cb) = make_uint4(w0, w1, w2, w3);
        }
        __syncwarp();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// Operands from the factors (per call, like k_rows_prep): [Wruns_hi; Wruns_lo] (2 npc rows,
// padded to np, x qp bf16) and XFfull (r_dim x k2 fp32, bias in slot bslot, sigmoid pre-scale).
__global__ void k_runs_prep(RunTable rt, int q, int qp, int r_dim, int n, int rank, int npc, int np,
                            int k2, int bslot, const float *xf, const float *wf, const float *bias,
                            float scale, __nv_bfloat16 *wr, float *xff) {
  griddep_wait();
  const int64_t nw = (int64_t)np * qp, tot = nw + (int64_t)r_dim * k2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < nw) {
      const int row = (int)(e / qp), i = (int)(e - (int64_t)row * qp);
      const int h = row / npc, rr = row - h * npc;  // h: 0 hi, 1 lo (rows >= 2 npc: zero)
      float v = 0.f;
      if (h < 2) {
        const int t = rr / rank, k = rr - t * rank;
        if (i >= rt.i0[t] && i < rt.i0[t] + rt.len[t]) v = wf[(int64_t)k * n + rt.c0[t] + i - rt.i0[t]];
      }
      const __nv_bfloat16 hb = __float2bfloat16_rn(v);
      wr[e] = (h == 0) ? hb : (h == 1 ? __float2bfloat16_rn(v - __bfloat162float(hb)) : hb);
    } else {
      const int64_t f = e - nw;
      const int j = (int)(f / k2), kk = (int)(f - (int64_t)j * k2);
      float v = 0.f;
      if (kk == bslot) {
        v = bias ? bias[j] : 0.f;
      } else if (kk < npc) {
        const int t = kk / rank, k = kk - t * rank, ph = j % rt.period;
        const int64_t a0 = ((int64_t)j * q) / n;
        for (int o = 0; o < rt.nord; ++o)
          if (rt.prun[ph][o] == t) v = xf[(a0 + o) * rank + k];
      }
      xff[f] = v * scale;
    }
  }
}

using RunsFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, RunsParams);

template <int ACT>
RunsFn runs_fn() { return k_tc_runs<ACT>; }

// run table of a geometry (host, cached): the distinct (x offset, wf offset, length) runs over
// all phases (kernel.py:99-164 _Layout), each phase's runs in aux-row order
bool run_table(const Geo &g, RunTable &rt) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int64_t>, std::pair<bool, RunTable>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(g.q, g.n, g.r_dim);
  auto it = cache.find(key);
  if (it != cache.end()) {
    rt = it->second.second;
    return it->second.first;
  }
  RunTable t{};
  bool ok = true;
  const int64_t period = g.n / std::gcd(g.n, g.q);
  if (period > uMaxPeriod) ok = false;
  std::vector<std::tuple<int, int, int>> runs;
  for (int64_t ph = 0; ok && ph < std::min<int64_t>(period, g.r_dim); ++ph) {
    for (int o = 0; o < uMaxOrd; ++o) t.prun[ph][o] = -1;
    int64_t i0 = 0, c0 = (ph * g.q) % g.n;
    int o = 0;
    while (i0 < g.q) {
      const int64_t len = std::min(g.n - c0, g.q - i0);
      const auto r = std::make_tuple((int)i0, (int)c0, (int)len);
      int id = -1;
      for (size_t k = 0; k < runs.size(); ++k)
        if (runs[k] == r) id = (int)k;
      if (id < 0) {
        id = (int)runs.size();
        runs.push_back(r);
      }
      if (o >= uMaxOrd || id >= uMaxRuns) { ok = false; break; }
      t.prun[ph][o++] = (signed char)id;
      i0 += len;
      c0 = 0;
    }
    t.nord = std::max(t.nord, o);
  }
  if (ok) {
    t.nruns = (int)runs.size();
    t.period = (int)std::min<int64_t>(period, g.r_dim);
    for (int k = 0; k < t.nruns; ++k) std::tie(t.i0[k], t.c0[k], t.len[k]) = runs[k];
  }
  cache[key] = {ok, t};
  rt = t;
  return ok;
}

struct RunsGeo {
  int npc, np, k2, ka, bslot, qp, nkb;
};
bool runs_geo(const Geo &g, RunsGeo &u, RunTable &rt) {
  if (g.reuse || !run_table(g, rt)) return false;
  u.npc = rt.nruns * (int)g.rank;
  u.np = (2 * u.npc + 15) / 16 * 16;
  u.k2 = (u.npc + 1 + 7) / 8 * 8;
  u.ka = (u.k2 + 31) / 32;
  u.bslot = u.npc;
  u.qp = (int)((g.q + 63) / 64 * 64);
  u.nkb = u.qp / 64;
  return 2 * u.np <= (int)uDCol && u.k2 <= 64;  // P double buffer below the D buffers
}

}  // namespace

bool tc_runs_ok(const Geo &g, int x_dtype, int y_dtype) {
  if (x_dtype != DT_BF16 || y_dtype != DT_BF16 || g.q % 8 != 0 || g.r_dim % 8 != 0) return false;
  RunsGeo u;
  RunTable rt;
  return runs_geo(g, u, rt);
}

size_t tc_runs_ws(const Geo &g) {
  RunsGeo u;
  RunTable rt;
  if (!runs_geo(g, u, rt)) return 0;
  return (size_t)((int64_t)u.np * u.qp * 2 + 255) / 256 * 256 + (size_t)g.r_dim * u.k2 * 4;
}

int tc_runs_forward(const Geo &g, int64_t batch, const void *x, const float *wf, const float *xf,
                    const float *bias, int act, float act_arg, void *y, char *ws, cudaStream_t st) {
  if (batch == 0) return DT_OK;
  RunsGeo u;
  RunTable rt;
  if (!runs_geo(g, u, rt)) {
    set_error("runs kernel: geometry not eligible");
    return DT_E_UNSUPPORTED;
  }
  __nv_bfloat16 *wr = reinterpret_cast<__nv_bfloat16 *>(ws);
  float *xff = reinterpret_cast<float *>(ws + ((int64_t)u.np * u.qp * 2 + 255) / 256 * 256);
  const float scale = act == DT_ACT_SIGMOID ? 0.5f : 1.f;
  {
    const int64_t tot = (int64_t)u.np * u.qp + g.r_dim * (int64_t)u.k2;
    cudaLaunchConfig_t pc{};
    pc.gridDim = dim3((unsigned)std::min<int64_t>((tot + 255) / 256, 4 * 148));
    pc.blockDim = dim3(256);
    pc.stream = st;
    cudaLaunchAttribute pa[1];
    pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pa[0].val.programmaticStreamSerializationAllowed = 1;
    pc.attrs = pa;
    pc.numAttrs = 1;
    DT_CUDA_CHECK(cudaLaunchKernelEx(&pc, k_runs_prep, rt, (int)g.q, u.qp, (int)g.r_dim, (int)g.n,
                                     (int)g.rank, u.npc, u.np, u.k2, u.bslot, xf, wf, bias, scale, wr,
                                     xff));
    if (int rc = check_launch("runs_prep")) return rc;
  }
  RunsParams p{};
  p.batch = batch;
  p.q = (int)g.q;
  p.r_dim = (int)g.r_dim;
  p.n_tiles = (int)((batch + uTM - 1) / uTM);
  p.nkb = u.nkb;
  p.npc = u.npc;
  p.np = u.np;
  p.k2 = u.k2;
  p.ka = u.ka;
  p.bslot = u.bslot;
  p.n_chunks = (int)((g.r_dim + uNc - 1) / uNc);
  p.y = y;
  p.arg = act_arg;
  p.stage_bytes = (uint32_t)(uTM * 128 + u.np * 128);
  p.off_x = 0;
  p.off_a2 = (p.off_x + uXS * p.stage_bytes + 1023) & ~1023u;
  p.off_b = (p.off_a2 + (uint32_t)(uTM * u.k2 * 4) + 1023) & ~1023u;
  p.off_out = p.off_b + uBS * (uint32_t)(u.ka * uNc * 128);
  p.off_bar = p.off_out + uEpi * 32u * 64u;
  const uint32_t smem_bytes = p.off_bar + 256 + 1024;
  if (smem_bytes > 227 * 1024) {
    set_error("runs kernel: shared memory budget exceeded");
    return DT_E_UNSUPPORTED;
  }
  CUtensorMap tm_x, tm_w, tm_xf;
  if (int rc = encode_tensor_map_2d(&tm_x, DT_BF16, const_cast<void *>(x), (uint64_t)g.q,
                                    (uint64_t)batch, (uint64_t)g.q * 2, 64, uTM, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_w, DT_BF16, wr, (uint64_t)u.qp, (uint64_t)u.np,
                                    (uint64_t)u.qp * 2, 64, (uint32_t)u.np, true))
    return rc;
  if (int rc = encode_tensor_map_2d(&tm_xf, DT_F32, xff, (uint64_t)u.k2, (uint64_t)g.r_dim,
                                    (uint64_t)u.k2 * 4, 32, uNc, true))
    return rc;
  RunsFn fn;
  switch (act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act) {
    case DT_ACT_RELU: fn = runs_fn<DT_ACT_RELU>(); break;
    case DT_ACT_SIGMOID: fn = runs_fn<DT_ACT_SIGMOID>(); break;
    case DT_ACT_TANH: fn = runs_fn<DT_ACT_TANH>(); break;
    case DT_ACT_CLIPPED_RELU: fn = runs_fn<DT_ACT_CLIPPED_RELU>(); break;
    default: fn = runs_fn<DT_ACT_IDENTITY>(); break;
  }
  if (int rc = set_smem_limit(reinterpret_cast<const void *>(fn), (int)smem_bytes)) return rc;
  int dev = 0, nsm = 148;
  DT_CUDA_CHECK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)std::min(p.n_tiles, nsm));
  cfg.blockDim = dim3(uThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  DT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fn, tm_x, tm_w, tm_xf, p));
  if (int rc = check_launch("tc_runs")) return rc;
  return act == DT_ACT_SOFTMAX ? launch_row_softmax(batch, g.r_dim, y, DT_BF16, st) : DT_OK;
}

}  // namespace dt
