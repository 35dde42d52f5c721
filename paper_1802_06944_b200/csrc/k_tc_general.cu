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
//    the block's flat range [j0*q, (j0+128)*q) are one small MMA
//    I_rows(128 x n) = xf_rows(128 x rank) @ wf(rank x n) into TMEM; the
//    epilogue warps read it back (tcgen05.ld), round to bf16 and scatter every
//    element f -> (jj, i) = divmod(f - j0*q, q) into the 128B-swizzled K-major
//    operand layout. The discarded tail (f >= q*r_dim) is never produced.
//  * Main loop: D[j, b] (TMEM, fp32) += W_blk[j, :] . x[b, :] with
//    tcgen05.mma.cta_group::1.kind::f16, M = 128 output columns, N = 128 batch
//    rows, A = the resident W block, B = TMA-staged x tiles (S-stage mbarrier
//    ring). Accumulators are double-buffered in TMEM so the epilogue of tile t
//    overlaps the MMAs of tile t+1.
//  * Epilogue: lanes are output columns, TMEM columns are batch rows, so each
//    warp store instruction writes 32 consecutive outputs of one batch row
//    (coalesced), fused with bias + activation.
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA issuer,
// warps 2-5 regeneration + epilogue.

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "dt_internal.h"
#include "sm100_ptx.cuh"

namespace dt {
namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;
constexpr int BMW = 128;   // W rows (output columns) per block == UMMA M
constexpr int BNB = 128;   // batch rows per tile == UMMA N
constexpr int KATOM = 64;  // bf16 elements per 128-byte swizzle row
constexpr uint32_t kXStage = BNB * 128;   // bytes per x stage (128 rows x 64 bf16)
constexpr uint32_t kWKBlk = BMW * 128;    // bytes per W k-block
constexpr uint32_t kTmemCols = 512;
constexpr int kSmemBudget = 227 * 1024;

struct TcParams {
  int64_t q, r_dim, rank, m, n, batch, ldy;
  int KB, S, RK, Nc, n_chunks, n_cb, n_bt, items, per_cta;
  const __nv_bfloat16 *xf, *wf;
  const float *bias;
  void *y;
  int y_dtype, act;
  float arg;
  uint32_t off_w, off_x, off_ar, off_br, off_bar;
};

__device__ __forceinline__ float act_apply(int act, float z, float arg) {
  switch (act) {
    case DT_ACT_RELU: return z > 0.f ? z : 0.f;
    case DT_ACT_SIGMOID: return 1.f / (1.f + __expf(-z));
    case DT_ACT_TANH: return tanhf(z);
    case DT_ACT_CLIPPED_RELU: return fminf(fmaxf(z, 0.f), arg);
    default: return z;
  }
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// Byte offset of W-block element (jj, i) in the K-major SWIZZLE_128B operand layout.
__device__ __forceinline__ uint32_t w_off(int64_t jj, int64_t i) {
  uint32_t kb = (uint32_t)(i >> 6), col = (uint32_t)(i & 63);
  return kb * kWKBlk + (uint32_t)jj * 128u + ((((col >> 3) ^ (uint32_t)(jj & 7))) << 4) +
         ((col & 7) << 1);
}

// No-swizzle K-major ("interleave") layout of the small regeneration operands:
// 8-row x 16-byte core matrices, K-adjacent cores 128 B apart (LBO), 8-row groups SBO apart.
__device__ __forceinline__ uint32_t core_off(int row, int k, uint32_t sbo) {
  return (uint32_t)(row >> 3) * sbo + (uint32_t)(k >> 3) * 128u + (uint32_t)(row & 7) * 16u +
         (uint32_t)(k & 7) * 2u;
}

// Regenerate the W block of column block cb into shared memory (128 epilogue threads).
__device__ void regen_block(const TcParams &p, int64_t cb, uint8_t *wblk, uint8_t *ar, uint8_t *br,
                            uint64_t *rbar, uint32_t &rphase, uint32_t tbase, int et, int wq,
                            int lane) {
  const int64_t q = p.q, n = p.n, rank = p.rank;
  const int64_t j0 = cb * BMW;
  const int64_t jrows = (int64_t)min((int64_t)BMW, p.r_dim - j0);
  const int64_t fbeg = j0 * q, fend = (j0 + jrows) * q;
  const int64_t a_lo = fbeg / n, a_hi = (int64_t)min(p.m - 1, (fend - 1) / n);
  const uint32_t sbo = (uint32_t)(p.RK / 8) * 128u;
  const int L = 32 * wq + lane;  // TMEM lane (= aux row offset) this thread reads
  const bool pairs = ((n & 1) == 0) && ((q & 1) == 0);
  const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)p.Nc);
  const uint32_t ar_s = smem_u32(ar), br_s = smem_u32(br);

  for (int64_t a0 = a_lo; a0 <= a_hi; a0 += 128) {
    {  // A operand: xf rows a0 .. a0+127 (zero beyond a_hi / rank)
      const int64_t a = a0 + et;
      for (int k = 0; k < p.RK; k += 8) {
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          v[e] = (a <= a_hi && k + e < rank) ? p.xf[a * rank + k + e] : __float2bfloat16(0.f);
        *reinterpret_cast<uint4 *>(ar + core_off(et, k, sbo)) = *reinterpret_cast<uint4 *>(v);
      }
    }
    for (int chunk = 0; chunk < p.n_chunks; ++chunk) {
      const int64_t c0 = (int64_t)chunk * p.Nc;
      for (int nn = et; nn < p.Nc; nn += kEpiThreads) {  // B operand: wf[:, c0+nn]^T
        const int64_t c = c0 + nn;
        for (int k = 0; k < p.RK; k += 8) {
          __align__(16) __nv_bfloat16 v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] = (c < n && k + e < rank) ? p.wf[(k + e) * n + c] : __float2bfloat16(0.f);
          *reinterpret_cast<uint4 *>(br + core_off(nn, k, sbo)) = *reinterpret_cast<uint4 *>(v);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, kEpiThreads);
      if (et == 0) {
        tc_fence_after();
        for (int kk = 0; kk < p.RK / 16; ++kk) {
          uint64_t ad = smem_desc(ar_s + kk * 256u, 128u, sbo, SL_NONE);
          uint64_t bd = smem_desc(br_s + kk * 256u, 128u, sbo, SL_NONE);
          mma_bf16_ss(tbase, ad, bd, idesc, kk > 0);
        }
        mma_commit(rbar);
      }
      mbar_wait(rbar, rphase);
      rphase ^= 1;
      tc_fence_after();
      const int64_t a = a0 + L;
      for (int col0 = 0; col0 < p.Nc; col0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)col0, v);
        tmem_ld_wait();
        if (a > a_hi) continue;
        const int64_t cstart = c0 + col0;
        const int64_t f0 = a * n + cstart - fbeg;
        int64_t jj = floordiv(f0, q), i = f0 - jj * q;
        if (pairs) {
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            if (cstart + t < n && jj >= 0 && jj < jrows) {
              __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[t]), __uint_as_float(v[t + 1]));
              *reinterpret_cast<__nv_bfloat162 *>(wblk + w_off(jj, i)) = h;
            }
            i += 2;
            if (i >= q) { i -= q; ++jj; }
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            if (cstart + t < n && jj >= 0 && jj < jrows)
              *reinterpret_cast<__nv_bfloat16 *>(wblk + w_off(jj, i)) =
                  __float2bfloat16_rn(__uint_as_float(v[t]));
            if (++i == q) { i = 0; ++jj; }
          }
        }
      }
      tc_fence_before();
      named_bar_sync(1, kEpiThreads);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_tc_general(const __grid_constant__ CUtensorMap tm_x, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t *wblk = smem + p.off_w;
  uint8_t *xst = smem + p.off_x;
  uint8_t *ar = smem + p.off_ar;
  uint8_t *br = smem + p.off_br;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *full = bars, *empty = bars + p.S, *tfull = bars + 2 * p.S, *tempty = tfull + 2;
  uint64_t *bready = tempty + 2, *rbar = bready + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(rbar + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t item_beg = (int64_t)blockIdx.x * p.per_cta;
  const int64_t item_end = (int64_t)min((int64_t)p.items, item_beg + (int64_t)p.per_cta);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], kEpiThreads); }
    mbar_init(bready, 1);
    mbar_init(rbar, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tm_x);
  if (warp == 1) tmem_alloc(tslot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t it = item_beg; it < item_end; ++it) {
        const int32_t b0 = (int32_t)((it % p.n_bt) * BNB);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kXStage);
          tma_load_2d(xst + (size_t)stage * kXStage, &tm_x, &full[stage], kb * KATOM, b0);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(BMW, BNB);
      const uint32_t w_s = smem_u32(wblk), x_s = smem_u32(xst);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0, bphase = 0;
      int64_t cur_cb = -1;
      for (int64_t it = item_beg; it < item_end; ++it) {
        const int64_t cb = it / p.n_bt;
        if (cb != cur_cb) {
          mbar_wait(bready, bphase);
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
            uint64_t ad = smem_desc(w_s + kb * kWKBlk + k * 32, 16, 1024, SL_SW128);
            uint64_t bd = smem_desc(x_s + stage * kXStage + k * 32, 16, 1024, SL_SW128);
            mma_bf16_ss(d, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == p.S) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------- regeneration + epilogue (warps 2-5) ----------------
    const int et = threadIdx.x - 64;
    const int wq = warp & 3;
    const int jl = 32 * wq + lane;  // output column within the block (TMEM lane)
    // zero the K padding [q, KB*64) of every W row once
    for (int64_t i = p.q; i < (int64_t)p.KB * KATOM; ++i)
      *reinterpret_cast<__nv_bfloat16 *>(wblk + w_off(et, i)) = __float2bfloat16(0.f);
    uint32_t rphase = 0, acc_phase = 0;
    int acc = 0;
    int64_t cur_cb = -1;
    float bias_j = 0.f;
    for (int64_t it = item_beg; it < item_end; ++it) {
      const int64_t cb = it / p.n_bt, bt = it % p.n_bt;
      const int64_t j = cb * BMW + jl;
      if (cb != cur_cb) {
        regen_block(p, cb, wblk, ar, br, rbar, rphase, tbase, et, wq, lane);
        fence_proxy_async_smem();
        tc_fence_before();
        named_bar_sync(1, kEpiThreads);
        if (et == 0) mbar_arrive(bready);
        cur_cb = cb;
        bias_j = (p.bias && j < p.r_dim) ? p.bias[j] : 0.f;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t b0 = bt * BNB;
      const bool jok = j < p.r_dim;
      for (int c32 = 0; c32 < BNB / 32; ++c32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * wq) << 16) + (uint32_t)(acc * BNB + c32 * 32), v);
        tmem_ld_wait();
        if (!jok) continue;
        const int64_t bb = b0 + c32 * 32;
        if (p.y_dtype == DT_BF16) {
          __nv_bfloat16 *y = reinterpret_cast<__nv_bfloat16 *>(p.y);
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (bb + r < p.batch)
              y[(bb + r) * p.ldy + j] =
                  __float2bfloat16_rn(act_apply(p.act, __uint_as_float(v[r]) + bias_j, p.arg));
        } else {
          float *y = reinterpret_cast<float *>(p.y);
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (bb + r < p.batch)
              y[(bb + r) * p.ldy + j] = act_apply(p.act, __uint_as_float(v[r]) + bias_j, p.arg);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kTmemCols);
  }
}

// x (fp32 or bf16, row stride q) -> bf16 with row stride ldx (zero padded).
__global__ void k_pack_x(int64_t batch, int64_t q, int64_t ldx, const void *x, int x_dtype,
                         __nv_bfloat16 *out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= batch * ldx) return;
  int64_t b = idx / ldx, i = idx % ldx;
  float v = 0.f;
  if (i < q)
    v = x_dtype == DT_BF16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(x)[b * q + i])
                           : reinterpret_cast<const float *>(x)[b * q + i];
  out[idx] = __float2bfloat16_rn(v);
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
  int KB, S, RK, Nc, n_chunks;
  uint32_t off_w, off_x, off_ar, off_br, off_bar, total;
};

bool make_layout(const Geo &g, Layout *L) {
  L->KB = (int)((g.q + KATOM - 1) / KATOM);
  L->RK = (int)((g.rank + 15) / 16 * 16);
  L->n_chunks = (int)((g.n + 255) / 256);
  L->Nc = (int)(((g.n + L->n_chunks - 1) / L->n_chunks + 31) / 32 * 32);
  if (L->RK > 64) return false;
  uint32_t w = (uint32_t)L->KB * kWKBlk;
  uint32_t arb = 128u * L->RK * 2, brb = (uint32_t)L->Nc * L->RK * 2;
  uint32_t fixed = w + arb + brb + 1024 /*barriers*/ + 1024 /*alignment slack*/;
  int S = 0;
  for (int s = 8; s >= 2; --s)
    if (fixed + (uint32_t)s * kXStage <= (uint32_t)kSmemBudget) { S = s; break; }
  if (S == 0) return false;
  L->S = S;
  L->off_w = 0;
  L->off_x = w;
  L->off_ar = L->off_x + (uint32_t)S * kXStage;
  L->off_br = L->off_ar + arb;
  L->off_bar = (L->off_br + brb + 15) / 16 * 16;
  L->total = L->off_bar + 512 + 1024;
  return true;
}

}  // namespace

size_t tc_general_ws(const Geo &g, int64_t batch) {
  int64_t ldx = (g.q + 7) / 8 * 8;
  return (size_t)batch * ldx * 2 + 256;
}

int tc_general_forward(const Geo &g, int64_t batch, const void *x, int x_dtype,
                       const uint16_t *xf_bf16, const uint16_t *wf_bf16, const float *bias,
                       int act, float act_arg, void *y, int y_dtype, char *ws, size_t ws_bytes,
                       cudaStream_t st) {
  Layout L;
  if (!make_layout(g, &L)) {
    set_error("tcgen05 general path: q=" + std::to_string(g.q) + ", rank=" +
              std::to_string(g.rank) + " does not fit the resident-W-block kernel "
              "(needs ceil(q/64)*16 KB + stages <= 227 KB and rank <= 64)");
    return DT_E_UNSUPPORTED;
  }
  if (batch == 0) return DT_OK;
  PFN_encode_tiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable from the driver");
    return DT_E_CUDA;
  }
  // TMA needs a bf16 x whose row pitch is a multiple of 16 bytes.
  const void *xt = x;
  int64_t ldx = g.q;
  if (x_dtype != DT_BF16 || (g.q % 8) != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
    ldx = (g.q + 7) / 8 * 8;
    size_t need = (size_t)batch * ldx * 2;
    if (need > ws_bytes) {
      set_error("forward workspace too small for the packed bf16 input");
      return DT_E_ARG;
    }
    int64_t tot = batch * ldx;
    k_pack_x<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(batch, g.q, ldx, x, x_dtype,
                                                             reinterpret_cast<__nv_bfloat16 *>(ws));
    if (int rc = check_launch("pack_x")) return rc;
    xt = ws;
  }
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)g.q, (cuuint64_t)batch};
  cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
  cuuint32_t box[2] = {KATOM, BNB};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(xt), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(x) failed: " + std::to_string((int)cr));
    return DT_E_CUDA;
  }
  TcParams p{};
  p.q = g.q; p.r_dim = g.r_dim; p.rank = g.rank; p.m = g.m; p.n = g.n; p.batch = batch;
  p.ldy = g.r_dim;
  p.KB = L.KB; p.S = L.S; p.RK = L.RK; p.Nc = L.Nc; p.n_chunks = L.n_chunks;
  p.n_cb = (int)((g.r_dim + BMW - 1) / BMW);
  p.n_bt = (int)((batch + BNB - 1) / BNB);
  p.items = p.n_cb * p.n_bt;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  p.per_cta = (p.items + nsm - 1) / nsm;
  int grid = (p.items + p.per_cta - 1) / p.per_cta;
  p.xf = reinterpret_cast<const __nv_bfloat16 *>(xf_bf16);
  p.wf = reinterpret_cast<const __nv_bfloat16 *>(wf_bf16);
  p.bias = bias;
  p.y = y;
  p.y_dtype = y_dtype;
  p.act = act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act;
  p.arg = act_arg;
  p.off_w = L.off_w; p.off_x = L.off_x; p.off_ar = L.off_ar; p.off_br = L.off_br;
  p.off_bar = L.off_bar;
  static bool attr_set = false;
  if (!attr_set) {
    DT_CUDA_CHECK(cudaFuncSetAttribute(k_tc_general, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBudget));
    attr_set = true;
  }
  k_tc_general<<<grid, kThreads, L.total, st>>>(tm, p);
  if (int rc = check_launch("tc_general")) return rc;
  if (act == DT_ACT_SOFTMAX) return launch_row_softmax(batch, g.r_dim, y, y_dtype, st);
  return DT_OK;
}

}  // namespace dt
