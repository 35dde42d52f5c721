// Tensor-core training step of reuse geometries (n_f | q): the forward + MSE gradient and the
// backward through the inverse re-layout, every contraction on our own tcgen05 GEMMs
// (k_tc_xgemm.cu). BASELINE config 5. Reference: grad.py:63-95 (layer_backward), :98-103
// (loss_and_grad "mse"), train.py:86-117 (DeepThinWeights), restated without W:
//
//   P    = x.view(B*s, n) @ wf^T              bf16 x, wf as bf16 hi + lo (two column halves of
//                                              one GEMM, added in its epilogue), fp32 P
//   z    = P.view(B, s*r) @ XF2^T + b          tf32; epilogue: g = 2 (z - t) / N, sum (z - t)^2
//                                              (fp64 partials), fixed-order column sums of g
//   d_b  = sum_b g                             (the column sums, reduced in row-block order)
//   dXF2 = g^T @ P.view(B, s*r) -> d_xf        tf32, both operands MN-major (no transpose copy),
//                                              split-K, fixed-order reduce; zero tail rows
//   H    = g @ XF2                             tf32, XF2 MN-major; epilogue writes H re-laid as
//                                              (B*s x r) bf16 hi | lo
//   d_wf = H'^T @ x'                           computed as x'^T @ [H'_hi | H'_lo] (bf16, both
//                                              MN-major, split-K), reduced transposed with the
//                                              hi + lo halves added
//   d_in = H' @ wf                             tf32 (only when requested)
//
// XF2 = xf viewed (r_dim x s*r): the reuse identity (kernel.py:1-16) — output column j reads aux
// rows j*s .. j*s+s-1 — so the re-layout is a view, never a copy. No float atomics anywhere:
// results are bitwise repeatable.

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "dt_internal.h"

namespace dt {
namespace {

int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

int num_sms() {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

// [hi | lo] bf16 rows of an fp32 matrix: hi (rows x cols) then lo (rows x cols), contiguous
__global__ void k_split_hi_lo(int64_t count, const float *src, __nv_bfloat16 *hi, __nv_bfloat16 *lo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[i];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi[i] = h;
    lo[i] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

int split_wf(const Geo &g, const float *wf, __nv_bfloat16 *wf2, cudaStream_t st) {
  const int64_t cnt = g.rank * g.n;
  k_split_hi_lo<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 1184), 256, 0, st>>>(
      cnt, wf, wf2, wf2 + cnt);
  return check_launch("split_hi_lo");
}

// GEMM descriptors (shared by the workspace sizing and the launches)
XGemm gemm_p(const Geo &g, int64_t batch) {  // P = x' @ [wf_hi; wf_lo]^T, halves added
  XGemm x;
  x.M = batch * g.s; x.N = 2 * g.rank; x.K = g.n;
  x.a_mn = 0; x.b_mn = 0; x.el = 0;
  x.BN = x.N <= 64 ? 64 : (x.N <= 128 ? 128 : 256);
  x.epi = 2; x.pair_half = (int)g.rank;
  return x;
}
XGemm gemm_z(const Geo &g, int64_t batch) {  // z = P2 @ XF2^T (+ b), MSE epilogue
  XGemm x;
  x.M = batch; x.N = g.r_dim; x.K = g.s * g.rank;
  x.a_mn = 0; x.b_mn = 0; x.el = 1; x.BN = 256;
  x.epi = 1;
  if (int bn = DT_DBG_ENV("DEEPTHIN_MSE_BN")) x.BN = bn;  // timing builds: tile experiments
  return x;
}
XGemm gemm_dxf(const Geo &g, int64_t batch) {  // dXF2 = g^T @ P2
  XGemm x;
  const int64_t SR = g.s * g.rank;
  x.M = g.r_dim; x.N = SR; x.K = batch;
  x.a_mn = 1; x.b_mn = 1; x.el = 1;
  x.BN = SR > 128 ? 256 : (SR > 64 ? 128 : 64);
  x.splits = xgemm_splits(x.M, x.N, x.K, x.BN, 1, num_sms());
  x.ks_major = 1;  // the splits' P slices are shared by every row block: run them together
  return x;
}
XGemm gemm_h(const Geo &g, int64_t batch, int epi) {  // H = g @ XF2
  XGemm x;
  const int64_t SR = g.s * g.rank;
  x.M = batch; x.N = SR; x.K = g.r_dim;
  x.a_mn = 0; x.b_mn = 1; x.el = 1;
  x.BN = SR > 128 ? 256 : (SR > 64 ? 128 : 64);
  x.epi = epi;
  x.h_r = (int)g.rank; x.h_s = (int)g.s;
  return x;
}
XGemm gemm_dwf(const Geo &g, int64_t batch) {  // D' (n x 2r) = x'^T @ H2, then transposed + paired
  XGemm x;
  x.M = g.n; x.N = 2 * g.rank; x.K = batch * g.s;
  x.a_mn = 1; x.b_mn = 1; x.el = 0;
  x.BN = x.N <= 128 ? 128 : 256;  // bf16 MN-major B: >= 64 columns per CTA half
  x.splits = xgemm_splits(x.M, x.N, x.K, x.BN, 0, num_sms());
  x.reduce_transpose = 1;
  x.reduce_pair_half = (int)g.rank;
  return x;
}
XGemm gemm_din(const Geo &g, int64_t batch) {  // d_in (B*s x n) = H' @ wf
  XGemm x;
  x.M = batch * g.s; x.N = g.n; x.K = g.rank;
  x.a_mn = 0; x.b_mn = 1; x.el = 1;
  x.BN = g.n > 128 ? 256 : (g.n > 64 ? 128 : 64);
  return x;
}

int64_t n_mb(int64_t rows) { return (rows + 255) / 256; }

// Forward + MSE workspace: wf2 | x16 | P | loss partials | column-sum partials | reduce scratch
struct FwdWs {
  size_t wf2, x16, p, loss, cols, scratch, total;
  FwdWs(const Geo &g, int64_t batch) {
    const XGemm z = gemm_z(g, batch);
    wf2 = 0;
    x16 = wf2 + rup(2 * g.rank * g.n * 2, 256);
    p = x16 + rup(batch * g.q * 2, 256);
    loss = p + rup(batch * g.s * g.rank * 4, 256);
    cols = loss + rup(n_mb(z.M) * ((z.N + 255) / 256) * 16 * 8, 256);
    scratch = cols + rup(2 * n_mb(z.M) * z.N * 4, 256);
    total = scratch + rup(xgemm_reduce_scratch((int)(2 * n_mb(z.M)), z.N), 256);
  }
};

// Backward workspace: pre | gbuf | x16 | wf2 | P | H2 | H (d_in) | part | colsum | ffma
struct BwdWs {
  size_t pre, gbuf, x16, wf2, p, h2, h, part, cols, ffma, total;
  BwdWs(const Geo &g, int64_t batch) {
    const int64_t SR = g.s * g.rank;
    pre = 0;
    gbuf = pre + rup(batch * g.r_dim * 4, 256);
    x16 = gbuf + rup(batch * g.r_dim * 4, 256);
    wf2 = x16 + rup(batch * g.q * 2, 256);
    p = wf2 + rup(2 * g.rank * g.n * 2, 256);
    h2 = p + rup(batch * SR * 4, 256);
    h = h2 + rup(batch * SR * 4, 256);
    part = h + rup(batch * SR * 4, 256);
    cols = part + rup(std::max(xgemm_ws(gemm_dxf(g, batch)), xgemm_ws(gemm_dwf(g, batch))), 256);
    ffma = cols + rup(colsum_ws(batch, g.r_dim), 256);
    total = ffma + rup(ffma_forward_ws(g, batch), 256);
  }
};

int x_bf16(const Geo &g, int64_t batch, const void *x, int x_dtype, char *x16, const void **xt,
           cudaStream_t st) {
  *xt = x;
  if (x_dtype != DT_BF16 || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
    if (int rc = launch_pack_x(batch, g.q, g.q, x, x_dtype, x16, st)) return rc;
    *xt = x16;
  }
  return DT_OK;
}

int run_p(const Geo &g, int64_t batch, const void *xt, const __nv_bfloat16 *wf2, float *P,
          cudaStream_t st) {
  XGemm x = gemm_p(g, batch);
  x.A = xt; x.lda = g.n;
  x.B = wf2; x.ldb = g.n;
  x.out = P; x.ldo = g.rank;
  return xgemm(x, st);
}

}  // namespace

bool xtrain_ok(const Geo &g) {
  return g.reuse && g.n % 8 == 0 && g.rank % 4 == 0 && 2 * g.rank <= 256 && g.r_dim % 4 == 0 &&
         g.q % 8 == 0 && g.m * g.rank < INT32_MAX && g.q * g.r_dim < ((int64_t)1 << 40);
}

size_t xtrain_forward_mse_ws(const Geo &g, int64_t batch) { return FwdWs(g, batch).total; }

int xtrain_forward_mse(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                       const float *wf, const float *bias, const float *target, double scale,
                       float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st,
                       float *d_bias, float *p_out) {
  const FwdWs L(g, batch);
  if (ws_bytes < L.total) {
    set_error("forward+mse workspace too small: need " + std::to_string(L.total));
    return DT_E_ARG;
  }
  __nv_bfloat16 *wf2 = reinterpret_cast<__nv_bfloat16 *>(ws + L.wf2);
  float *P = p_out ? p_out : reinterpret_cast<float *>(ws + L.p);
  double *loss = reinterpret_cast<double *>(ws + L.loss);
  float *cols = reinterpret_cast<float *>(ws + L.cols);
  const void *xt;
  if (int rc = x_bf16(g, batch, x, x_dtype, ws + L.x16, &xt, st)) return rc;
  if (int rc = split_wf(g, wf, wf2, st)) return rc;
  if (int rc = run_p(g, batch, xt, wf2, P, st)) return rc;
  const int64_t SR = g.s * g.rank;
  XGemm z = gemm_z(g, batch);
  z.A = P; z.lda = SR;
  z.B = xf; z.ldb = SR;
  z.out = grad; z.ldo = g.r_dim;
  z.bias = bias;
  z.target = target; z.ldt = g.r_dim;
  z.scale = (float)scale;
  z.loss_part = loss;
  int64_t n_part = 0;
  z.n_loss_part = &n_part;
  z.colsum_part = cols;
  if (int rc = xgemm(z, st)) return rc;
  if (loss_sum)
    if (int rc = xgemm_sum_f64(n_part, loss, loss_sum, ws + L.scratch, st)) return rc;
  if (d_bias)
    if (int rc = xgemm_colsum((int)(2 * n_mb(batch)), g.r_dim, cols, d_bias, ws + L.scratch, st))
      return rc;
  return DT_OK;
}

size_t xtrain_backward_ws(const Geo &g, int64_t batch) { return BwdWs(g, batch).total; }

int xtrain_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                    const float *wf, const float *bias, int act, float act_arg, const float *up,
                    float *d_xf, float *d_wf, float *d_bias, float *d_input, char *ws,
                    size_t ws_bytes, cudaStream_t st, const float *p_in) {
  const BwdWs L(g, batch);
  if (ws_bytes < L.total) {
    set_error("backward workspace too small: need " + std::to_string(L.total));
    return DT_E_ARG;
  }
  if (batch == 0) {  // zero gradients of an empty batch
    DT_CUDA_CHECK(cudaMemsetAsync(d_xf, 0, (size_t)g.m * g.rank * 4, st));
    DT_CUDA_CHECK(cudaMemsetAsync(d_wf, 0, (size_t)g.rank * g.n * 4, st));
    if (d_bias) DT_CUDA_CHECK(cudaMemsetAsync(d_bias, 0, (size_t)g.r_dim * 4, st));
    return DT_OK;
  }
  const int64_t SR = g.s * g.rank;
  float *pre = reinterpret_cast<float *>(ws + L.pre);
  float *gbuf = reinterpret_cast<float *>(ws + L.gbuf);
  __nv_bfloat16 *wf2 = reinterpret_cast<__nv_bfloat16 *>(ws + L.wf2);
  __nv_bfloat16 *H2 = reinterpret_cast<__nv_bfloat16 *>(ws + L.h2);
  float *part = reinterpret_cast<float *>(ws + L.part);
  const float *gp = up;
  if (act != DT_ACT_IDENTITY) {
    // g = up * act'(pre), pre recomputed in exact fp32 (FFMA): act' is sensitive where |pre| ~ 1
    // while a tensor-core forward's error scales with max|pre|
    if (int rc = ffma_forward(g, batch, x, x_dtype, xf, wf, bias, DT_ACT_IDENTITY, 0.f, pre,
                              DT_F32, ws + L.ffma, ffma_forward_ws(g, batch), st))
      return rc;
    if (int rc = launch_act_grad(batch * g.r_dim, up, pre, act, act_arg, gbuf, st)) return rc;
    gp = gbuf;
  }
  if (d_bias)
    if (int rc = launch_colsum(batch, g.r_dim, gp, d_bias, reinterpret_cast<float *>(ws + L.cols), st))
      return rc;
  const void *xt;
  if (int rc = x_bf16(g, batch, x, x_dtype, ws + L.x16, &xt, st)) return rc;
  const float *P = p_in;
  if (!P) {
    if (int rc = split_wf(g, wf, wf2, st)) return rc;
    float *Pw = reinterpret_cast<float *>(ws + L.p);
    if (int rc = run_p(g, batch, xt, wf2, Pw, st)) return rc;
    P = Pw;
  }
  // d_xf rows [0, r_dim*s) = dXF2 = g^T @ P2; the discarded tail rows get 0 (grad.py:88-90)
  {
    XGemm d = gemm_dxf(g, batch);
    d.A = gp; d.lda = g.r_dim;
    d.B = P; d.ldb = SR;
    d.out = d_xf; d.ldo = SR;
    d.part = part;
    if (int rc = xgemm(d, st)) return rc;
    const int64_t tail = (g.m - g.r_dim * g.s) * g.rank;
    if (tail > 0) DT_CUDA_CHECK(cudaMemsetAsync(d_xf + g.r_dim * SR, 0, (size_t)tail * 4, st));
  }
  // d_xf and d_bias are final: a data-parallel caller's all-reduce of them may start now
  // (dist.GradReducer), overlapping H and d_wf below
  if (int rc = backward_event_record(st)) return rc;
  // H = g @ XF2, written re-laid as H2 = [hi | lo] (B*s x 2r bf16)
  {
    XGemm h = gemm_h(g, batch, 3);
    h.A = gp; h.lda = g.r_dim;
    h.B = xf; h.ldb = SR;
    h.out16 = H2;
    if (int rc = xgemm(h, st)) return rc;
  }
  // d_wf = H'^T @ x' = (x'^T @ [H'_hi | H'_lo])^T with the halves added
  {
    XGemm w = gemm_dwf(g, batch);
    w.A = xt; w.lda = g.n;
    w.B = H2; w.ldb = 2 * g.rank;
    w.out = d_wf; w.ldo = g.n;
    w.part = part;
    if (int rc = xgemm(w, st)) return rc;
  }
  if (d_input) {  // d_in (B*s x n) = H' @ wf, H in fp32 (tf32 products)
    float *H = reinterpret_cast<float *>(ws + L.h);
    XGemm h = gemm_h(g, batch, 0);
    h.A = gp; h.lda = g.r_dim;
    h.B = xf; h.ldb = SR;
    h.out = H; h.ldo = SR;
    if (int rc = xgemm(h, st)) return rc;
    XGemm d = gemm_din(g, batch);
    d.A = H; d.lda = g.rank;
    d.B = wf; d.ldb = g.n;
    d.out = d_input; d.ldo = g.n;
    if (int rc = xgemm(d, st)) return rc;
  }
  return DT_OK;
}


// =============================================================================================
// Backward of general (straddling) geometries on the tensor cores (grad.py:63-95):
//   g       = upstream (.* act'(pre), pre recomputed in exact fp32)
//   d_bias  = sum_b g
//   d_W^T   = g^T @ x   (r_dim x q)   = d_v[0 : q*r_dim], the flat inverse re-layout: row j of
//             d_W^T is v[j*q : (j+1)*q] (factor.py:87-93), so the row-major product IS d_v and
//             d_aux = d_v viewed (m x n) with a zero tail — no scatter kernel
//             bf16 x (exact) against g split hi | lo and stacked along K (two bf16 products in
//             one GEMM: B's rows wrap), fp32 accumulate
//   d_xf    = d_aux @ wf^T                    (tf32)
//   d_wf    = xf^T @ d_aux = (d_aux^T @ xf)^T (tf32, both MN-major, transposed reduce)
//   d_input = g @ W^T                         (tf32, W = decompress(fp) in fp32; only if asked)
// =============================================================================================
namespace {

__global__ void k_split_g_rows(int64_t rows, int64_t cols, int64_t rows_p, const float *g,
                               __nv_bfloat16 *g2) {
  // g2 rows [0, rows_p): hi (zero past rows), rows [rows_p, 2 rows_p): lo
  const int64_t tot = rows_p * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const float v = r < rows ? g[i] : 0.f;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    g2[i] = h;
    g2[tot + i] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

XGemm gemm_dwt(const Geo &g, int64_t batch) {  // d_W^T (r_dim x q) = [g_hi; g_lo]^T @ [x; x]
  XGemm x;
  const int64_t bp = rup(batch, 64);
  x.M = g.r_dim; x.N = g.q; x.K = 2 * bp;
  x.a_mn = 1; x.b_mn = 1; x.el = 0;
  x.b_wrap_k = bp; x.b_rows = batch;
  x.BN = g.q > 128 ? 256 : 128;
  x.splits = xgemm_splits(x.M, x.N, x.K, x.BN, 0, num_sms());
  x.ks_major = 1;
  x.force_part = (g.q % 4) ? 1 : 0;
  return x;
}
XGemm gemm_gdxf(const Geo &g) {  // d_xf (m x r) = d_aux (m x n) @ wf^T
  XGemm x;
  x.M = g.m; x.N = g.rank; x.K = g.n;
  x.a_mn = 0; x.b_mn = 0; x.el = 1;
  x.BN = g.rank <= 64 ? 64 : (g.rank <= 128 ? 128 : 256);
  x.splits = xgemm_splits(x.M, x.N, x.K, x.BN, 1, num_sms());
  x.force_part = 1;  // any rank: output pitch r
  return x;
}
XGemm gemm_gdwf(const Geo &g) {  // D' (n x r) = d_aux^T @ xf, reduced transposed into d_wf
  XGemm x;
  x.M = g.n; x.N = g.rank; x.K = g.m;
  x.a_mn = 1; x.b_mn = 1; x.el = 1;
  x.BN = g.rank <= 64 ? 64 : (g.rank <= 128 ? 128 : 256);
  x.splits = xgemm_splits(x.M, x.N, x.K, x.BN, 1, num_sms());
  x.reduce_transpose = 1;
  return x;
}
XGemm gemm_gdin(const Geo &g, int64_t batch) {  // d_input (B x q) = g @ W^T, W (q x r_dim)
  XGemm x;
  x.M = batch; x.N = g.q; x.K = g.r_dim;
  x.a_mn = 0; x.b_mn = 0; x.el = 1;
  x.BN = g.q > 128 ? 256 : (g.q > 64 ? 128 : 64);
  x.force_part = (g.q % 4) ? 1 : 0;
  return x;
}

struct GenWs {
  size_t pre, gbuf, g2, x16, dwt, w, part, cols, ffma, total;
  GenWs(const Geo &g, int64_t batch) {
    const int64_t bp = rup(batch, 64), ldx = rup(g.q, 8);
    pre = 0;
    gbuf = pre + rup(batch * g.r_dim * 4, 256);
    g2 = gbuf + rup(batch * g.r_dim * 4, 256);
    x16 = g2 + rup(2 * bp * g.r_dim * 2, 256);
    dwt = x16 + rup(batch * ldx * 2, 256);
    w = dwt + rup(g.m * g.n * 4, 256);
    part = w + rup(g.q * g.r_dim * 4, 256);
    const size_t pb = std::max(std::max(xgemm_ws(gemm_dwt(g, batch)), xgemm_ws(gemm_gdxf(g))),
                               std::max(xgemm_ws(gemm_gdwf(g)), xgemm_ws(gemm_gdin(g, batch))));
    cols = part + rup(pb, 256);
    ffma = cols + rup(colsum_ws(batch, g.r_dim), 256);
    total = ffma + rup(ffma_forward_ws(g, batch), 256);
  }
};

}  // namespace

bool xback_general_ok(const Geo &g) {
  return !g.reuse && g.r_dim % 8 == 0 && g.n % 4 == 0 && g.rank % 4 == 0 && g.rank <= 256 &&
         g.m * g.n < ((int64_t)1 << 31) && g.q * g.r_dim < ((int64_t)1 << 31);
}

size_t xback_general_ws(const Geo &g, int64_t batch) { return GenWs(g, batch).total; }

int xback_general(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                  const float *wf, const float *bias, int act, float act_arg, const float *up,
                  float *d_xf, float *d_wf, float *d_bias, float *d_input, char *ws,
                  size_t ws_bytes, cudaStream_t st) {
  const GenWs L(g, batch);
  if (ws_bytes < L.total) {
    set_error("backward workspace too small: need " + std::to_string(L.total));
    return DT_E_ARG;
  }
  if (batch == 0) {
    DT_CUDA_CHECK(cudaMemsetAsync(d_xf, 0, (size_t)g.m * g.rank * 4, st));
    DT_CUDA_CHECK(cudaMemsetAsync(d_wf, 0, (size_t)g.rank * g.n * 4, st));
    if (d_bias) DT_CUDA_CHECK(cudaMemsetAsync(d_bias, 0, (size_t)g.r_dim * 4, st));
    return DT_OK;
  }
  const float *gp = up;
  if (act != DT_ACT_IDENTITY) {
    float *pre = reinterpret_cast<float *>(ws + L.pre);
    float *gbuf = reinterpret_cast<float *>(ws + L.gbuf);
    if (int rc = ffma_forward(g, batch, x, x_dtype, xf, wf, bias, DT_ACT_IDENTITY, 0.f, pre,
                              DT_F32, ws + L.ffma, ffma_forward_ws(g, batch), st))
      return rc;
    if (int rc = launch_act_grad(batch * g.r_dim, up, pre, act, act_arg, gbuf, st)) return rc;
    gp = gbuf;
  }
  if (d_bias)
    if (int rc = launch_colsum(batch, g.r_dim, gp, d_bias, reinterpret_cast<float *>(ws + L.cols), st))
      return rc;
  // bf16 x with a 16-byte pitch (TMA)
  const int64_t ldx = rup(g.q, 8);
  const void *xt = x;
  if (x_dtype != DT_BF16 || ldx != g.q || (reinterpret_cast<uintptr_t>(x) & 15) != 0) {
    if (int rc = launch_pack_x(batch, g.q, ldx, x, x_dtype, ws + L.x16, st)) return rc;
    xt = ws + L.x16;
  }
  // g -> [g_hi; g_lo] (bf16, K-stacked)
  const int64_t bp = rup(batch, 64);
  __nv_bfloat16 *g2 = reinterpret_cast<__nv_bfloat16 *>(ws + L.g2);
  k_split_g_rows<<<(unsigned)std::min<int64_t>((bp * g.r_dim + 255) / 256, 4 * 1184), 256, 0, st>>>(
      batch, g.r_dim, bp, gp, g2);
  if (int rc = check_launch("split_g_rows")) return rc;
  float *part = reinterpret_cast<float *>(ws + L.part);
  // d_v = d_W^T flat; zero tail of the aux matrix
  float *dv = reinterpret_cast<float *>(ws + L.dwt);
  {
    XGemm d = gemm_dwt(g, batch);
    d.A = g2; d.lda = g.r_dim;
    d.B = xt; d.ldb = ldx;
    d.out = dv; d.ldo = g.q;
    d.part = part;
    if (int rc = xgemm(d, st)) return rc;
    const int64_t tail = g.m * g.n - g.q * g.r_dim;
    if (tail > 0) DT_CUDA_CHECK(cudaMemsetAsync(dv + g.q * g.r_dim, 0, (size_t)tail * 4, st));
  }
  {
    XGemm d = gemm_gdxf(g);
    d.A = dv; d.lda = g.n;
    d.B = wf; d.ldb = g.n;
    d.out = d_xf; d.ldo = g.rank;
    d.part = part;
    if (int rc = xgemm(d, st)) return rc;
  }
  {
    XGemm d = gemm_gdwf(g);
    d.A = dv; d.lda = g.n;
    d.B = xf; d.ldb = g.rank;
    d.out = d_wf; d.ldo = g.n;
    d.part = part;
    if (int rc = xgemm(d, st)) return rc;
  }
  if (d_input) {
    float *w = reinterpret_cast<float *>(ws + L.w);
    if (int rc = launch_decompress(g, xf, wf, w, st)) return rc;
    XGemm d = gemm_gdin(g, batch);
    d.A = gp; d.lda = g.r_dim;
    d.B = w; d.ldb = g.r_dim;
    d.out = d_input; d.ldo = g.q;
    d.part = part;
    if (int rc = xgemm(d, st)) return rc;
  }
  return DT_OK;
}

}  // namespace dt
