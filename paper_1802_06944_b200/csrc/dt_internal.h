// Internal declarations shared by the C-ABI translation unit and the kernel files.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>

#include "../../include/deepthin_b200.h"

namespace dt {

// Thread-local error message behind dt_last_error().
void set_error(const std::string &msg);

// ---- geometry -------------------------------------------------------------
struct Geo {
  int64_t q, r_dim, rank, m, n;
  int64_t period, phase_count, rows_per_period, tail;
  bool reuse;
  int64_t s;  // q / n on the reuse path
};
int make_geo(const dt_plan *plan, Geo *g);

// ---- fp32 CUDA-core (FFMA) path: k_simt.cu -----------------------------------
int ffma_forward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                 const float *wf, const float *bias, int act, float act_arg, void *y,
                 int y_dtype, char *ws, size_t ws_bytes, cudaStream_t st);
size_t ffma_forward_ws(const Geo &g, int64_t batch);
int ffma_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                  const float *wf, const float *bias, int act, float act_arg,
                  const float *upstream, float *d_xf, float *d_wf, float *d_bias,
                  float *d_input, char *ws, size_t ws_bytes, cudaStream_t st);
size_t ffma_backward_ws(const Geo &g, int64_t batch);

int launch_decompress(const Geo &g, const float *xf, const float *wf, float *w, cudaStream_t st);
int launch_cast_bf16(int64_t count, const float *src, uint16_t *dst, cudaStream_t st);
int launch_row_softmax(int64_t rows, int64_t cols, void *y, int y_dtype, cudaStream_t st);
int launch_mse_grad(int64_t rows, int64_t cols, const float *y, const float *t, double norm,
                    float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st);
size_t mse_ws(int64_t rows, int64_t cols);
int launch_sgd(int64_t count, float *p, const float *g, float lr, cudaStream_t st);
// config-4 recurrent step: the four H -> H reuse-geometry gate contractions of h (fp32, exact)
bool lstm_gates_ok(const Geo &g);
size_t lstm_gates_ws(const Geo &g, int64_t batch);
int lstm_gates(const Geo &g, int64_t batch, const float *h, const float *const *xf,
               const float *const *wf, const float *const *bias, float *const *gh, char *ws,
               cudaStream_t st);
// the whole recurrence (T steps, batch <= 64) in one cooperative persistent kernel
bool lstm_seq_ok(const Geo &g, int64_t batch);
size_t lstm_seq_ws(const Geo &g, int64_t batch);
int lstm_seq(const Geo &g, int64_t T, int64_t batch, const void *const *gx, const float *const *xf,
             const float *const *wf, const float *const *bias, void *out, char *ws, cudaStream_t st);
int launch_lstm_cell(int64_t batch, int64_t hidden, const void *const *gx, int64_t ld_gx,
                     const float *const *gh, float *c, float *h32, void *h16, cudaStream_t st);
int launch_act_grad(int64_t count, const float *up, const float *pre, int act, float act_arg,
                    float *out, cudaStream_t st);
// fixed-order column sums of a rows x cols fp32 matrix (partials in `part`, colsum_ws bytes)
size_t colsum_ws(int64_t rows, int64_t cols);
int launch_colsum(int64_t rows, int64_t cols, const float *g, float *out, float *part,
                  cudaStream_t st);

// ---- tcgen05 tensor-core path: k_tc_general.cu ---------------------------------
// `packed` (nullable): regeneration operands from tc_general_pack; else packed into ws.
int tc_general_forward(const Geo &g, int64_t batch, const void *x, int x_dtype,
                       const uint16_t *xf_bf16, const uint16_t *wf_bf16, const void *packed,
                       const float *bias, int act, float act_arg, void *y, int y_dtype, char *ws,
                       size_t ws_bytes, cudaStream_t st);
size_t tc_general_ws(const Geo &g, int64_t batch);
size_t tc_general_packed_bytes(const Geo &g);
int tc_general_pack(const Geo &g, const uint16_t *xf_bf16, const uint16_t *wf_bf16, void *packed,
                    cudaStream_t st);

// x (fp32 or bf16, pitch q) -> bf16 with pitch ldx (>= q, zero padded), for TMA.
int launch_pack_x(int64_t batch, int64_t q, int64_t ldx, const void *x, int x_dtype, void *out,
                  cudaStream_t st);
// 2-D tiled tensor map (dtype DT_BF16 / DT_F32), optional 128-byte swizzle.
int encode_tensor_map_2d(CUtensorMap *tm, int dtype, void *base, uint64_t inner, uint64_t outer,
                         uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                         bool swizzle128);
// ... with an explicit CUtensorMapSwizzle mode (e.g. CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, the
// layout tcgen05 requires for MN-major tf32 operands)
int encode_tensor_map_mn3d(CUtensorMap *tm, int dtype, void *base, uint64_t mn, uint64_t k,
                           uint64_t pitch_bytes, uint32_t bk, uint32_t nchunks, int swizzle);
int encode_tensor_map_2d_sw(CUtensorMap *tm, int dtype, void *base, uint64_t inner, uint64_t outer,
                            uint64_t pitch_bytes, uint32_t box_inner, uint32_t box_outer,
                            int swizzle);

// ---- row-tile tensor-core forward for reuse geometries: k_tc_rows.cu ------------------
// One persistent kernel: P = x_seg @ wf^T (bf16, TMEM) -> tf32 A operand -> y = act(P XF2^T + b),
// TMA-stored. A prep kernel writes the bf16 wf and the K-padded XF2 into ws (tc_rows_ws bytes).
// Softmax is not fused (caller post-pass).
bool tc_rows_ok(const Geo &g, int x_dtype, int y_dtype);
size_t tc_rows_ws(const Geo &g);
// prepared: ws already holds the operands tc_rows_prepare derived (same bias / act / y_dtype)
int tc_rows_forward(const Geo &g, int64_t batch, const void *x, const float *wf, const float *xf,
                    const float *bias, int act, float act_arg, void *y, int y_dtype, char *ws,
                    cudaStream_t st, bool prepared = false);
// Row-slab variant (k_tc_slab.cu): no clusters, every CTA a contiguous slab of batch rows, x
// viewed (batch * s) x n so one UMMA covers whole batch rows; same prepared operands (wf16 /
// xf2p / bslot as tc_rows_prepare lays them out). Dispatched from tc_rows_forward.
bool tc_slab_ok(const Geo &g, int64_t batch, int softmax);
int tc_slab_forward(const Geo &g, int64_t batch, const void *x, const void *wf16, const void *xf2p,
                    const float *bias, int bslot, int act, float act_arg, void *y, int y_dtype,
                    cudaStream_t st);
// Fused layer chain (k_tc_chain.cu): L reuse layers sharing n, s and rank in one persistent
// kernel; hidden activations stay in shared memory. prepared[l]: tc_rows_prepare output of layer
// l (hidden layers with hidden_act / bf16 output, the last with identity / bf16 output).
bool tc_chain_ok(const Geo *g, int L);
int tc_chain_forward(const Geo *g, int L, int64_t batch, const void *x, void *const *prepared,
                     int hidden_act, float act_arg, void *y, cudaStream_t st);
// Low-rank straddling layers as the reference's memoized runs (k_tc_runs.cu): bf16 in / out,
// P' = x . Wruns^T (wf hi + lo), y = act(P' . XFfull^T + b); W never exists.
bool tc_runs_ok(const Geo &g, int x_dtype, int y_dtype);
// dt_forward_path for the two-phase entry (tc_forward_impl's own choice, aligned operands)
int tc_forward_path(const Geo &g, int x_dtype, int f_dtype, int y_dtype);
size_t tc_runs_ws(const Geo &g);
int tc_runs_forward(const Geo &g, int64_t batch, const void *x, const float *wf, const float *xf,
                    const float *bias, int act, float act_arg, void *y, char *ws, cudaStream_t st);
// layer chaining for the next tc_rows_forward on this thread (prepared operands only)
void rows_chain(const unsigned *wait, unsigned target, unsigned *post);
int rows_posts_per_tile(const Geo &g);
int tc_rows_prepare(const Geo &g, const float *wf, const float *xf, const float *bias, int act,
                    int y_dtype, char *ws, cudaStream_t st);

// ---- any-major tcgen05 GEMM on CTA pairs: k_tc_xgemm.cu ------------------------------------
// D[M x N] = sum_k A(m, k) B(n, k); A stored K-major (A[m*lda + k]) or MN-major (A[k*lda + m]),
// B likewise; tf32 (el = 1, fp32 in memory) or bf16 (el = 0). Epilogue `epi`: 0 store
// (alpha * D + bias[n]), 1 fused MSE gradient, 2 hi + lo column-half sum, 3 H -> [hi | lo]
// bf16 re-laid rows. splits > 1 (or a transposed / column-paired result, store epilogue
// only): partial slices into `part` (xgemm_ws bytes), then a fixed-order sum into out.
struct XGemm {
  int64_t M = 0, N = 0, K = 0;
  const void *A = nullptr;
  int64_t lda = 0;
  int a_mn = 0;
  const void *B = nullptr;
  int64_t ldb = 0;
  int b_mn = 0;
  int64_t b_wrap_k = 0;  // > 0: B's rows (K) wrap modulo this (A = [hi; lo] stacked along K)
  int64_t b_rows = 0;    // K extent B actually stores (zero fill past it; with b_wrap_k: < wrap)
  int force_part = 0;    // result through the partial buffer + reduce (any output pitch)
  int el = 1;
  int BN = 256;
  int splits = 1;
  float *part = nullptr;
  int reduce_transpose = 0, reduce_pair_half = 0;
  int epi = 0;
  float *out = nullptr;
  int64_t ldo = 0;
  float alpha = 1.f;
  const float *bias = nullptr;
  const float *target = nullptr;  // epi 1
  int64_t ldt = 0;
  float scale = 1.f;
  double *loss_part = nullptr;
  int64_t *n_loss_part = nullptr;
  float *colsum_part = nullptr;   // epi 1: [2 * ceil(M / 256)][N]
  __nv_bfloat16 *out16 = nullptr; // epi 3
  int h_r = 0, h_s = 0;
  int pair_half = 0;              // epi 2
  int ks_major = 0;               // units ordered with the K split slowest (operand reuse in L2)
  // epi 4 (transposed store): out_t[n][m] = act(D[m][n] + bias[m]), y_dtype DT_F32 / DT_BF16
  void *out_t = nullptr;
  int y_dtype = DT_F32, act = DT_ACT_IDENTITY;
  float act_arg = 0.f;
  int chain = 0;                  // pipelined forward (PDL trigger after the prologue)
  // > 0: every stage also multiplies A at K offset dual_k (a K-major A whose rows hold two
  // halves, e.g. [W_hi | W_lo]) by the same B tile; K is then the length of ONE half
  int64_t dual_k = 0;
};
size_t xgemm_ws(const XGemm &g);
int xgemm_splits(int64_t M, int64_t N, int64_t K, int BN, int el, int nsm);
int xgemm(const XGemm &g, cudaStream_t st);
// fixed-order reductions of XE_MSE's partials (scratch: xgemm_reduce_scratch bytes)
size_t xgemm_reduce_scratch(int rows, int64_t N);
int xgemm_colsum(int rows, int64_t N, const float *part, float *out, void *scratch, cudaStream_t st);
int xgemm_sum_f64(int64_t count, const double *part, double *out, void *scratch, cudaStream_t st);

// ---- tensor-core training step of reuse geometries: k_train.cu -------------------------------
bool xtrain_ok(const Geo &g);
size_t xtrain_forward_mse_ws(const Geo &g, int64_t batch);
int xtrain_forward_mse(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                       const float *wf, const float *bias, const float *target, double scale,
                       float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st,
                       float *d_bias, float *p_out);
size_t xtrain_backward_ws(const Geo &g, int64_t batch);
int xtrain_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                    const float *wf, const float *bias, int act, float act_arg, const float *up,
                    float *d_xf, float *d_wf, float *d_bias, float *d_input, char *ws,
                    size_t ws_bytes, cudaStream_t st, const float *p_in);
// general (straddling) geometries: d_W^T = g^T x on tcgen05 (bf16 x, g hi | lo), the flat
// inverse re-layout as a view, then d_xf / d_wf / d_input as tf32 GEMMs (k_train.cu)
bool xback_general_ok(const Geo &g);
size_t xback_general_ws(const Geo &g, int64_t batch);
int xback_general(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                  const float *wf, const float *bias, int act, float act_arg, const float *up,
                  float *d_xf, float *d_wf, float *d_bias, float *d_input, char *ws,
                  size_t ws_bytes, cudaStream_t st);

// ---- two-phase tensor-core path: k_tc_gemm.cu ---------------------------------------
// W^T (r_dim x round_up(q, 8), bf16) regenerated from the factors (f_dtype DT_F32 or DT_BF16)
// into the workspace, then a persistent tcgen05 GEMM y = act(x W + bias). Any geometry.
int tc_gemm_forward(const Geo &g, int64_t batch, const void *x, int x_dtype, const void *xf,
                    const void *wf, int f_dtype, const float *bias, int act, float act_arg,
                    void *y, int y_dtype, char *ws, size_t ws_bytes, cudaStream_t st);
size_t tc_gemm_ws(const Geo &g, int64_t batch);
// Forward with the MSE gradient fused into the final GEMM's epilogue (identity activation):
// grad = scale * (x W + b - target), loss_sum = fixed-order fp64 sum of squared errors.
int tc_forward_mse(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                   const float *wf, const float *bias, const float *target, double scale,
                   float *grad, double *loss_sum, char *ws, size_t ws_bytes, cudaStream_t st,
                   float *d_bias = nullptr, float *p_out = nullptr);
size_t tc_forward_mse_ws(const Geo &g, int64_t batch);
int launch_sum_f64(int64_t count, const double *part, double *out, cudaStream_t st);
// fixed-order fp64 sum of (g * inv)^2 (part: mse_ws(1, count) bytes), out nullable
// one pass over g (rows x cols): column sums into out (fixed order) and sum (g*inv)^2 into loss
int launch_colsum_sumsq(int64_t rows, int64_t cols, const float *g, double inv, float *out,
                        float *cpart, double *sq_part, double *loss, cudaStream_t st);
int launch_sumsq(int64_t count, const float *g, double inv, double *part, double *out, cudaStream_t st);
// Tensor-core backward of reuse geometries in factored form (cuBLASLt for the plain GEMMs over
// transposed views); returns DT_E_UNSUPPORTED when the geometry does not qualify.
bool tc_backward_ok(const Geo &g);
int tc_backward(const Geo &g, int64_t batch, const void *x, int x_dtype, const float *xf,
                const float *wf, const float *bias, int act, float act_arg,
                const float *upstream, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                char *ws, size_t ws_bytes, cudaStream_t st, const float *p_in = nullptr);
size_t tc_backward_ws(const Geo &g, int64_t batch);

// dt_profile_kernel_events: events to record around the next dominant-kernel launch on this
// thread (both null when disarmed / exhausted).
void profile_next(cudaEvent_t *before, cudaEvent_t *after, int kind);
// dt_set_forward_pipeline state of this thread.
bool forward_pipeline();
bool forward_pipeline_external_x();
// records (once) the event set by dt_set_backward_event on st; no-op when none is pending
int backward_event_record(cudaStream_t st);

// Raise fn's dynamic shared-memory limit to at least `bytes` on the CURRENT device (function
// attributes are per device context: a process driving several GPUs sets them on each).
// Cached per (device, fn), thread-safe.
int set_smem_limit(const void *fn, int bytes);
// Ask for the maximum shared-memory carveout for fn on the current device (once per (device,
// fn)): a small kernel meant to run on the same SMs as a large-shared-memory one.
int prefer_max_smem_carveout(const void *fn);
// Allow non-portable cluster sizes for fn on the current device (once per (device, fn)).
int allow_nonportable_clusters(const void *fn);

// Timing-experiment switches (DEEPTHIN_DBG_*, DEEPTHIN_*_TRACE, DEEPTHIN_REGEN_SERIAL): some
// drop work (stores, loads, a phase) and produce wrong outputs, so they exist only in builds
// made with -DDEEPTHIN_TIMING_SWITCHES (python -m paper_1802_06944_b200.build --timing). The
// product library reads none of them: DT_DBG_ENV is the constant 0 there.
#ifdef DEEPTHIN_TIMING_SWITCHES
#define DT_DBG_ENV(name) (getenv(name) ? atoi(getenv(name)) : 0)
constexpr bool kTimingSwitches = true;
#else
#define DT_DBG_ENV(name) 0
constexpr bool kTimingSwitches = false;
#endif

// Every kernel launch goes through check_launch, which also counts it (dt_launch_counter).
int check_launch(const char *what);
int64_t launch_count();

}  // namespace dt

#define DT_CUDA_CHECK(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      dt::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));           \
      return DT_E_CUDA;                                                            \
    }                                                                              \
  } while (0)
