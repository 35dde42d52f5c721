/*
 * deepthin_b200.h — C ABI of the B200-native DeepThin compressed-layer hot path.
 *
 * Notation is the reference's (deepthin, /root/reference/pkg/src/deepthin):
 * a layer maps q inputs to r_dim outputs; its weight W (q x r_dim) is the
 * column-major refill of v = (xf @ wf).ravel() with xf m x rank and wf
 * rank x n (factor.py:1-9, 87-93). The trailing m*n - q*r_dim elements of v
 * are discarded. y = x @ W + bias.
 *
 * Conventions
 *  - Every device pointer is caller-owned (PyTorch allocates). Calls are
 *    stream-ordered and asynchronous; none synchronises the host except the
 *    dt_session_* host-buffer entry points.
 *  - Matrices are dense row-major with the leading dimension equal to the
 *    row length (x: batch x q, y: batch x r_dim, xf: m x rank, wf: rank x n).
 *  - Return value is a dt_status; on failure dt_last_error() holds a
 *    thread-local message. The Python shim maps DT_E_DIM → DimensionError,
 *    DT_E_ARG → ArgumentError, DT_E_UNSUPPORTED → UnsupportedConfigurationError
 *    (deepthin/errors.py:10-31), DT_E_CUDA → RuntimeError.
 *  - Results are deterministic: no float atomics; every reduction has a
 *    fixed order independent of launch geometry (kernel.py:264-266 analogue).
 */
#ifndef DEEPTHIN_B200_H
#define DEEPTHIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *dt_stream; /* == cudaStream_t; NULL = legacy default stream */

/* Geometry of one compressed matrix — replaces planner.py:27-60 LayerPlan
 * (q, r_dim, rank, m, n; validation m*n >= q*r_dim, all >= 1). */
typedef struct {
  int64_t q, r_dim, rank, m, n;
} dt_plan;

/* Derived geometry (factor.py:96-110, kernel.py:99-149). */
typedef struct {
  int64_t period;      /* n / gcd(n, q): columns per phase cycle            */
  int64_t phase_count; /* min(period, r_dim)              (factor.py:108)   */
  int64_t reuse;       /* 1 iff n | q: the factored-reuse path (a)          */
  int64_t segments;    /* q / n on the reuse path, else 0                   */
  int64_t tail;        /* m*n - q*r_dim discarded aux elements              */
  int64_t rows_per_period; /* q / gcd(n, q): aux rows advanced per period   */
} dt_plan_info;

enum dt_status {
  DT_OK = 0,
  DT_E_DIM = 1,         /* DimensionError                  */
  DT_E_ARG = 2,         /* ArgumentError                   */
  DT_E_UNSUPPORTED = 3, /* UnsupportedConfigurationError   */
  DT_E_CUDA = 4,        /* CUDA launch / runtime failure   */
  DT_E_FORMAT = 5       /* ModelFormatError (dt_model_parse; details in dt_format_error) */
};

/* DT_FACTORS_PACKED is valid only as dt_forward's f_dtype: xf points at the buffer
 * dt_pack_factors filled (wf is ignored). */
enum dt_dtype { DT_F32 = 0, DT_BF16 = 1, DT_FACTORS_PACKED = 2, DT_F64 = 3 /* dt_unpack_values */,
               DT_FACTORS_ROWS = 4 /* dt_rows_prepare output, dt_forward f_dtype */ };

/* Arithmetic of the contraction.
 *  DT_MMA_FFMA: fp32 CUDA-core FFMA, fp32 operands (parity rtol 1e-5).
 *  DT_MMA_BF16: tcgen05 kind::f16 tensor cores, bf16 operands, fp32 accumulate;
 *               reuse-path partials stay fp32 (tf32 MMA) (parity rtol 2e-3).  */
enum dt_mma { DT_MMA_FFMA = 0, DT_MMA_BF16 = 1 };

/* kernel.py:39-48 (+ clipped ReLU and row softmax, used by BASELINE configs 3/4). */
enum dt_act {
  DT_ACT_IDENTITY = 0,
  DT_ACT_RELU = 1,
  DT_ACT_SIGMOID = 2,
  DT_ACT_TANH = 3,
  DT_ACT_CLIPPED_RELU = 4, /* min(max(z, 0), act_arg) */
  DT_ACT_SOFTMAX = 5       /* row softmax (forward only) */
};

const char *dt_version(void);
/* Thread-local message of the last failing call on this thread. */
const char *dt_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
int64_t dt_launch_counter(void);
/* Profiling hook (this thread): the next n launches of the forward's dominant kernel (the
 * tcgen05 GEMM of the bf16 path; the whole FFMA forward on the fp32 path) are bracketed by
 * cudaEventRecord(before[i]) / cudaEventRecord(after[i]) on their stream. n = 0 disarms.
 * Events are cudaEvent_t handles created by the caller. No reference counterpart: used by
 * bench.py for the roofline of the dominant kernel. */
int dt_profile_kernel_events(void *const *before, void *const *after, int n);
/* Which launches dt_profile_kernel_events brackets (this thread): DT_PROF_ANY (default), the
 * two-phase GEMM / FFMA forward (DT_PROF_GEMM), or the row-tile reuse kernel (DT_PROF_ROWS). */
enum { DT_PROF_ANY = 0, DT_PROF_GEMM = 1, DT_PROF_ROWS = 2 };
int dt_profile_kernel_kind(int kind);
/* Inference pipelining (this thread): with enable = 1, consecutive bf16 tensor-core forwards
 * on one stream overlap each call's W regeneration with the previous call's GEMM (programmatic
 * dependent launch; W^T alternates between two workspace slots). The caller promises that the
 * factor buffers are not written while pipelined calls are in flight on the stream (a forward
 * never waits for a factor update launched after the previous forward). Every call still
 * regenerates its own W^T. Default 0. No reference counterpart (kernel.py has no pipelining).
 * Mode 1 makes no promise about x: a call whose x is the previous call's output (a layer chain)
 * waits for that call before loading x. Mode DT_PIPELINE_EXTERNAL_X also promises that no x
 * is written by a call still in flight (independent inputs), so each call's first x stages load
 * while the previous call is still running. */
enum { DT_PIPELINE_OFF = 0, DT_PIPELINE_ON = 1, DT_PIPELINE_EXTERNAL_X = 2 };
int dt_set_forward_pipeline(int enable);

/* ---- geometry (host-only, no GPU needed) ---------------------------------- */
/* planner.py:38-47 LayerPlan.__post_init__ validation. */
int dt_plan_validate(const dt_plan *plan);
int dt_plan_query(const dt_plan *plan, dt_plan_info *info);
/* factor.py:96-105 phase(col, plan). */
int dt_phase(const dt_plan *plan, int64_t col, int64_t *out_phase);
/* factor.py:74-84 relayout_index(flat, plan). */
int dt_relayout_index(const dt_plan *plan, int64_t flat, int64_t *row, int64_t *col);
/* kernel.py:184-205 predict_reuse(plan, batch): per-row distinct / total runs. */
int dt_predict_reuse(const dt_plan *plan, int64_t batch, int64_t *distinct_runs,
                     int64_t *total_runs);
/* kernel.py:277-280 OpCount of the run-memoized algorithm over `batch` rows. */
int dt_op_count(const dt_plan *plan, int64_t batch, int64_t *multiplies, int64_t *adds);

/* ---- device compute --------------------------------------------------------- */
/* Replaces factor.py:87-93 decompress(fp): W (q x r_dim, row-major fp32). */
int dt_decompress(const dt_plan *plan, const float *xf, const float *wf, float *w,
                  dt_stream stream);

/* Round fp32 → bf16 (RNE); used to make the bf16 operand copies of factors. */
int dt_cast_bf16(int64_t count, const float *src, uint16_t *dst, dt_stream stream);

/* Derived per-pair operand layout for the bf16 tensor-core path (the analogue of the
 * reference's per-pair cached combine weights, kernel.py:157-164): bf16 factors
 * re-laid into the on-chip regeneration operands' core-matrix order, zero padded.
 * Build once per factor update; pass to dt_forward with f_dtype = DT_FACTORS_PACKED.
 * Returns 0 bytes for plans the tensor-core path does not support. */
size_t dt_packed_factors_bytes(const dt_plan *plan, int mma);
int dt_pack_factors(const dt_plan *plan, int mma, const uint16_t *xf_bf16,
                    const uint16_t *wf_bf16, void *packed, dt_stream stream);

size_t dt_forward_workspace_bytes(const dt_plan *plan, int64_t batch, int mma);

/* Replaces kernel.py:222-293 fused_matmul and kernel.py:296-320 layer_forward:
 * y = act(x @ W + bias) without materialising W.
 *   x      batch x q, dtype x_dtype (DT_F32 or DT_BF16)
 *   xf, wf fp32 masters (DT_MMA_FFMA) or bf16 copies (DT_MMA_BF16): f_dtype
 *   bias   r_dim fp32, nullable (= zero)
 *   y      batch x r_dim, dtype y_dtype
 * Reuse path (n | q) and general path (straddling rows) are chosen from the plan. */
int dt_forward(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
               const void *xf, const void *wf, int f_dtype, const float *bias, int act,
               float act_arg, void *y, int y_dtype, void *workspace, size_t workspace_bytes,
               dt_stream stream);

/* Which kernel family dt_forward takes for (plan, mma, x/f/y dtypes) with 16-byte-aligned
 * operands (misaligned pointers fall back to the staged two-phase forms). Each family states its
 * own arithmetic contract; tests pick the matching emulation from it.
 * Returns a DT_PATH_* value, or a negative dt_status on a bad plan / argument. */
enum dt_path {
  DT_PATH_FFMA = 1,     /* fp32 FFMA                                               */
  DT_PATH_ROWS = 2,     /* one-kernel row-tile reuse form (k_tc_rows.cu)           */
  DT_PATH_FACTORED = 3, /* factored reuse, two GEMMs (P = x wf^T, y = P XF2^T)     */
  DT_PATH_RUNS = 4,     /* memoized runs, low-rank straddling layers (k_tc_runs.cu) */
  DT_PATH_HILO = 5,     /* two-phase, W^T as bf16 hi + lo (fp32 outputs)           */
  DT_PATH_PAIR = 6,     /* two-phase, W^T rounded once to bf16                     */
  DT_PATH_FUSED = 7     /* single kernel, W regenerated in-kernel (packed factors) */
};
int dt_forward_path(const dt_plan *plan, int mma, int x_dtype, int f_dtype, int y_dtype);

size_t dt_backward_workspace_bytes(const dt_plan *plan, int64_t batch, int mma);

/* Replaces grad.py:63-95 layer_backward: gradients through activation, bias,
 * the contraction, the inverse re-layout (tail gets zero) and the factor product.
 *   upstream batch x r_dim fp32 (dLoss/dy)
 *   d_xf m x rank, d_wf rank x n, d_bias r_dim fp32 (d_bias nullable)
 *   d_input batch x q fp32, nullable (skipped)
 * Pre-activations are recomputed (grad.py:81-83) unless act == IDENTITY. */
int dt_backward(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
                const float *xf, const float *wf, const float *bias, int act, float act_arg,
                const float *upstream, float *d_xf, float *d_wf, float *d_bias,
                float *d_input, void *workspace, size_t workspace_bytes, dt_stream stream);
/* dt_backward with p_in (nullable): the P that dt_forward_mse_ex kept for these x and factors
 * (tensor-core backward of reuse geometries only). d_bias may be NULL to skip the column sums
 * (already produced by dt_forward_mse_ex). */
int dt_backward_ex(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
                   const float *xf, const float *wf, const float *bias, int act, float act_arg,
                   const float *upstream, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                   const float *p_in, void *workspace, size_t workspace_bytes, dt_stream stream);

/* grad.py:98-103 loss_and_grad("mse") for one shard of rows:
 *   grad = 2 (y - t) / norm_count;  loss_sum[0] = sum (y - t)^2  (fp64, fixed order).
 * norm_count is the GLOBAL y.size when the batch is sharded across ranks. */
int dt_mse_grad(int64_t rows, int64_t cols, const float *y, const float *target,
                double norm_count, float *grad, double *loss_sum, void *workspace,
                size_t workspace_bytes, dt_stream stream);
size_t dt_mse_workspace_bytes(int64_t rows, int64_t cols);

/* Fused forward + MSE gradient, identity activation (grad.py:98-103 applied to
 * kernel.py:296-320's output without materialising y): grad = 2 (x W + b - target) /
 * norm_count (fp32, batch x r_dim) and loss_sum[0] = sum (y - target)^2 (fp64, fixed order).
 * bf16 tensor-core path (x bf16 or fp32, fp32 factors); the MSE runs in the final GEMM's
 * epilogue. */
size_t dt_forward_mse_workspace_bytes(const dt_plan *plan, int64_t batch);
int dt_forward_mse(const dt_plan *plan, int64_t batch, const void *x, int x_dtype, const float *xf,
                   const float *wf, const float *bias, const float *target, double norm_count,
                   float *grad, double *loss_sum, void *workspace, size_t workspace_bytes,
                   dt_stream stream);
/* dt_forward_mse plus two outputs for the step that follows (both nullable):
 *   d_bias (r_dim fp32): the column sums of grad (grad.py:85), computed in the loss pass;
 *   p_out (dt_forward_p_bytes bytes, reuse geometries only): the factored forward's
 *     P = x.view(B*s, n) @ wf^T (fp32), for dt_backward_ex to reuse instead of recomputing. */
size_t dt_forward_p_bytes(const dt_plan *plan, int64_t batch);
int dt_forward_mse_ex(const dt_plan *plan, int64_t batch, const void *x, int x_dtype,
                      const float *xf, const float *wf, const float *bias, const float *target,
                      double norm_count, float *grad, double *loss_sum, float *d_bias,
                      float *p_out, void *workspace, size_t workspace_bytes, dt_stream stream);

/* A run of consecutive reuse layers of a network (model_io.py:46-63 CompressedModel, each layer
 * kernel.py:296-320 layer_forward) fused into ONE persistent kernel: every 128-row tile goes
 * through all n_layers layers with the hidden activations kept in shared memory (only the run's
 * input and its last layer's output touch HBM). Eligible: n_layers in [2, 8], every plan a reuse
 * geometry taking the row-tile kernel (dt_rows_prepared_bytes > 0 with bf16 x and y), all sharing
 * n, rank and q/n, plans[l].q == plans[l-1].r_dim (dt_chain_ok). x: batch x plans[0].q bf16; y:
 * batch x plans[n_layers-1].r_dim bf16. prepared[l]: dt_rows_prepare of layer l with hidden_act
 * (l < n_layers-1) or DT_ACT_IDENTITY (the last layer), y_dtype DT_BF16, and the layer's bias.
 * last_act: DT_ACT_IDENTITY, or DT_ACT_SOFTMAX (a row softmax over y after the chain). */
int dt_chain_ok(const dt_plan *plans, int n_layers);
int dt_chain_forward(const dt_plan *plans, int n_layers, int64_t batch, const void *x,
                     void *const *prepared, int hidden_act, float act_arg, int last_act, void *y,
                     dt_stream stream);

/* core.py:63-77 matmul (np.matmul after as_matrix) on the tensor cores, for the transposed views
 * the backward contracts (grad.py:86-94): c (M x N fp32, pitch ldc) = op(a) @ op(b), op(a) M x K,
 * op(b) K x N. a_trans = 0: a stored M x K (pitch lda); 1: a stored K x M. b_trans = 0: b stored
 * K x N (pitch ldb); 1: b stored N x K. dtype DT_F32 (tf32 products, fp32 accumulate) or DT_BF16
 * (bf16 products, fp32 accumulate). Pitches are in elements and 16-byte aligned. The transposed
 * orders need no copy (tcgen05 reads either major order). Deterministic: split-K partials are
 * summed in a fixed order. */
size_t dt_matmul_workspace_bytes(int64_t M, int64_t N, int64_t K, int dtype);
int dt_matmul(int64_t M, int64_t N, int64_t K, const void *a, int64_t lda, int a_trans,
              const void *b, int64_t ldb, int b_trans, int dtype, float *c, int64_t ldc,
              void *workspace, size_t workspace_bytes, dt_stream stream);

/* Data-parallel overlap hook (this thread): the next dt_backward / dt_backward_ex records
 * `event` (a cudaEvent_t) on its stream as soon as d_xf and d_bias are final — on the
 * tensor-core path right after d_xf's GEMM, before H and d_wf — so a caller can start their
 * all-reduce on another stream while the backward still runs; at the latest when the call's
 * work is enqueued. One-shot. No reference counterpart (the reference is single-process). */
int dt_set_backward_event(void *event);

/* train.py:107-111 DeepThinWeights.step: param -= lr * grad (fp32 masters). */
int dt_sgd_step(int64_t count, float *param, const float *grad, float lr, dt_stream stream);
/* Row-tile reuse kernel operands derived once per factor pair (the analogue of the reference's
 * per-pair derived-weight cache, kernel.py:157-164): bf16 wf and the K-padded XF2 with the bias
 * and the bf16-sigmoid pre-scale folded in. dt_rows_prepared_bytes returns 0 when the geometry
 * (n_f | q, n_f % 64 == 0, s * round_up(rank, 4) <= 32) or the dtypes do not take that kernel.
 * Pass the buffer to dt_forward as xf with f_dtype = DT_FACTORS_ROWS (wf ignored) and the SAME
 * act, y_dtype and bias as here; rebuild it after the factors or the bias change. */
size_t dt_rows_prepared_bytes(const dt_plan *plan, int x_dtype, int y_dtype);
int dt_rows_prepare(const dt_plan *plan, int act, int y_dtype, const float *xf, const float *wf,
                    const float *bias, void *out, dt_stream stream);
/* Layer chaining of consecutive row-tile layers (this thread, the NEXT dt_forward with
 * DT_FACTORS_ROWS only): instead of waiting for the whole previous kernel, the launch loads
 * 128-row tile t of x once ((unsigned *)wait_flags)[t] >= wait_target, and its epilogue warps
 * add 1 to ((unsigned *)post_flags)[t] (release) after storing their part of tile t —
 * dt_rows_posts_per_tile(plan) additions per tile per launch. wait_flags / post_flags may be
 * NULL. The caller keeps the flags monotone across calls (targets grow by the producer's posts
 * per tile each forward) and must not let a layer write a buffer that an earlier, still
 * running layer reads in rows it has not finished (three rotating activation buffers). */
int dt_rows_chain(const void *wait_flags, unsigned wait_target, void *post_flags);
int dt_rows_posts_per_tile(const dt_plan *plan);
/* The four recurrent gate contractions of one LSTM step (BASELINE config 4): gh[g] = h @ W_g +
 * bias[g] for four DeepThin layers sharing one square reuse geometry (plan: q == r_dim, n | q),
 * h fp32 (batch x q), 3xTF32 tensor-core tiles (~fp32 accuracy, fixed order) in the reference's factored reuse form
 * (kernel.py:1-16, 296-320). xf/wf/bias/gh: four pointers each (bias may be NULL). */
size_t dt_lstm_gates_workspace_bytes(const dt_plan *plan, int64_t batch);
int dt_lstm_gates(const dt_plan *plan, int64_t batch, const float *h, const float *const *xf,
                  const float *const *wf, const float *const *bias, float *const *gh,
                  void *workspace, size_t workspace_bytes, dt_stream stream);
/* The whole LSTM recurrence of BASELINE config 4 in one persistent cooperative kernel: for
 * t < T, gates = gx[g][t] + h_{t-1} @ W_g + bias[g] (the dt_lstm_gates contractions, 3xTF32 ~fp32),
 * then the dt_lstm_cell update; h_{-1} = c_{-1} = 0. gx[g]: bf16, T*batch x q (time-major rows);
 * out: bf16 T*batch x q (the h sequence). batch <= 64. */
size_t dt_lstm_sequence_workspace_bytes(const dt_plan *plan, int64_t batch);
int dt_lstm_sequence(const dt_plan *plan, int64_t T, int64_t batch, const void *const *gx,
                     const float *const *xf, const float *const *wf, const float *const *bias,
                     void *out, void *workspace, size_t workspace_bytes, dt_stream stream);
/* LSTM cell step of BASELINE config 4 (no reference counterpart: SURVEY.md §8(a) a8 lists LSTM
 * gates as outside the reference). Gate order i, f, g, o; gx[g]: bf16 input projections
 * (batch rows, row stride ld_gx, biases included); gh[g]: fp32 recurrent projections (batch x
 * hidden, contiguous). c (fp32, batch x hidden) is updated in place; h32 (fp32) and/or h16
 * (bf16) receive h' = o * tanh(c'). */
int dt_lstm_cell(int64_t batch, int64_t hidden, const void *const *gx, int64_t ld_gx,
                 const float *const *gh, float *c, float *h32, void *h16, dt_stream stream);

/* ---- host-buffer entry points (the binding a numpy caller would use) -------- */
/* A session owns device-resident copies of one layer's factors and bias — the
 * analogue of FactorPair's private read-only copies (factor.py:42-50). */
typedef struct dt_session dt_session;
int dt_session_create(const dt_plan *plan, int mma, const float *xf_host, const float *wf_host,
                      const float *bias_host, dt_session **out);
/* Host x (batch x q fp32) → device, forward, device → host y (batch x r_dim
 * fp32); synchronous. Internally the rows go in chunks (DEEPTHIN_SESSION_CHUNK_ROWS, default
 * 1024) alternating between two streams, so H2D, compute and D2H of neighbouring chunks
 * overlap; pinned host buffers make the copies asynchronous. Returns the bytes moved in
 * *h2d / *d2h when non-NULL. */
int dt_session_forward(dt_session *s, int64_t batch, const float *x_host, int act,
                       float act_arg, float *y_host, int64_t *h2d_bytes, int64_t *d2h_bytes);
void dt_session_destroy(dt_session *s);

/* ---- .dthn model image (reference model_io.py:1-224) ------------------------- */
/* Host-only parse of a serialized model held in memory: validates the image exactly as
 * deserialize does (model_io.py:141-210, same checks in the same order, same failing byte
 * offsets) and indexes it in place — names, metadata strings and payloads are reported as byte
 * offsets into the image, nothing is copied. Records are written up to meta_cap / layer_cap
 * (either may be 0); hdr->meta_read / hdr->layers_read count the records the parse started,
 * including a partial one at the failure point (unread spans have length -1), so a caller
 * sizes its arrays with a first call at cap 0. Returns DT_OK, or DT_E_FORMAT with *err set. */
typedef struct { int64_t offset, length; } dt_span;
typedef struct { dt_span key, value; } dt_model_meta;
typedef struct {
  uint32_t version, layer_count;
  uint64_t payload_bytes;
  double target_ratio;
  uint32_t meta_count, reserved;
  int64_t meta_read, layers_read;
} dt_model_header;
typedef struct {
  dt_span name;
  dt_plan plan;        /* u64 fields of the file (values above INT64_MAX wrap) */
  int32_t dtype_code;  /* 0 float32, 1 float64 */
  int32_t floor_hit;
  int64_t bias_len;
  int64_t xf_offset, wf_offset, bias_offset; /* payload byte offsets into the image */
} dt_model_layer;
enum dt_format_kind {
  DT_FMT_OK = 0,
  DT_FMT_TRUNCATED = 1,        /* need/have bytes while reading `what`                 */
  DT_FMT_BAD_MAGIC = 2,
  DT_FMT_BAD_VERSION = 3,      /* need = version                                      */
  DT_FMT_PAYLOAD_MISMATCH = 4, /* need = declared payload, have = actual              */
  DT_FMT_BAD_DTYPE = 5,        /* need = code                                         */
  DT_FMT_INVALID_PLAN = 6,     /* layer = index (its plan is in the layer record)     */
  DT_FMT_TRAILING = 7          /* need = trailing byte count                          */
};
enum dt_format_what {
  DT_WHAT_HEADER = 0, DT_WHAT_META_COUNT, DT_WHAT_META_KEY_LEN, DT_WHAT_META_KEY,
  DT_WHAT_META_VALUE_LEN, DT_WHAT_META_VALUE, DT_WHAT_NAME_LEN, DT_WHAT_NAME, DT_WHAT_PLAN,
  DT_WHAT_FLAGS, DT_WHAT_BIAS_LEN, DT_WHAT_XF, DT_WHAT_WF, DT_WHAT_BIAS
};
typedef struct {
  int32_t kind, what;
  int64_t offset; /* the failing byte offset (ModelFormatError.offset) */
  int64_t layer;  /* layer (or metadata item) index, -1 when none      */
  int64_t need, have;
} dt_format_error;
int dt_model_parse(const void *image, size_t size, dt_model_header *hdr, dt_model_meta *meta,
                   int64_t meta_cap, dt_model_layer *layers, int64_t layer_cap,
                   dt_format_error *err);

/* Device-side payload decode: `count` little-endian values of src_dtype (DT_F32 / DT_F64) at
 * any byte alignment (a payload inside a device copy of the image) -> aligned fp32 `dst`
 * (float64 rounded to nearest even), plus the bf16 (RNE) copy when dst_bf16 is non-NULL. */
int dt_unpack_values(int64_t count, const void *src, int src_dtype, float *dst,
                     uint16_t *dst_bf16, dt_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* DEEPTHIN_B200_H */
