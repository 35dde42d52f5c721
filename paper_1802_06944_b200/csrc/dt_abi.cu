// extern "C" entry points of libdeepthin_b200.so (declared in include/deepthin_b200.h).
//
// Validation and error conventions mirror the reference: shape problems are
// DT_E_DIM (DimensionError), bad scalars DT_E_ARG (ArgumentError), an
// unsupported configuration DT_E_UNSUPPORTED (UnsupportedConfigurationError)
// — deepthin/errors.py:10-31, core.py:21-36, kernel.py:238-246, grad.py:74-79.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "dt_internal.h"

namespace dt {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

// planner.py:38-47 (LayerPlan.__post_init__) plus the derived geometry of
// factor.py:96-110 and kernel.py:102-106.
int make_geo(const dt_plan *plan, Geo *g) {
  if (!plan) {
    set_error("plan is NULL");
    return DT_E_ARG;
  }
  const char *names[5] = {"q", "r_dim", "rank", "m", "n"};
  const int64_t vals[5] = {plan->q, plan->r_dim, plan->rank, plan->m, plan->n};
  for (int i = 0; i < 5; ++i)
    if (vals[i] < 1) {
      set_error(std::string(names[i]) + " must be >= 1, got " + std::to_string(vals[i]));
      return DT_E_ARG;
    }
  if (plan->m * plan->n < plan->q * plan->r_dim) {
    set_error("m*n = " + std::to_string(plan->m * plan->n) + " must cover q*r_dim = " +
              std::to_string(plan->q * plan->r_dim));
    return DT_E_ARG;
  }
  g->q = plan->q;
  g->r_dim = plan->r_dim;
  g->rank = plan->rank;
  g->m = plan->m;
  g->n = plan->n;
  const int64_t gc = std::gcd(plan->n, plan->q);
  g->period = plan->n / gc;
  g->phase_count = std::min(g->period, plan->r_dim);
  g->rows_per_period = plan->q / gc;
  g->tail = plan->m * plan->n - plan->q * plan->r_dim;
  g->reuse = (plan->q % plan->n) == 0;
  g->s = g->reuse ? plan->q / plan->n : 0;
  return DT_OK;
}

}  // namespace dt

using namespace dt;

namespace {

int check_dtype(int dt, const char *what) {
  if (dt != DT_F32 && dt != DT_BF16) {
    set_error(std::string(what) + ": unknown dtype " + std::to_string(dt));
    return DT_E_ARG;
  }
  return DT_OK;
}

int check_act(int act) {
  if (act < DT_ACT_IDENTITY || act > DT_ACT_SOFTMAX) {
    set_error("unknown activation " + std::to_string(act));
    return DT_E_ARG;
  }
  return DT_OK;
}

thread_local void *const *g_prof_before = nullptr;
thread_local void *const *g_prof_after = nullptr;
thread_local int g_prof_n = 0, g_prof_used = 0, g_prof_kind = 0;
thread_local int g_pipeline = 0;

}  // namespace

void dt::profile_next(cudaEvent_t *before, cudaEvent_t *after, int kind) {
  if (g_prof_used < g_prof_n && (g_prof_kind == 0 || g_prof_kind == kind)) {
    *before = (cudaEvent_t)g_prof_before[g_prof_used];
    *after = (cudaEvent_t)g_prof_after[g_prof_used];
    ++g_prof_used;
  } else {
    *before = *after = nullptr;
  }
}

bool dt::forward_pipeline() { return g_pipeline != 0; }

namespace {
thread_local cudaEvent_t g_bwd_event = nullptr;
}  // namespace
// The backward records the pending event as soon as d_xf (and d_bias) are final, once.
int dt::backward_event_record(cudaStream_t st) {
  if (!g_bwd_event) return DT_OK;
  cudaEvent_t e = g_bwd_event;
  g_bwd_event = nullptr;
  DT_CUDA_CHECK(cudaEventRecord(e, st));
  return DT_OK;
}
bool dt::forward_pipeline_external_x() { return g_pipeline == DT_PIPELINE_EXTERNAL_X; }

extern "C" {

const char *dt_version(void) { return "deepthin_b200 0.1.0 (sm_100a)"; }

const char *dt_last_error(void) { return g_last_error.c_str(); }

int64_t dt_launch_counter(void) { return launch_count(); }

int dt_set_backward_event(void *event) {
  g_bwd_event = reinterpret_cast<cudaEvent_t>(event);
  return DT_OK;
}

int dt_set_forward_pipeline(int enable) {
  if (enable < 0 || enable > DT_PIPELINE_EXTERNAL_X) {
    set_error("dt_set_forward_pipeline: mode must be 0, 1 or DT_PIPELINE_EXTERNAL_X");
    return DT_E_ARG;
  }
  g_pipeline = enable;
  return DT_OK;
}

int dt_profile_kernel_kind(int kind) {
  if (kind < DT_PROF_ANY || kind > DT_PROF_ROWS) {
    set_error("dt_profile_kernel_kind: unknown kind " + std::to_string(kind));
    return DT_E_ARG;
  }
  g_prof_kind = kind;
  return DT_OK;
}

int dt_profile_kernel_events(void *const *before, void *const *after, int n) {
  if (n < 0 || (n > 0 && (!before || !after))) {
    set_error("dt_profile_kernel_events: n >= 0 event pairs");
    return DT_E_ARG;
  }
  g_prof_before = before;
  g_prof_after = after;
  g_prof_n = n;
  g_prof_used = 0;
  return DT_OK;
}

int dt_plan_validate(const dt_plan *plan) {
  Geo g;
  return make_geo(plan, &g);
}

int dt_plan_query(const dt_plan *plan, dt_plan_info *info) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  info->period = g.period;
  info->phase_count = g.phase_count;
  info->reuse = g.reuse ? 1 : 0;
  info->segments = g.s;
  info->tail = g.tail;
  info->rows_per_period = g.rows_per_period;
  return DT_OK;
}

int dt_phase(const dt_plan *plan, int64_t col, int64_t *out) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (col < 0 || col >= g.r_dim) {
    set_error("col " + std::to_string(col) + " out of range for r_dim " + std::to_string(g.r_dim));
    return DT_E_ARG;
  }
  *out = (col * g.q) % g.n;
  return DT_OK;
}

int dt_relayout_index(const dt_plan *plan, int64_t flat, int64_t *row, int64_t *col) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (flat < 0 || flat >= g.q * g.r_dim) {
    set_error("flat index " + std::to_string(flat) + " out of range for " + std::to_string(g.q) +
              "x" + std::to_string(g.r_dim) + " target");
    return DT_E_ARG;
  }
  *row = flat % g.q;
  *col = flat / g.q;
  return DT_OK;
}

// kernel.py:184-205: per phase slot t, runs = 1 + (p + q - 1) // n with p = t*q mod n.
int dt_predict_reuse(const dt_plan *plan, int64_t batch, int64_t *distinct, int64_t *total) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (batch < 1) {
    set_error("batch must be >= 1, got " + std::to_string(batch));
    return DT_E_ARG;
  }
  int64_t d = 0, t = 0;
  for (int64_t ph = 0; ph < g.phase_count; ++ph) {
    const int64_t p = (ph * g.q) % g.n;
    const int64_t runs = 1 + (p + g.q - 1) / g.n;
    const int64_t cols = (g.r_dim - ph + g.period - 1) / g.period;
    d += runs;
    t += runs * cols;
  }
  *distinct = d;
  *total = t;
  return DT_OK;
}

// kernel.py:277-280: multiplies = B*(sum_len + total), adds = B*(sum_len - distinct) + B*(total - r_dim)
// where sum_len is the summed length of the distinct runs (kernel.py:107-121).
int dt_op_count(const dt_plan *plan, int64_t batch, int64_t *mul, int64_t *add) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  int64_t distinct, total;
  if (int rc = dt_predict_reuse(plan, 1, &distinct, &total)) return rc;
  int64_t sum_len = 0;
  for (int64_t t = 0; t < g.phase_count; ++t) {
    const int64_t p = (t * g.q) % g.n;
    // run starts: 0, then n-p, n-p+n, ... < q; first run at wf offset p, others at 0
    const int64_t first = std::min(g.n - p, g.q);
    sum_len += first;
    for (int64_t s = g.n - p; s < g.q; s += g.n) sum_len += std::min(g.n, g.q - s);
  }
  *mul = batch * (sum_len + total);
  *add = batch * (sum_len - distinct) + batch * (total - g.r_dim);
  return DT_OK;
}

int dt_decompress(const dt_plan *plan, const float *xf, const float *wf, float *w,
                  dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  return launch_decompress(g, xf, wf, w, (cudaStream_t)stream);
}

int dt_cast_bf16(int64_t count, const float *src, uint16_t *dst, dt_stream stream) {
  if (count < 0) {
    set_error("count must be >= 0");
    return DT_E_ARG;
  }
  return launch_cast_bf16(count, src, dst, (cudaStream_t)stream);
}

size_t dt_packed_factors_bytes(const dt_plan *plan, int mma) {
  Geo g;
  if (make_geo(plan, &g) || mma != DT_MMA_BF16 || g.reuse) return 0;
  return tc_general_packed_bytes(g);
}

int dt_pack_factors(const dt_plan *plan, int mma, const uint16_t *xf_bf16,
                    const uint16_t *wf_bf16, void *packed, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (mma != DT_MMA_BF16 || g.reuse) {
    set_error("packed factors exist only for the bf16 tensor-core general path");
    return DT_E_UNSUPPORTED;
  }
  if (!xf_bf16 || !wf_bf16 || !packed) {
    set_error("NULL operand pointer");
    return DT_E_ARG;
  }
  return tc_general_pack(g, xf_bf16, wf_bf16, packed, (cudaStream_t)stream);
}

size_t dt_forward_workspace_bytes(const dt_plan *plan, int64_t batch, int mma) {
  Geo g;
  if (make_geo(plan, &g) || batch < 0) return 0;
  if (mma == DT_MMA_BF16)  // two-phase path, or the fused kernel (general geometries)
    return std::max(tc_gemm_ws(g, batch), g.reuse ? (size_t)0 : tc_general_ws(g, batch));
  return ffma_forward_ws(g, batch);
}

int dt_forward(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
               const void *xf, const void *wf, int f_dtype, const float *bias, int act,
               float act_arg, void *y, int y_dtype, void *workspace, size_t workspace_bytes,
               dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  if (int rc = check_dtype(x_dtype, "x")) return rc;
  if (int rc = check_dtype(y_dtype, "y")) return rc;
  if (f_dtype != DT_FACTORS_PACKED && f_dtype != DT_FACTORS_ROWS)
    if (int rc = check_dtype(f_dtype, "factors")) return rc;
  if (int rc = check_act(act)) return rc;
  if (batch > 0 && (!x || !xf || (!wf && f_dtype != DT_FACTORS_PACKED && f_dtype != DT_FACTORS_ROWS) || !y)) {
    set_error("NULL operand pointer");
    return DT_E_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (mma == DT_MMA_FFMA) {
    if (f_dtype != DT_F32) {
      set_error("the FFMA path takes fp32 factors");
      return DT_E_ARG;
    }
    if (batch == 0) return DT_OK;
    cudaEvent_t eb, ea;
    profile_next(&eb, &ea, DT_PROF_GEMM);
    if (eb) DT_CUDA_CHECK(cudaEventRecord(eb, st));
    int rc = ffma_forward(g, batch, x, x_dtype, (const float *)xf, (const float *)wf, bias, act,
                          act_arg, y, y_dtype, (char *)workspace, workspace_bytes, st);
    if (ea && rc == DT_OK) DT_CUDA_CHECK(cudaEventRecord(ea, st));
    return rc;
  }
  if (mma == DT_MMA_BF16 && f_dtype == DT_FACTORS_ROWS) {
    // operands prepared once per factor pair by dt_rows_prepare: the row-tile kernel alone
    if (!tc_rows_ok(g, x_dtype, y_dtype) ||
        ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
          reinterpret_cast<uintptr_t>(bias) | reinterpret_cast<uintptr_t>(xf)) & 15) != 0) {
      set_error("DT_FACTORS_ROWS: geometry/operands not eligible for the row-tile kernel "
                "(dt_rows_prepared_bytes == 0) or misaligned pointers");
      return DT_E_UNSUPPORTED;
    }
    if (batch == 0) return DT_OK;
    return tc_rows_forward(g, batch, x, nullptr, nullptr, bias, act, act_arg, y, y_dtype,
                           (char *)const_cast<void *>(xf), (cudaStream_t)stream, true);
  }
  if (f_dtype == DT_FACTORS_ROWS) {
    set_error("DT_FACTORS_ROWS operands are for the bf16 tensor-core path");
    return DT_E_ARG;
  }
  if (mma == DT_MMA_BF16) {
    // DT_FACTORS_PACKED: the fused single-kernel path (in-kernel W regeneration, general
    // geometries only). DT_F32 / DT_BF16 factors: the two-phase path (W^T regenerated into
    // the workspace, then the tcgen05 GEMM), any geometry. DEEPTHIN_TC_FUSED=1 routes bf16
    // factors on general geometries to the fused kernel (comparison runs).
    static const int want_fused = getenv("DEEPTHIN_TC_FUSED") ? atoi(getenv("DEEPTHIN_TC_FUSED")) : 0;
    const bool pk = f_dtype == DT_FACTORS_PACKED;
    if (pk || (want_fused && f_dtype == DT_BF16 && !g.reuse)) {
      if (g.reuse) {
        set_error("packed factors exist only for general (straddling-row) geometries");
        return DT_E_UNSUPPORTED;
      }
      return tc_general_forward(g, batch, x, x_dtype, pk ? nullptr : (const uint16_t *)xf,
                                pk ? nullptr : (const uint16_t *)wf, pk ? xf : nullptr, bias, act,
                                act_arg, y, y_dtype, (char *)workspace, workspace_bytes, st);
    }
    return tc_gemm_forward(g, batch, x, x_dtype, xf, wf, f_dtype, bias, act, act_arg, y, y_dtype,
                           (char *)workspace, workspace_bytes, st);
  }
  set_error("unknown mma kind " + std::to_string(mma));
  return DT_E_ARG;
}

int dt_forward_path(const dt_plan *plan, int mma, int x_dtype, int f_dtype, int y_dtype) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return -rc;
  if (int rc = check_dtype(x_dtype, "x")) return -rc;
  if (int rc = check_dtype(y_dtype, "y")) return -rc;
  if (mma == DT_MMA_FFMA) {
    if (f_dtype == DT_F32) return DT_PATH_FFMA;
    set_error("the FFMA path takes fp32 factors");
    return -DT_E_ARG;
  }
  if (mma != DT_MMA_BF16) {
    set_error("unknown mma kind " + std::to_string(mma));
    return -DT_E_ARG;
  }
  if (f_dtype == DT_FACTORS_ROWS) return tc_rows_ok(g, x_dtype, y_dtype) ? DT_PATH_ROWS : -DT_E_UNSUPPORTED;
  static const int want_fused = getenv("DEEPTHIN_TC_FUSED") ? atoi(getenv("DEEPTHIN_TC_FUSED")) : 0;
  if (f_dtype == DT_FACTORS_PACKED || (want_fused && f_dtype == DT_BF16 && !g.reuse))
    return g.reuse ? -DT_E_UNSUPPORTED : DT_PATH_FUSED;
  return tc_forward_path(g, x_dtype, f_dtype, y_dtype);
}

size_t dt_backward_workspace_bytes(const dt_plan *plan, int64_t batch, int mma) {
  Geo g;
  if (make_geo(plan, &g) || batch < 0) return 0;
  if (mma == DT_MMA_BF16 && tc_backward_ok(g)) return tc_backward_ws(g, batch);
  if (mma == DT_MMA_BF16 && xback_general_ok(g)) return xback_general_ws(g, batch);
  return ffma_backward_ws(g, batch);
}

int dt_backward(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
                const float *xf, const float *wf, const float *bias, int act, float act_arg,
                const float *upstream, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                void *workspace, size_t workspace_bytes, dt_stream stream) {
  return dt_backward_ex(plan, batch, mma, x, x_dtype, xf, wf, bias, act, act_arg, upstream, d_xf,
                        d_wf, d_bias, d_input, nullptr, workspace, workspace_bytes, stream);
}

int dt_backward_ex(const dt_plan *plan, int64_t batch, int mma, const void *x, int x_dtype,
                   const float *xf, const float *wf, const float *bias, int act, float act_arg,
                   const float *upstream, float *d_xf, float *d_wf, float *d_bias, float *d_input,
                   const float *p_in, void *workspace, size_t workspace_bytes, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  if (int rc = check_dtype(x_dtype, "x")) return rc;
  if (int rc = check_act(act)) return rc;
  if (act == DT_ACT_SOFTMAX) {
    set_error("softmax is forward-only (use the fused softmax cross-entropy gradient)");
    return DT_E_UNSUPPORTED;
  }
  if (!xf || !wf || !d_xf || !d_wf || (batch > 0 && (!x || !upstream))) {
    set_error("NULL operand pointer");
    return DT_E_ARG;
  }
  if (mma != DT_MMA_FFMA && mma != DT_MMA_BF16) {
    set_error("unknown mma kind " + std::to_string(mma));
    return DT_E_ARG;
  }
  // bf16 / tf32 tensor cores for reuse geometries (factored); every other case runs the exact
  // fp32 FFMA backward. A pending dt_set_backward_event is recorded when d_xf is final (the
  // factored path: after its first GEMM), at the latest when the call's work is enqueued.
  const cudaStream_t st = (cudaStream_t)stream;
  auto done = [&](int rc) { return rc ? rc : backward_event_record(st); };
  if (mma == DT_MMA_BF16 && tc_backward_ok(g))
    return done(tc_backward(g, batch, x, x_dtype, xf, wf, bias, act, act_arg, upstream, d_xf,
                            d_wf, d_bias, d_input, (char *)workspace, workspace_bytes, st, p_in));
  if (p_in) {
    set_error("backward: a kept P applies to the tensor-core backward of reuse geometries only");
    return DT_E_UNSUPPORTED;
  }
  // general (straddling) geometries on the tensor cores (k_train.cu)
  if (mma == DT_MMA_BF16 && xback_general_ok(g))
    return done(xback_general(g, batch, x, x_dtype, xf, wf, bias, act, act_arg, upstream, d_xf,
                              d_wf, d_bias, d_input, (char *)workspace, workspace_bytes, st));
  return done(ffma_backward(g, batch, x, x_dtype, xf, wf, bias, act, act_arg, upstream, d_xf,
                            d_wf, d_bias, d_input, (char *)workspace, workspace_bytes, st));
}

size_t dt_forward_mse_workspace_bytes(const dt_plan *plan, int64_t batch) {
  Geo g;
  if (make_geo(plan, &g) || batch < 0) return 0;
  return tc_forward_mse_ws(g, batch);
}

int dt_forward_mse(const dt_plan *plan, int64_t batch, const void *x, int x_dtype, const float *xf,
                   const float *wf, const float *bias, const float *target, double norm_count,
                   float *grad, double *loss_sum, void *workspace, size_t workspace_bytes,
                   dt_stream stream) {
  return dt_forward_mse_ex(plan, batch, x, x_dtype, xf, wf, bias, target, norm_count, grad,
                           loss_sum, nullptr, nullptr, workspace, workspace_bytes, stream);
}

size_t dt_forward_p_bytes(const dt_plan *plan, int64_t batch) {
  Geo g;
  if (make_geo(plan, &g) || batch < 0 || !tc_backward_ok(g)) return 0;
  return (size_t)batch * g.s * g.rank * 4;
}

int dt_forward_mse_ex(const dt_plan *plan, int64_t batch, const void *x, int x_dtype,
                      const float *xf, const float *wf, const float *bias, const float *target,
                      double norm_count, float *grad, double *loss_sum, float *d_bias,
                      float *p_out, void *workspace, size_t workspace_bytes, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  if (int rc = check_dtype(x_dtype, "x")) return rc;
  if (!(norm_count > 0)) {
    set_error("norm_count must be > 0");
    return DT_E_ARG;
  }
  if (batch > 0 && (!x || !xf || !wf || !target || !grad)) {
    set_error("NULL operand pointer");
    return DT_E_ARG;
  }
  return tc_forward_mse(g, batch, x, x_dtype, xf, wf, bias, target, 2.0 / norm_count, grad,
                        loss_sum, (char *)workspace, workspace_bytes, (cudaStream_t)stream, d_bias,
                        p_out);
}

size_t dt_mse_workspace_bytes(int64_t rows, int64_t cols) { return mse_ws(rows, cols); }

int dt_mse_grad(int64_t rows, int64_t cols, const float *y, const float *target,
                double norm_count, float *grad, double *loss_sum, void *workspace,
                size_t workspace_bytes, dt_stream stream) {
  if (rows < 0 || cols < 0) {
    set_error("negative shape");
    return DT_E_DIM;
  }
  if (!(norm_count > 0)) {
    set_error("norm_count must be > 0");
    return DT_E_ARG;
  }
  return launch_mse_grad(rows, cols, y, target, norm_count, grad, loss_sum, (char *)workspace,
                         workspace_bytes, (cudaStream_t)stream);
}

int dt_chain_ok(const dt_plan *plans, int n_layers) {
  if (!plans || n_layers < 2 || n_layers > 8) return 0;
  Geo g[8];
  for (int l = 0; l < n_layers; ++l)
    if (make_geo(&plans[l], &g[l])) return 0;
  return tc_chain_ok(g, n_layers) ? 1 : 0;
}

int dt_chain_forward(const dt_plan *plans, int n_layers, int64_t batch, const void *x,
                     void *const *prepared, int hidden_act, float act_arg, int last_act, void *y,
                     dt_stream stream) {
  if (!plans || n_layers < 2 || n_layers > 8) {
    set_error("dt_chain_forward: 2 to 8 layers");
    return DT_E_ARG;
  }
  Geo g[8];
  for (int l = 0; l < n_layers; ++l)
    if (int rc = make_geo(&plans[l], &g[l])) return rc;
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  if (int rc = check_act(hidden_act)) return rc;
  if (hidden_act == DT_ACT_SOFTMAX || (last_act != DT_ACT_IDENTITY && last_act != DT_ACT_SOFTMAX)) {
    set_error("dt_chain_forward: hidden_act must be elementwise, last_act identity or softmax");
    return DT_E_ARG;
  }
  if (batch > 0 && (!x || !y || !prepared)) {
    set_error("NULL operand pointer");
    return DT_E_ARG;
  }
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) {
    set_error("dt_chain_forward: x and y must be 16-byte aligned");
    return DT_E_ARG;
  }
  const cudaStream_t st = (cudaStream_t)stream;
  if (int rc = tc_chain_forward(g, n_layers, batch, x, prepared, hidden_act, act_arg, y, st)) return rc;
  if (last_act == DT_ACT_SOFTMAX && batch > 0)
    return launch_row_softmax(batch, g[n_layers - 1].r_dim, y, DT_BF16, st);
  return DT_OK;
}

namespace {
XGemm matmul_desc(int64_t M, int64_t N, int64_t K, const void *a, int64_t lda, int a_trans,
                  const void *b, int64_t ldb, int b_trans, int dtype) {
  XGemm x;
  x.M = M; x.N = N; x.K = K;
  x.A = a; x.lda = lda; x.a_mn = a_trans ? 1 : 0;      // a stored K x M: M contiguous
  x.B = b; x.ldb = ldb; x.b_mn = b_trans ? 0 : 1;      // b stored K x N: N contiguous
  x.el = dtype == DT_F32 ? 1 : 0;
  x.BN = N > 128 ? 256 : (N > 64 || (x.b_mn && x.el == 0) ? 128 : 64);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  x.splits = xgemm_splits(M, N, K, x.BN, x.el, nsm);
  return x;
}
}  // namespace

size_t dt_matmul_workspace_bytes(int64_t M, int64_t N, int64_t K, int dtype) {
  if (M < 0 || N < 0 || K < 0) return 0;
  return xgemm_ws(matmul_desc(M, N, K, nullptr, 0, 0, nullptr, 0, 0, dtype)) + 256;
}

int dt_matmul(int64_t M, int64_t N, int64_t K, const void *a, int64_t lda, int a_trans,
              const void *b, int64_t ldb, int b_trans, int dtype, float *c, int64_t ldc,
              void *workspace, size_t workspace_bytes, dt_stream stream) {
  if (M < 0 || N < 0 || K < 0) {
    set_error("dt_matmul: negative shape");
    return DT_E_DIM;
  }
  if (dtype != DT_F32 && dtype != DT_BF16) {
    set_error("dt_matmul: dtype must be DT_F32 or DT_BF16");
    return DT_E_ARG;
  }
  const int esz = dtype == DT_F32 ? 4 : 2;
  if ((lda * esz) % 16 || (ldb * esz) % 16 || (ldc * 4) % 16 ||
      (reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
       reinterpret_cast<uintptr_t>(c)) % 16) {
    set_error("dt_matmul: pointers and pitches must be 16-byte aligned");
    return DT_E_ARG;
  }
  if (M == 0 || N == 0) return DT_OK;
  if (K == 0) {
    for (int64_t i = 0; i < M; ++i)
      DT_CUDA_CHECK(cudaMemsetAsync(c + i * ldc, 0, (size_t)N * 4, (cudaStream_t)stream));
    return DT_OK;
  }
  XGemm x = matmul_desc(M, N, K, a, lda, a_trans, b, ldb, b_trans, dtype);
  x.out = c;
  x.ldo = ldc;
  if (x.splits > 1) {
    if (workspace_bytes < xgemm_ws(x)) {
      set_error("dt_matmul: workspace too small (dt_matmul_workspace_bytes)");
      return DT_E_ARG;
    }
    x.part = reinterpret_cast<float *>(workspace);
  }
  return xgemm(x, (cudaStream_t)stream);
}

int dt_sgd_step(int64_t count, float *param, const float *grad, float lr, dt_stream stream) {
  if (count < 0) {
    set_error("count must be >= 0");
    return DT_E_ARG;
  }
  if (!(lr > 0.f)) {
    set_error("learning_rate must be > 0");
    return DT_E_ARG;
  }
  return launch_sgd(count, param, grad, lr, (cudaStream_t)stream);
}

int dt_rows_chain(const void *wait_flags, unsigned wait_target, void *post_flags) {
  rows_chain(reinterpret_cast<const unsigned *>(wait_flags), wait_target,
             reinterpret_cast<unsigned *>(post_flags));
  return DT_OK;
}

int dt_rows_posts_per_tile(const dt_plan *plan) {
  Geo g;
  if (make_geo(plan, &g)) return 0;
  return rows_posts_per_tile(g);
}

size_t dt_rows_prepared_bytes(const dt_plan *plan, int x_dtype, int y_dtype) {
  Geo g;
  if (make_geo(plan, &g) || !tc_rows_ok(g, x_dtype, y_dtype)) return 0;
  return tc_rows_ws(g);
}

int dt_rows_prepare(const dt_plan *plan, int act, int y_dtype, const float *xf, const float *wf,
                    const float *bias, void *out, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (int rc = check_act(act)) return rc;
  if (int rc = check_dtype(y_dtype, "y")) return rc;
  if (!tc_rows_ok(g, DT_BF16, y_dtype)) {
    set_error("dt_rows_prepare: geometry not eligible for the row-tile kernel");
    return DT_E_UNSUPPORTED;
  }
  if (!xf || !wf || !out || (reinterpret_cast<uintptr_t>(out) & 255)) {
    set_error("dt_rows_prepare: NULL operand or output not 256-byte aligned");
    return DT_E_ARG;
  }
  const int eact = act == DT_ACT_SOFTMAX ? DT_ACT_IDENTITY : act;
  return tc_rows_prepare(g, wf, xf, bias, eact, y_dtype, (char *)out, (cudaStream_t)stream);
}

size_t dt_lstm_gates_workspace_bytes(const dt_plan *plan, int64_t batch) {
  Geo g;
  if (make_geo(plan, &g) || batch < 0 || !lstm_gates_ok(g)) return 0;
  return std::max<size_t>(256, lstm_gates_ws(g, batch));
}

int dt_lstm_gates(const dt_plan *plan, int64_t batch, const float *h, const float *const *xf,
                  const float *const *wf, const float *const *bias, float *const *gh,
                  void *workspace, size_t workspace_bytes, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  if (!lstm_gates_ok(g)) {
    set_error("lstm_gates: needs a square reuse geometry (n | q, q == r_dim), rank <= 64, "
              "s*rank <= 256 and a multiple of 4, n <= 1024");
    return DT_E_UNSUPPORTED;
  }
  if (batch > 0) {
    if (!h || !xf || !wf || !gh || !workspace) {
      set_error("lstm_gates: NULL operand pointer");
      return DT_E_ARG;
    }
    for (int i = 0; i < 4; ++i)
      if (!xf[i] || !wf[i] || !gh[i]) {
        set_error("lstm_gates: NULL gate pointer");
        return DT_E_ARG;
      }
    if (workspace_bytes < lstm_gates_ws(g, batch)) {
      set_error("lstm_gates: workspace too small");
      return DT_E_ARG;
    }
  }
  return lstm_gates(g, batch, h, xf, wf, bias, gh, (char *)workspace, (cudaStream_t)stream);
}

size_t dt_lstm_sequence_workspace_bytes(const dt_plan *plan, int64_t batch) {
  Geo g;
  if (make_geo(plan, &g) || !lstm_seq_ok(g, batch)) return 0;
  return lstm_seq_ws(g, batch);
}

int dt_lstm_sequence(const dt_plan *plan, int64_t T, int64_t batch, const void *const *gx,
                     const float *const *xf, const float *const *wf, const float *const *bias,
                     void *out, void *workspace, size_t workspace_bytes, dt_stream stream) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (T < 0 || batch < 0) {
    set_error("lstm_sequence: T, batch >= 0");
    return DT_E_DIM;
  }
  if (T == 0 || batch == 0) return DT_OK;
  if (!lstm_seq_ok(g, batch)) {
    set_error("lstm_sequence: needs batch <= 64 and a square reuse geometry dt_lstm_gates takes");
    return DT_E_UNSUPPORTED;
  }
  if (!gx || !xf || !wf || !out || !workspace) {
    set_error("lstm_sequence: NULL operand pointer");
    return DT_E_ARG;
  }
  for (int i = 0; i < 4; ++i)
    if (!gx[i] || !xf[i] || !wf[i]) {
      set_error("lstm_sequence: NULL gate pointer");
      return DT_E_ARG;
    }
  if (workspace_bytes < lstm_seq_ws(g, batch)) {
    set_error("lstm_sequence: workspace too small");
    return DT_E_ARG;
  }
  return lstm_seq(g, T, batch, gx, xf, wf, bias, out, (char *)workspace, (cudaStream_t)stream);
}

int dt_lstm_cell(int64_t batch, int64_t hidden, const void *const *gx, int64_t ld_gx,
                 const float *const *gh, float *c, float *h32, void *h16, dt_stream stream) {
  if (batch < 0 || hidden < 0 || ld_gx < hidden) {
    set_error("lstm_cell: batch, hidden >= 0 and ld_gx >= hidden");
    return DT_E_DIM;
  }
  if (batch > 0 && hidden > 0) {
    if (!gx || !gh || !c || (!h32 && !h16)) {
      set_error("lstm_cell: NULL operand pointer");
      return DT_E_ARG;
    }
    for (int g = 0; g < 4; ++g)
      if (!gx[g] || !gh[g]) {
        set_error("lstm_cell: NULL gate pointer");
        return DT_E_ARG;
      }
  }
  return launch_lstm_cell(batch, hidden, gx, ld_gx, gh, c, h32, h16, (cudaStream_t)stream);
}

// ---- host-buffer sessions ---------------------------------------------------------------
// Host-buffer sessions. A call is split into row chunks that alternate between two streams:
// chunk c's H2D copy, forward and D2H copy are ordered on stream c % 2, so the two copy
// directions and the kernels of neighbouring chunks overlap (PCIe is the bottleneck of this
// entry point: at config 2 the fp32 y read-back is 33.5 MB per call).
constexpr int kSessionStreams = 2;
struct dt_session {
  dt_plan plan;
  Geo geo;
  int mma;
  float *xf = nullptr, *wf = nullptr, *bias = nullptr;
  uint16_t *xf16 = nullptr, *wf16 = nullptr;
  void *packed = nullptr;  // dt_pack_factors buffer (DEEPTHIN_TC_FUSED comparison runs only)
  float *x = nullptr, *y = nullptr;
  char *ws[kSessionStreams] = {nullptr, nullptr};
  size_t ws_bytes = 0;
  int64_t cap_batch = 0, cap_chunk = 0;
  cudaStream_t stream = nullptr;  // stream 0 of the pipeline
  cudaStream_t stream2 = nullptr;
};

static void session_free_io(dt_session *s) {
  cudaFree(s->x);
  cudaFree(s->y);
  for (auto &w : s->ws) cudaFree(w), w = nullptr;
  s->x = s->y = nullptr;
  s->cap_batch = s->cap_chunk = 0;
}

// Rows per chunk: DEEPTHIN_SESSION_CHUNK_ROWS, else 1024 (a multiple of the GEMM's 256-row
// batch tile), never fewer than 4 chunks' worth of overlap when the batch allows.
static int64_t session_chunk_rows(int64_t batch) {
  static const int64_t env = getenv("DEEPTHIN_SESSION_CHUNK_ROWS")
                                 ? atoll(getenv("DEEPTHIN_SESSION_CHUNK_ROWS"))
                                 : 0;
  if (env > 0) return std::min(env, std::max<int64_t>(batch, 1));
  return std::min<int64_t>(std::max<int64_t>(batch, 1), 1024);
}

int dt_session_create(const dt_plan *plan, int mma, const float *xf_host, const float *wf_host,
                      const float *bias_host, dt_session **out) {
  Geo g;
  if (int rc = make_geo(plan, &g)) return rc;
  if (mma != DT_MMA_FFMA && mma != DT_MMA_BF16) {
    set_error("unknown mma kind");
    return DT_E_ARG;
  }
  dt_session *s = new dt_session();
  s->plan = *plan;
  s->geo = g;
  s->mma = mma;
  const size_t nx = (size_t)g.m * g.rank, nw = (size_t)g.rank * g.n;
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->stream2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&s->xf, nx * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->wf, nw * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->bias, (size_t)g.r_dim * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->xf16, nx * 2);
  if (e == cudaSuccess) e = cudaMalloc(&s->wf16, nw * 2);
  if (e == cudaSuccess) e = cudaMemcpy(s->xf, xf_host, nx * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->wf, wf_host, nw * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    if (bias_host)
      e = cudaMemcpy(s->bias, bias_host, (size_t)g.r_dim * 4, cudaMemcpyHostToDevice);
    else
      e = cudaMemset(s->bias, 0, (size_t)g.r_dim * 4);
  }
  if (e != cudaSuccess) {
    set_error(std::string("session create: ") + cudaGetErrorString(e));
    dt_session_destroy(s);
    return DT_E_CUDA;
  }
  int rc = launch_cast_bf16((int64_t)nx, s->xf, s->xf16, s->stream);
  if (!rc) rc = launch_cast_bf16((int64_t)nw, s->wf, s->wf16, s->stream);
  // The fused kernel's packed operands, only for DEEPTHIN_TC_FUSED comparison runs; the
  // default bf16 path regenerates W^T from the fp32 factors each call.
  const size_t pkb = getenv("DEEPTHIN_TC_FUSED") ? dt_packed_factors_bytes(plan, mma) : 0;
  if (!rc && pkb) {
    if (cudaMalloc(&s->packed, pkb) != cudaSuccess) rc = DT_E_CUDA;
    if (!rc) rc = dt_pack_factors(plan, mma, s->xf16, s->wf16, s->packed, (dt_stream)s->stream);
  }
  if (!rc && cudaStreamSynchronize(s->stream) != cudaSuccess) rc = DT_E_CUDA;
  if (rc) {
    dt_session_destroy(s);
    return rc;
  }
  *out = s;
  return DT_OK;
}

int dt_session_forward(dt_session *s, int64_t batch, const float *x_host, int act, float act_arg,
                       float *y_host, int64_t *h2d, int64_t *d2h) {
  if (!s) {
    set_error("NULL session");
    return DT_E_ARG;
  }
  if (batch < 0) {
    set_error("batch must be >= 0");
    return DT_E_DIM;
  }
  const Geo &g = s->geo;
  const int64_t chunk = session_chunk_rows(batch);
  if (batch > s->cap_batch || chunk > s->cap_chunk) {
    session_free_io(s);
    const size_t ws = dt_forward_workspace_bytes(&s->plan, chunk, s->mma);
    cudaError_t e = cudaMalloc(&s->x, (size_t)std::max<int64_t>(batch, 1) * g.q * 4);
    if (e == cudaSuccess) e = cudaMalloc(&s->y, (size_t)std::max<int64_t>(batch, 1) * g.r_dim * 4);
    for (auto &w : s->ws)
      if (e == cudaSuccess) e = cudaMalloc(&w, ws ? ws : 256);
    if (e != cudaSuccess) {
      set_error(std::string("session alloc: ") + cudaGetErrorString(e));
      session_free_io(s);
      return DT_E_CUDA;
    }
    s->ws_bytes = ws;
    s->cap_batch = batch;
    s->cap_chunk = chunk;
  }
  const bool tc = s->mma == DT_MMA_BF16;
  const void *fx = s->xf, *fw = s->wf;
  int fdt = DT_F32;
  if (tc && s->packed) {
    fx = s->packed; fw = nullptr; fdt = DT_FACTORS_PACKED;
  }
  cudaStream_t st[kSessionStreams] = {s->stream, s->stream2};
  int c = 0;
  for (int64_t r0 = 0; r0 < batch; r0 += chunk, ++c) {
    const int64_t rows = std::min(chunk, batch - r0);
    cudaStream_t cs = st[c % kSessionStreams];
    float *xd = s->x + r0 * g.q, *yd = s->y + r0 * g.r_dim;
    DT_CUDA_CHECK(cudaMemcpyAsync(xd, x_host + r0 * g.q, (size_t)rows * g.q * 4,
                                  cudaMemcpyHostToDevice, cs));
    int rc = dt_forward(&s->plan, rows, s->mma, xd, DT_F32, fx, fw, fdt, s->bias, act, act_arg, yd,
                        DT_F32, s->ws[c % kSessionStreams], s->ws_bytes, (dt_stream)cs);
    if (rc) return rc;
    DT_CUDA_CHECK(cudaMemcpyAsync(y_host + r0 * g.r_dim, yd, (size_t)rows * g.r_dim * 4,
                                  cudaMemcpyDeviceToHost, cs));
  }
  for (auto cs : st) DT_CUDA_CHECK(cudaStreamSynchronize(cs));
  if (h2d) *h2d = batch * g.q * 4;
  if (d2h) *d2h = batch * g.r_dim * 4;
  return DT_OK;
}

void dt_session_destroy(dt_session *s) {
  if (!s) return;
  session_free_io(s);
  cudaFree(s->xf);
  cudaFree(s->wf);
  cudaFree(s->bias);
  cudaFree(s->xf16);
  cudaFree(s->wf16);
  cudaFree(s->packed);
  if (s->stream) cudaStreamDestroy(s->stream);
  if (s->stream2) cudaStreamDestroy(s->stream2);
  delete s;
}

}  // extern "C"
