"""ctypes binding of libdeepthin_b200.so (include/deepthin_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute call raises CudaError.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ArgumentError, CudaError, DimensionError, UnsupportedConfigurationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DEEPTHIN_LIB") or os.path.join(_HERE, "_lib", "libdeepthin_b200.so")

DT_OK, DT_E_DIM, DT_E_ARG, DT_E_UNSUPPORTED, DT_E_CUDA, DT_E_FORMAT = range(6)
DT_F32, DT_BF16, DT_FACTORS_PACKED, DT_F64, DT_FACTORS_ROWS = 0, 1, 2, 3, 4
DT_MMA_FFMA, DT_MMA_BF16 = 0, 1
DT_PROF_ANY, DT_PROF_GEMM, DT_PROF_ROWS = 0, 1, 2
DT_PIPELINE_OFF, DT_PIPELINE_ON, DT_PIPELINE_EXTERNAL_X = 0, 1, 2
# dt_forward_path results (include/deepthin_b200.h enum dt_path)
PATHS = {1: "ffma", 2: "rows", 3: "factored", 4: "runs", 5: "hilo", 6: "pair", 7: "fused"}
ACT_CODES = {"identity": 0, "relu": 1, "sigmoid": 2, "tanh": 3, "clipped_relu": 4, "softmax": 5}

# Every symbol the header declares (checked by tests/test_abi.py).
EXPORTS = (
    "dt_version", "dt_last_error", "dt_launch_counter", "dt_profile_kernel_events", "dt_profile_kernel_kind", "dt_set_forward_pipeline", "dt_plan_validate", "dt_plan_query", "dt_phase",
    "dt_relayout_index", "dt_predict_reuse", "dt_op_count", "dt_decompress", "dt_cast_bf16",
    "dt_packed_factors_bytes", "dt_pack_factors",
    "dt_forward_workspace_bytes", "dt_forward", "dt_forward_path", "dt_backward_workspace_bytes", "dt_backward",
    "dt_mse_grad", "dt_mse_workspace_bytes", "dt_forward_mse", "dt_forward_mse_workspace_bytes", "dt_forward_mse_ex", "dt_forward_p_bytes", "dt_backward_ex", "dt_sgd_step", "dt_matmul_workspace_bytes", "dt_matmul", "dt_chain_ok", "dt_chain_forward", "dt_set_backward_event", "dt_rows_prepared_bytes", "dt_rows_prepare", "dt_rows_chain", "dt_rows_posts_per_tile", "dt_lstm_gates_workspace_bytes", "dt_lstm_gates", "dt_lstm_sequence_workspace_bytes", "dt_lstm_sequence", "dt_lstm_cell", "dt_session_create",
    "dt_session_forward", "dt_session_destroy", "dt_model_parse", "dt_unpack_values",
)


class Plan(C.Structure):
    _fields_ = [("q", C.c_int64), ("r_dim", C.c_int64), ("rank", C.c_int64),
                ("m", C.c_int64), ("n", C.c_int64)]


class PlanInfo(C.Structure):
    _fields_ = [("period", C.c_int64), ("phase_count", C.c_int64), ("reuse", C.c_int64),
                ("segments", C.c_int64), ("tail", C.c_int64), ("rows_per_period", C.c_int64)]


class Span(C.Structure):
    _fields_ = [("offset", C.c_int64), ("length", C.c_int64)]


class ModelMeta(C.Structure):
    _fields_ = [("key", Span), ("value", Span)]


class ModelHeader(C.Structure):
    _fields_ = [("version", C.c_uint32), ("layer_count", C.c_uint32),
                ("payload_bytes", C.c_uint64), ("target_ratio", C.c_double),
                ("meta_count", C.c_uint32), ("reserved", C.c_uint32),
                ("meta_read", C.c_int64), ("layers_read", C.c_int64)]


class ModelLayer(C.Structure):
    _fields_ = [("name", Span), ("plan", Plan), ("dtype_code", C.c_int32),
                ("floor_hit", C.c_int32), ("bias_len", C.c_int64), ("xf_offset", C.c_int64),
                ("wf_offset", C.c_int64), ("bias_offset", C.c_int64)]


class FormatError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("what", C.c_int32), ("offset", C.c_int64),
                ("layer", C.c_int64), ("need", C.c_int64), ("have", C.c_int64)]


(DT_FMT_OK, DT_FMT_TRUNCATED, DT_FMT_BAD_MAGIC, DT_FMT_BAD_VERSION, DT_FMT_PAYLOAD_MISMATCH,
 DT_FMT_BAD_DTYPE, DT_FMT_INVALID_PLAN, DT_FMT_TRAILING) = range(8)
(DT_WHAT_HEADER, DT_WHAT_META_COUNT, DT_WHAT_META_KEY_LEN, DT_WHAT_META_KEY,
 DT_WHAT_META_VALUE_LEN, DT_WHAT_META_VALUE, DT_WHAT_NAME_LEN, DT_WHAT_NAME, DT_WHAT_PLAN,
 DT_WHAT_FLAGS, DT_WHAT_BIAS_LEN, DT_WHAT_XF, DT_WHAT_WF, DT_WHAT_BIAS) = range(14)

_lib = None


def _declare(lib):
    P, I64, VP, F, D, SZ = C.POINTER(Plan), C.c_int64, C.c_void_p, C.c_float, C.c_double, C.c_size_t
    i = C.c_int
    sig = {
        "dt_version": ([], C.c_char_p),
        "dt_last_error": ([], C.c_char_p),
        "dt_launch_counter": ([], I64),
        "dt_profile_kernel_events": ([C.POINTER(VP), C.POINTER(VP), i], i),
        "dt_profile_kernel_kind": ([i], i),
        "dt_set_forward_pipeline": ([i], i),
        "dt_forward_mse_workspace_bytes": ([P, I64], SZ),
        "dt_forward_mse": ([P, I64, VP, i, VP, VP, VP, VP, D, VP, VP, VP, SZ, VP], i),
        "dt_forward_mse_ex": ([P, I64, VP, i, VP, VP, VP, VP, D, VP, VP, VP, VP, VP, SZ, VP], i),
        "dt_forward_p_bytes": ([P, I64], SZ),
        "dt_plan_validate": ([P], i),
        "dt_plan_query": ([P, C.POINTER(PlanInfo)], i),
        "dt_phase": ([P, I64, C.POINTER(I64)], i),
        "dt_relayout_index": ([P, I64, C.POINTER(I64), C.POINTER(I64)], i),
        "dt_predict_reuse": ([P, I64, C.POINTER(I64), C.POINTER(I64)], i),
        "dt_op_count": ([P, I64, C.POINTER(I64), C.POINTER(I64)], i),
        "dt_decompress": ([P, VP, VP, VP, VP], i),
        "dt_cast_bf16": ([I64, VP, VP, VP], i),
        "dt_packed_factors_bytes": ([P, i], SZ),
        "dt_pack_factors": ([P, i, VP, VP, VP, VP], i),
        "dt_forward_workspace_bytes": ([P, I64, i], SZ),
        "dt_forward": ([P, I64, i, VP, i, VP, VP, i, VP, i, F, VP, i, VP, SZ, VP], i),
        "dt_backward_workspace_bytes": ([P, I64, i], SZ),
        "dt_backward": ([P, I64, i, VP, i, VP, VP, VP, i, F, VP, VP, VP, VP, VP, VP, SZ, VP], i),
        "dt_backward_ex": ([P, I64, i, VP, i, VP, VP, VP, i, F, VP, VP, VP, VP, VP, VP, VP, SZ, VP], i),
        "dt_mse_workspace_bytes": ([I64, I64], SZ),
        "dt_mse_grad": ([I64, I64, VP, VP, D, VP, VP, VP, SZ, VP], i),
        "dt_sgd_step": ([I64, VP, VP, F, VP], i),
        "dt_matmul_workspace_bytes": ([I64, I64, I64, i], SZ),
        "dt_chain_ok": ([P, i], i),
        "dt_set_backward_event": ([VP], i),
        "dt_chain_forward": ([P, i, I64, VP, C.POINTER(VP), i, F, i, VP, VP], i),
        "dt_forward_path": ([P, i, i, i, i], i),
        "dt_matmul": ([I64, I64, I64, VP, I64, i, VP, I64, i, i, VP, I64, VP, SZ, VP], i),
        "dt_rows_prepared_bytes": ([P, i, i], SZ),
        "dt_rows_chain": ([VP, C.c_uint, VP], i),
        "dt_rows_posts_per_tile": ([P], i),
        "dt_rows_prepare": ([P, i, i, VP, VP, VP, VP, VP], i),
        "dt_lstm_gates_workspace_bytes": ([P, I64], SZ),
        "dt_lstm_gates": ([P, I64, VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP), C.POINTER(VP), VP, SZ, VP], i),
        "dt_lstm_sequence_workspace_bytes": ([P, I64], SZ),
        "dt_lstm_sequence": ([P, I64, I64, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP), C.POINTER(VP), VP, VP, SZ, VP], i),
        "dt_lstm_cell": ([I64, I64, C.POINTER(VP), I64, C.POINTER(VP), VP, VP, VP, VP], i),
        "dt_session_create": ([P, i, VP, VP, VP, C.POINTER(VP)], i),
        "dt_session_forward": ([VP, I64, VP, i, F, VP, C.POINTER(I64), C.POINTER(I64)], i),
        "dt_session_destroy": ([VP], None),
        "dt_model_parse": ([VP, SZ, C.POINTER(ModelHeader), C.POINTER(ModelMeta), I64,
                            C.POINTER(ModelLayer), I64, C.POINTER(FormatError)], i),
        "dt_unpack_values": ([I64, VP, i, VP, VP, VP], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """Load (once) and return the native library; raise CudaError if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(
                f"native library {LIB_PATH} is missing; build it with "
                "`python -m paper_1802_06944_b200.build` (there is no CPU fallback)")
        handle = C.CDLL(LIB_PATH)
        _declare(handle)
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Raise the reference exception type matching a dt_status."""
    if rc == DT_OK:
        return
    msg = lib().dt_last_error().decode(errors="replace")
    if rc == DT_E_DIM:
        raise DimensionError(msg)
    if rc == DT_E_ARG:
        raise ArgumentError(msg)
    if rc == DT_E_UNSUPPORTED:
        raise UnsupportedConfigurationError(msg)
    raise CudaError(msg or f"dt status {rc}")


def plan_struct(plan) -> Plan:
    return Plan(plan.q, plan.r_dim, plan.rank, plan.m, plan.n)
