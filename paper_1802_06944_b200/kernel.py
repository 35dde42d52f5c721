"""Fused forward on the compressed form (reference kernel.py:39-320), on the GPU.

``fused_matmul`` / ``layer_forward`` keep the reference's names, argument
meaning and errors, and route to the sm_100a kernels through dt_forward:

* reuse path (n | q): every distinct run dot is computed once per input row
  (P = x.view(B*s, n) @ wf^T) and combined with xf (scale-after-dot);
* general path (straddling rows): W^T is regenerated from the factors on
  every call and contracted on tcgen05. The default two-phase form writes the
  bf16 W^T (2*q*r_dim bytes, 1.8 MB at config 2) to a workspace slot that
  stays L2-resident between the two kernels (it does reach HBM on write-back);
  the opt-in in-CTA form (DEEPTHIN_GEMM_WGEN=1) keeps every W block inside the
  SM. Nothing dense persists across calls: the layer's parameters in HBM are
  the factors.

Deliberate extensions: every rank is fused (the reference's rank-1 limit,
kernel.py:238-240, and its decompress fallback warning, :313-319, are
lifted), and activations include clipped ReLU and row softmax (BASELINE
configs 3/4). ``mma`` selects exact fp32 FFMA ("ffma", parity rtol 1e-5) or
bf16 tcgen05 tensor cores with fp32 accumulation ("bf16", rtol 2e-3).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import as_device_matrix, as_device_vector, device, stream_handle, workspace
from .errors import ArgumentError, DimensionError, UnsupportedConfigurationError
from .factor import FactorPair

ACTIVATIONS = ("identity", "relu", "sigmoid", "tanh")
EXTRA_ACTIVATIONS = ("clipped_relu", "softmax")


@dataclass
class OpCount:
    """kernel.py:65-77 — counts of the canonical run-memoized algorithm."""

    multiplies: int = 0
    adds: int = 0


@dataclass
class ReuseTable:
    """kernel.py:80-96 — hit/miss accounting (entries are not recorded on the GPU)."""

    hits: int = 0
    misses: int = 0
    record_entries: bool = False
    entries: dict = field(default_factory=dict)


class ReusePrediction(tuple):
    """(distinct_runs, total_runs) per input row (kernel.py:167-181)."""

    __slots__ = ()

    def __new__(cls, distinct_runs: int, total_runs: int):
        return super().__new__(cls, (distinct_runs, total_runs))

    @property
    def distinct_runs(self) -> int:
        return self[0]

    @property
    def total_runs(self) -> int:
        return self[1]


def predict_reuse(plan, batch: int = 1) -> ReusePrediction:
    """kernel.py:184-205 via dt_predict_reuse."""
    d, t = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().dt_predict_reuse(C.byref(_lib.plan_struct(plan)), int(batch),
                                           C.byref(d), C.byref(t)))
    return ReusePrediction(d.value, t.value)


def op_count(plan, batch: int) -> OpCount:
    mul, add = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().dt_op_count(C.byref(_lib.plan_struct(plan)), int(batch),
                                      C.byref(mul), C.byref(add)))
    return OpCount(multiplies=mul.value, adds=add.value)


def forward_path(plan, mma: str = "bf16", x_dtype=torch.bfloat16, y_dtype=torch.float32,
                 factors: str = "f32") -> str:
    """Kernel family layer_forward takes (dt_forward_path): "ffma", "rows", "factored", "runs",
    "hilo", "pair" or "fused" — each with its own arithmetic contract."""
    dt = {torch.bfloat16: _lib.DT_BF16, torch.float32: _lib.DT_F32}
    fd = {"f32": _lib.DT_F32, "bf16": _lib.DT_BF16, "packed": _lib.DT_FACTORS_PACKED,
          "rows": _lib.DT_FACTORS_ROWS}
    mk = {"ffma": _lib.DT_MMA_FFMA, "bf16": _lib.DT_MMA_BF16}
    if x_dtype not in dt or y_dtype not in dt or factors not in fd or mma not in mk:
        raise ArgumentError("forward_path: x/y dtype bf16|fp32, factors f32|bf16|packed|rows, "
                            "mma ffma|bf16")
    rc = _lib.lib().dt_forward_path(C.byref(_lib.plan_struct(plan)), mk[mma], dt[x_dtype],
                                    fd[factors], dt[y_dtype])
    if rc < 0:
        _lib.check(-rc)
    return _lib.PATHS[rc]


def _resolve_threads(threads):
    """kernel.py:208-214 — accepted for signature parity; GPU results never depend on it."""
    if threads is None:
        env = os.environ.get("DEEPTHIN_THREADS")
        threads = int(env) if env else 1
    if threads < 1:
        raise ArgumentError(f"threads must be >= 1, got {threads}")
    return threads


def _act_code(activation: str) -> int:
    try:
        return _lib.ACT_CODES[activation]
    except KeyError:
        raise ArgumentError(
            f"unknown activation {activation!r}; expected one of "
            f"{ACTIVATIONS + EXTRA_ACTIVATIONS}") from None


def resolve_mma(mma, x: torch.Tensor, plan) -> int:
    if mma is None:
        # bf16 inputs take the tensor-core path (any geometry); fp32 inputs the FFMA path
        mma = "bf16" if x.dtype == torch.bfloat16 else "ffma"
    if mma not in ("ffma", "bf16"):
        raise ArgumentError(f"mma must be 'ffma', 'bf16' or 'bf16_fused', got {mma!r}")
    return _lib.DT_MMA_BF16 if mma == "bf16" else _lib.DT_MMA_FFMA


class forward_pipeline:
    """Context manager / switch for inference pipelining on this thread (dt_set_forward_pipeline):
    consecutive bf16 tensor-core forwards on one stream overlap each call's W regeneration with
    the previous call's GEMM. Only for factors that are not updated while the calls run.
    ``external_x=True`` also promises that no call's input is produced by a call still in
    flight (independent batches, not a layer chain): the first x stages then load early too."""

    def __init__(self, enable: bool = True, external_x: bool = False):
        self.enable = enable
        self.external_x = external_x

    def __enter__(self):
        mode = (_lib.DT_PIPELINE_EXTERNAL_X if self.external_x else 1) if self.enable else 0
        _lib.check(_lib.lib().dt_set_forward_pipeline(mode))
        return self

    def __exit__(self, *exc):
        _lib.lib().dt_set_forward_pipeline(0)
        return False


def forward_into(x: torch.Tensor, fp: FactorPair, bias, act: int, act_arg: float, y: torch.Tensor,
                 mma: int, fused: bool = False, ws: torch.Tensor | None = None,
                 cached: bool = False) -> None:
    """Raw stream-ordered dt_forward on device tensors (no validation beyond the ABI's).

    bf16 tensor-core path: by default the two-phase kernels (W^T regenerated from the fp32
    factors, then the tcgen05 GEMM); ``fused=True`` runs the single fused kernel on the
    packed bf16 factors (general geometries only). ``ws``: a caller-owned workspace (grown
    here when too small); by default a fresh one per call. ``cached``: the caller keeps the
    factors and bias constant between calls, so the row-tile kernel's derived operands are
    built once per pair (FactorPair.rows_prepared) and the call launches that kernel alone."""
    p = fp.plan
    lib = _lib.lib()
    ps = _lib.plan_struct(p)
    batch = x.shape[0]
    if cached and mma == _lib.DT_MMA_BF16 and not fused and x.dtype == torch.bfloat16:
        ydt = _lib.DT_BF16 if y.dtype == torch.bfloat16 else _lib.DT_F32
        prep = fp.rows_prepared(bias, act, ydt)
        if prep is not None:
            _lib.check(lib.dt_forward(
                C.byref(ps), batch, mma, x.data_ptr(), _lib.DT_BF16, prep.data_ptr(), None,
                _lib.DT_FACTORS_ROWS, bias.data_ptr() if bias is not None else None, act,
                float(act_arg), y.data_ptr(), ydt, None, 0, stream_handle()))
            return
    ws_bytes = lib.dt_forward_workspace_bytes(C.byref(ps), batch, mma)
    if ws is None or ws.numel() < ws_bytes:
        ws = workspace(ws_bytes)
    if mma == _lib.DT_MMA_BF16 and fused:
        xf, wf, fdt = fp.packed(), None, _lib.DT_FACTORS_PACKED
        if xf is None:
            raise UnsupportedConfigurationError(
                "the fused tensor-core kernel needs a general (straddling-row) geometry")
    else:
        xf, wf, fdt = fp.xf, fp.wf, _lib.DT_F32
    _lib.check(lib.dt_forward(
        C.byref(ps), batch, mma, x.data_ptr(),
        _lib.DT_BF16 if x.dtype == torch.bfloat16 else _lib.DT_F32,
        xf.data_ptr(), wf.data_ptr() if wf is not None else None, fdt,
        bias.data_ptr() if bias is not None else None,
        act, float(act_arg), y.data_ptr(),
        _lib.DT_BF16 if y.dtype == torch.bfloat16 else _lib.DT_F32,
        ws.data_ptr(), ws.numel(), stream_handle()))


def _forward(x, fp: FactorPair, bias, activation, act_arg, mma, out_dtype):
    xt, host = as_device_matrix(x, name="input")
    p = fp.plan
    if xt.shape[1] != p.q:
        raise DimensionError(
            f"cannot multiply {xt.shape[0]}x{xt.shape[1]} by compressed {p.q}x{p.r_dim}")
    fused = mma == "bf16_fused"  # the single fused kernel (comparison / its own tests)
    code = resolve_mma("bf16" if fused else mma, xt, p)
    y = torch.empty((xt.shape[0], p.r_dim), dtype=out_dtype, device=device())
    forward_into(xt, fp, bias, _act_code(activation), act_arg, y, code, fused=fused)
    return (y.float().cpu().numpy() if host else y), xt.shape[0]


def fused_matmul(x, fp: FactorPair, *, reuse: ReuseTable | None = None, threads: int | None = None,
                 mma: str | None = None, out_dtype=torch.float32):
    """kernel.py:222-293: Y = X @ decompress(fp) computed from the factors.

    Returns (y, OpCount). OpCount / ReuseTable report the run-memoized
    algorithm's counts exactly as the reference does (kernel.py:277-283).
    """
    _resolve_threads(threads)
    y, batch = _forward(x, fp, None, "identity", 0.0, mma, out_dtype)
    if reuse is not None:
        pred = predict_reuse(fp.plan)
        reuse.misses += pred.distinct_runs * batch
        reuse.hits += pred.total_runs * batch - pred.distinct_runs * batch
    return y, op_count(fp.plan, batch)


def layer_forward(x, fp: FactorPair, bias, activation: str = "identity", *,
                  threads: int | None = None, mma: str | None = None, act_arg: float = 20.0,
                  out_dtype=torch.float32):
    """kernel.py:296-320: activation(X @ W + bias), fused at every rank."""
    _resolve_threads(threads)
    _act_code(activation)
    b = as_device_vector(bias, fp.plan.r_dim)
    y, _ = _forward(x, fp, b, activation, act_arg, mma, out_dtype)
    return y
