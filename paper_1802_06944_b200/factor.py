"""The compressed representation on the GPU (reference factor.py:23-110).

A FactorPair owns private, device-resident fp32 copies of the factors (the
reference's private read-only copies, factor.py:42-50) plus lazily cached
bf16 operand copies for the tensor-core path (the analogue of the per-pair
cached combine weights, kernel.py:157-164).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .core import as_device_matrix, device, sample_normal, stream_handle
from .errors import ArgumentError, DimensionError
from .planner import LayerPlan


@dataclass(frozen=True)
class FactorPair:
    """Learnable factors (xf: m x rank, wf: rank x n) plus their plan; device-resident."""

    xf: torch.Tensor
    wf: torch.Tensor
    plan: LayerPlan
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        host = not isinstance(self.xf, torch.Tensor)
        # the reference keeps float64 factors as float64 (core.as_matrix, factor.py:42-50) and
        # serializes them as such (model_io.py:100-110): remember the source dtype, and for
        # float64 sources a host float64 copy, so an untrained pair round-trips bit-exactly
        src = _source_dtype(self.xf, self.wf)
        if src == np.float64:
            self._cache["source64"] = tuple(
                np.array(_host64(a), dtype=np.float64, copy=True) for a in (self.xf, self.wf))
        self._cache["source_dtype"] = src
        xf, _ = as_device_matrix(self.xf, name="xf", keep_bf16=False)
        wf, _ = as_device_matrix(self.wf, name="wf", keep_bf16=False)
        p = self.plan
        if tuple(xf.shape) != (p.m, p.rank):
            raise DimensionError(f"xf must be {p.m}x{p.rank}, got {xf.shape[0]}x{xf.shape[1]}")
        if tuple(wf.shape) != (p.rank, p.n):
            raise DimensionError(f"wf must be {p.rank}x{p.n}, got {wf.shape[0]}x{wf.shape[1]}")
        # private copies: never alias (or later see edits to) the caller's buffers
        object.__setattr__(self, "xf", xf.clone() if xf.data_ptr() == _ptr(self.xf) else xf)
        object.__setattr__(self, "wf", wf.clone() if wf.data_ptr() == _ptr(self.wf) else wf)
        self._cache["host"] = host

    @classmethod
    def adopt(cls, xf: torch.Tensor, wf: torch.Tensor, plan: LayerPlan,
              bf16: tuple | None = None) -> "FactorPair":
        """Take ownership of freshly made contiguous fp32 CUDA factors (no private copy: the
        caller hands them over), optionally with their bf16 operand copies."""
        if tuple(xf.shape) != (plan.m, plan.rank) or tuple(wf.shape) != (plan.rank, plan.n):
            raise DimensionError(f"factors {tuple(xf.shape)} / {tuple(wf.shape)} do not match "
                                 f"the plan ({plan.m}x{plan.rank}, {plan.rank}x{plan.n})")
        for t in (xf, wf):
            if t.dtype != torch.float32 or t.device.type != "cuda" or not t.is_contiguous():
                raise ArgumentError("adopted factors must be contiguous fp32 CUDA tensors")
        fp = cls.__new__(cls)
        object.__setattr__(fp, "xf", xf)
        object.__setattr__(fp, "wf", wf)
        object.__setattr__(fp, "plan", plan)
        object.__setattr__(fp, "_cache", {"host": False})
        if bf16 is not None:
            fp._cache["bf16"] = tuple(bf16)
        return fp

    @property
    def dtype(self):
        return self.xf.dtype

    @property
    def from_numpy(self) -> bool:
        return bool(self._cache.get("host", False))

    def with_values(self, xf, wf) -> "FactorPair":
        return FactorPair(xf=xf, wf=wf, plan=self.plan)

    def bf16(self) -> tuple[torch.Tensor, torch.Tensor]:
        """bf16 (RNE) copies of the factors, made once per pair by dt_cast_bf16."""
        if "bf16" not in self._cache:
            lib = _lib.lib()
            out = []
            for t in (self.xf, self.wf):
                o = torch.empty(t.shape, dtype=torch.bfloat16, device=t.device)
                _lib.check(lib.dt_cast_bf16(t.numel(), t.data_ptr(), o.data_ptr(), stream_handle()))
                out.append(o)
            self._cache["bf16"] = tuple(out)
        return self._cache["bf16"]

    def packed(self):
        """Regeneration operands for the bf16 tensor-core general path (dt_pack_factors),
        made once per pair; None where that path does not use them (reuse geometries)."""
        if "packed" not in self._cache:
            lib = _lib.lib()
            ps = _lib.plan_struct(self.plan)
            nbytes = lib.dt_packed_factors_bytes(C.byref(ps), _lib.DT_MMA_BF16)
            buf = None
            if nbytes:
                xf16, wf16 = self.bf16()
                buf = torch.empty(nbytes, dtype=torch.uint8, device=self.xf.device)
                _lib.check(lib.dt_pack_factors(C.byref(ps), _lib.DT_MMA_BF16, xf16.data_ptr(),
                                               wf16.data_ptr(), buf.data_ptr(), stream_handle()))
            self._cache["packed"] = buf
        return self._cache["packed"]

    def rows_prepared(self, bias, act: int, y_dtype: int):
        """Row-tile reuse kernel operands (dt_rows_prepare: bf16 wf, K-padded XF2 with the bias
        and the activation pre-scale folded in), derived once per (pair, bias, activation,
        output dtype) like the reference's per-pair derived weights (kernel.py:157-164).
        None when the geometry does not take that kernel."""
        key = ("rows", act, y_dtype, bias.data_ptr() if bias is not None else 0)
        if key not in self._cache:
            lib = _lib.lib()
            ps = _lib.plan_struct(self.plan)
            nbytes = lib.dt_rows_prepared_bytes(C.byref(ps), _lib.DT_BF16, y_dtype)
            buf = None
            if nbytes:
                buf = torch.empty(nbytes, dtype=torch.uint8, device=self.xf.device)
                _lib.check(lib.dt_rows_prepare(C.byref(ps), act, y_dtype, self.xf.data_ptr(),
                                               self.wf.data_ptr(),
                                               bias.data_ptr() if bias is not None else None,
                                               buf.data_ptr(), stream_handle()))
            self._cache[key] = (buf, bias)
        return self._cache[key][0]

    @property
    def source_dtype(self) -> np.dtype:
        """The dtype the reference would hold these factors in (float32 or float64)."""
        return np.dtype(self._cache.get("source_dtype", np.float32))

    def host_values(self) -> tuple[np.ndarray, np.ndarray]:
        """(xf, wf) in source_dtype for serialization: the untouched float64 source while the
        device masters were never updated, else the device values widened."""
        if "source64" in self._cache:
            return self._cache["source64"]
        dt = self.source_dtype
        return tuple(t.detach().float().cpu().numpy().astype(dt) for t in (self.xf, self.wf))

    def refresh_derived(self) -> None:
        """Re-derive the cached bf16 / packed copies after the fp32 masters changed (SGD)."""
        self._cache.pop("source64", None)  # the masters moved on from the float64 source
        lib = _lib.lib()
        if "bf16" in self._cache:
            for src, dst in zip((self.xf, self.wf), self._cache["bf16"]):
                _lib.check(lib.dt_cast_bf16(src.numel(), src.data_ptr(), dst.data_ptr(),
                                            stream_handle()))
        for key in [k for k in self._cache if isinstance(k, tuple) and k[0] == "rows"]:
            buf, bias = self._cache[key]
            if buf is not None:
                _lib.check(lib.dt_rows_prepare(
                    C.byref(_lib.plan_struct(self.plan)), key[1], key[2], self.xf.data_ptr(),
                    self.wf.data_ptr(), bias.data_ptr() if bias is not None else None,
                    buf.data_ptr(), stream_handle()))
        if self._cache.get("packed") is not None:
            xf16, wf16 = self._cache["bf16"]
            _lib.check(lib.dt_pack_factors(C.byref(_lib.plan_struct(self.plan)), _lib.DT_MMA_BF16,
                                           xf16.data_ptr(), wf16.data_ptr(),
                                           self._cache["packed"].data_ptr(), stream_handle()))


def _ptr(a) -> int:
    return a.data_ptr() if isinstance(a, torch.Tensor) else -1


def init_factors(plan: LayerPlan, sigma: float, rng: np.random.Generator) -> FactorPair:
    """factor.py:60-71: xf ~ N(0, sigma^2), wf ~ N(0, 1/rank), drawn on the host."""
    if not sigma > 0:
        raise ArgumentError(f"sigma must be > 0, got {sigma}")
    xf = sample_normal(rng, 0.0, sigma, (plan.m, plan.rank))
    wf = sample_normal(rng, 0.0, 1.0 / math.sqrt(plan.rank), (plan.rank, plan.n))
    return FactorPair(xf=xf, wf=wf, plan=plan)


def relayout_index(flat: int, plan: LayerPlan) -> tuple[int, int]:
    """factor.py:74-84 via dt_relayout_index."""
    row, col = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().dt_relayout_index(C.byref(_lib.plan_struct(plan)), int(flat),
                                            C.byref(row), C.byref(col)))
    return row.value, col.value


def phase(col: int, plan: LayerPlan) -> int:
    """factor.py:96-105 via dt_phase."""
    out = C.c_int64()
    _lib.check(_lib.lib().dt_phase(C.byref(_lib.plan_struct(plan)), int(col), C.byref(out)))
    return out.value


def phase_count(plan: LayerPlan) -> int:
    """factor.py:108-110."""
    return int(plan.info().phase_count)


def decompress(fp: FactorPair):
    """factor.py:87-93: materialise the dense q x r_dim W (fp32) on the GPU.

    Debug/oracle helper — the forward and backward never call it. Returns a
    numpy array when the pair was built from numpy, else a CUDA tensor.
    """
    p = fp.plan
    w = torch.empty((p.q, p.r_dim), dtype=torch.float32, device=device())
    _lib.check(_lib.lib().dt_decompress(C.byref(_lib.plan_struct(p)), fp.xf.data_ptr(),
                                        fp.wf.data_ptr(), w.data_ptr(), stream_handle()))
    return w.cpu().numpy() if fp.from_numpy else w


def _source_dtype(*arrays) -> np.dtype:
    """core.as_matrix's dtype rule (core.py:21-36): float32 stays float32 only when every
    input is float32 (bf16 tensors count as float32), anything else is float64."""
    f32 = True
    for a in arrays:
        if isinstance(a, torch.Tensor):
            f32 &= a.dtype in (torch.float32, torch.bfloat16)
        else:
            f32 &= np.asarray(a).dtype == np.float32
    return np.dtype(np.float32 if f32 else np.float64)


def _host64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)
