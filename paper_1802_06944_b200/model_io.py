"""The ``.dthn`` compressed-model format (reference model_io.py:1-224), indexed natively.

Drop-in for the reference's ``CompressedModel`` / ``expected_file_size`` / ``serialize`` /
``deserialize`` / ``save_model`` / ``load_model``: the same byte layout, validation order, error
messages and failing-byte offsets, and bit-exact round trips.

B200 side of the design. ``deserialize`` does not walk the bytes in Python: the native parser
(``dt_model_parse``, csrc/dt_model.cu) validates the whole image and returns an index of byte
offsets (names, metadata strings, payloads). The host arrays are views materialised from those
offsets, and ``CompressedModel.to_device`` (model.py) ships the *image itself* to HBM with one
pinned host→device copy and decodes every payload on the GPU (``dt_unpack_values``) into
aligned fp32 masters plus bf16 operand copies — no per-layer host conversion or copy.

Layout (little-endian; model_io.py:1-25): header ``<4sIIQd`` (magic b"DTHN", version 1, layer
count, payload byte count, target ratio) | metadata: u32 count, then u32-length-prefixed utf-8
key and value | per layer: u32-length-prefixed utf-8 name, u64 q r_dim rank m n, u8 dtype code
(0 float32, 1 float64), u8 floor-hit flag, u64 bias length, xf (m*rank), wf (rank*n) and bias
payloads in the layer's dtype.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from .errors import ArgumentError, ModelFormatError
from .planner import LayerPlan, NetworkPlan

MAGIC = b"DTHN"
FORMAT_VERSION = 1
HEADER_BYTES = 28                      # struct "<4sIIQd"
LAYER_FIXED_BYTES = 4 + 5 * 8 + 2 + 8  # name length, plan, dtype + flag, bias length
_STORED = (np.dtype(np.float32), np.dtype(np.float64))  # index = dtype code


@dataclass(frozen=True)
class StoredFactors:
    """One layer's factors in their stored dtype, host side (the serialized content of the
    reference FactorPair, factor.py:23-57, whose copies are read-only too, :42-50).
    ``to_device`` turns them into device FactorPairs."""

    xf: np.ndarray
    wf: np.ndarray
    plan: LayerPlan

    def __post_init__(self):
        for label in ("xf", "wf"):
            a = np.array(getattr(self, label), copy=True)
            a.flags.writeable = False
            object.__setattr__(self, label, a)

    @property
    def dtype(self):
        return self.xf.dtype


@dataclass
class CompressedModel:
    """Plans, factors, biases and metadata of one network (reference model_io.py:46-63).

    ``factors`` may hold StoredFactors (what ``deserialize`` returns) or device FactorPairs.
    """

    plans: NetworkPlan
    factors: list
    biases: list
    metadata: dict = field(default_factory=dict)
    format_version: int = FORMAT_VERSION
    _image: bytes | None = field(default=None, repr=False, compare=False)
    _index: list | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        n = len(self.plans.layers)
        if n != len(self.factors) or n != len(self.biases):
            raise ArgumentError("factors and biases must match the plan's layer count")
        self.biases = [np.ascontiguousarray(_host(b)).ravel() for b in self.biases]

    @property
    def layer_names(self) -> list:
        return [name for name, _ in self.plans.layers]

    def image(self) -> tuple[bytes, list]:
        """The serialized bytes and their per-layer index. A model that came from
        ``deserialize`` reuses its source image while it still describes the model (same
        plans, metadata and read-only factor objects, equal biases); otherwise re-serialize."""
        if self._image is None or not self._image_current():
            data = serialize(self)
            self._index = [rec for _, rec in _parse(data)[2]]
            self._image = data
            self._stamp = self._snapshot()
        return self._image, self._index

    def _snapshot(self):
        return (id(self.plans), tuple(map(id, self.factors)), dict(self.metadata),
                self.format_version)

    def _image_current(self) -> bool:
        if getattr(self, "_stamp", None) != self._snapshot():
            return False
        # only read-only factors can be trusted unchanged (device FactorPairs are updated in
        # place by SGD under the same Python object)
        if not all(isinstance(fp, StoredFactors) for fp in self.factors):
            return False
        for rec, bias in zip(self._index, self.biases):
            dt = _STORED[rec.dtype_code]
            stored = np.frombuffer(self._image, dtype=dt, count=rec.bias_len, offset=rec.bias_offset)
            if bias.dtype != dt or not np.array_equal(stored.view(np.uint8), bias.view(np.uint8)):
                return False
        return True

    def to_device(self, activations=None, *, mma: str = "bf16", act_args=None,
                  pipeline: bool = True):
        """Device-resident network (model.DeviceModel) that runs on the GPU kernels."""
        from .model import DeviceModel
        return DeviceModel(self, activations=activations, mma=mma, act_args=act_args,
                           pipeline=pipeline)


def _host(a) -> np.ndarray:
    if hasattr(a, "detach"):  # a device tensor (FactorPair fields, torch biases)
        return a.detach().cpu().numpy()
    return np.asarray(a)


def _stored_dtype(fp) -> np.dtype:
    if hasattr(fp, "source_dtype"):  # device FactorPair: the dtype its source had
        return fp.source_dtype
    return np.dtype(_host(fp.xf[:0]).dtype) if hasattr(fp.xf, "detach") else np.dtype(fp.dtype)


def _factor_values(fp):
    return fp.host_values() if hasattr(fp, "host_values") else (fp.xf, fp.wf)


def _layer_bytes(name: str, plan: LayerPlan, item: int, bias_len: int) -> int:
    return (LAYER_FIXED_BYTES + len(name.encode()) + item * plan.rank * (plan.m + plan.n)
            + item * bias_len)


def _metadata_bytes(metadata: dict) -> int:
    return 4 + sum(8 + len(k.encode()) + len(v.encode()) for k, v in metadata.items())


def expected_file_size(model: CompressedModel) -> int:
    """Byte-exact file size from the plan accounting (reference model_io.py:66-81)."""
    total = HEADER_BYTES + _metadata_bytes(model.metadata)
    for (name, plan), fp, bias in zip(model.plans.layers, model.factors, model.biases):
        total += _layer_bytes(name, plan, _stored_dtype(fp).itemsize, bias.size)
    return total


def serialize(model: CompressedModel) -> bytes:
    """Encode ``model`` (reference model_io.py:84-119) into one preallocated buffer: the
    size is known up front (expected_file_size), payloads are written in place."""
    floors = set(model.plans.floor_hits)
    dtypes = []
    for (name, plan), fp in zip(model.plans.layers, model.factors):
        if fp.plan != plan:
            raise ArgumentError(f"factor pair for {name!r} does not match its plan")
        dt = _stored_dtype(fp)
        if dt not in _STORED:
            raise ArgumentError(f"unsupported dtype {dt} for layer {name!r}")
        dtypes.append(dt)
    buf = bytearray(expected_file_size(model))
    pos = HEADER_BYTES

    def put_bytes(raw: bytes):
        nonlocal pos
        struct.pack_into("<I", buf, pos, len(raw))
        buf[pos + 4:pos + 4 + len(raw)] = raw
        pos += 4 + len(raw)

    def put_array(values, dt: np.dtype):
        nonlocal pos
        flat = np.ascontiguousarray(_host(values), dtype=dt).ravel()
        np.frombuffer(buf, dtype=dt, count=flat.size, offset=pos)[:] = flat
        pos += flat.nbytes

    struct.pack_into("<I", buf, pos, len(model.metadata))
    pos += 4
    for key, value in model.metadata.items():
        put_bytes(key.encode())
        put_bytes(value.encode())
    for (name, plan), fp, bias, dt in zip(model.plans.layers, model.factors, model.biases, dtypes):
        put_bytes(name.encode())
        struct.pack_into("<5QBBQ", buf, pos, plan.q, plan.r_dim, plan.rank, plan.m, plan.n,
                         _STORED.index(dt), int(name in floors), bias.size)
        pos += 5 * 8 + 2 + 8
        xv, wv = _factor_values(fp)
        put_array(xv, dt)
        put_array(wv, dt)
        put_array(bias, dt)
    assert pos == len(buf)
    struct.pack_into("<4sIIQd", buf, 0, MAGIC, model.format_version, len(model.factors),
                     len(buf) - HEADER_BYTES, model.plans.target_ratio)
    return bytes(buf)


# ---- parsing ---------------------------------------------------------------------------------

def _parse(data: bytes):
    """dt_model_parse twice (count, then fill); strings decoded in file order exactly as the
    reference decodes them while reading (a bad utf-8 name fails before any later check);
    native format errors become the reference's ModelFormatError text."""
    lib = _lib.lib()
    size = len(data)
    hdr, err = _lib.ModelHeader(), _lib.FormatError()
    rc = lib.dt_model_parse(data, size, C.byref(hdr), None, 0, None, 0, C.byref(err))
    meta = (_lib.ModelMeta * max(hdr.meta_read, 1))()
    layers = (_lib.ModelLayer * max(hdr.layers_read, 1))()
    if rc in (_lib.DT_OK, _lib.DT_E_FORMAT):
        rc = lib.dt_model_parse(data, size, C.byref(hdr), meta, hdr.meta_read, layers,
                                hdr.layers_read, C.byref(err))
    if rc not in (_lib.DT_OK, _lib.DT_E_FORMAT):
        _lib.check(rc)

    def text(span):
        return data[span.offset:span.offset + span.length].decode()

    metadata = {}
    for rec in meta[:hdr.meta_read]:
        if rec.key.length < 0:
            break
        key = text(rec.key)
        if rec.value.length < 0:
            break
        metadata[key] = text(rec.value)
    names = []
    for rec in layers[:hdr.layers_read]:
        if rec.name.length < 0:
            break
        names.append(text(rec.name))
    if rc == _lib.DT_E_FORMAT:
        raise ModelFormatError(_format_message(data, hdr, err, layers, names), err.offset)
    return hdr, metadata, [(names[i], layers[i]) for i in range(hdr.layers_read)]


_WHAT = {
    _lib.DT_WHAT_HEADER: "header", _lib.DT_WHAT_META_COUNT: "metadata count",
    _lib.DT_WHAT_META_KEY_LEN: "metadata key length", _lib.DT_WHAT_META_KEY: "metadata key",
    _lib.DT_WHAT_META_VALUE_LEN: "metadata value length",
    _lib.DT_WHAT_META_VALUE: "metadata value",
}
_LAYER_WHAT = {
    _lib.DT_WHAT_PLAN: "plan", _lib.DT_WHAT_FLAGS: "flags",
    _lib.DT_WHAT_BIAS_LEN: "bias length", _lib.DT_WHAT_XF: "xf payload",
    _lib.DT_WHAT_WF: "wf payload", _lib.DT_WHAT_BIAS: "bias payload",
}


def _u64(v: int) -> int:
    return v & 0xFFFFFFFFFFFFFFFF


def _format_message(data, hdr, err, layers, names) -> str:
    kind = err.kind
    if kind == _lib.DT_FMT_BAD_MAGIC:
        return f"bad magic {bytes(data[:4])!r}, expected {MAGIC!r}"
    if kind == _lib.DT_FMT_BAD_VERSION:
        return f"unsupported format version {err.need}"
    if kind == _lib.DT_FMT_PAYLOAD_MISMATCH:
        return f"declared payload of {_u64(err.need)} bytes but file carries {err.have}"
    if kind == _lib.DT_FMT_BAD_DTYPE:
        return f"unknown dtype code {err.need}"
    if kind == _lib.DT_FMT_TRAILING:
        return f"{err.need} trailing bytes after last layer"
    if kind == _lib.DT_FMT_INVALID_PLAN:
        p = layers[err.layer].plan
        try:
            LayerPlan(q=_u64(p.q), r_dim=_u64(p.r_dim), rank=_u64(p.rank), m=_u64(p.m),
                      n=_u64(p.n))
            reason = "invalid plan"
        except ArgumentError as exc:
            reason = str(exc)
        return f"invalid plan for layer {names[err.layer]!r}: {reason}"
    # truncation: reconstruct the reader's label and the exact byte count asked for
    need = err.need
    if err.what in _WHAT:
        what = _WHAT[err.what]
    elif err.what == _lib.DT_WHAT_NAME_LEN:
        what = f"layer {err.layer} name length"
    elif err.what == _lib.DT_WHAT_NAME:
        what = f"layer {err.layer} name"
    else:
        what = f"layer {names[err.layer]!r} {_LAYER_WHAT[err.what]}"
        rec = layers[err.layer]
        item = _STORED[rec.dtype_code].itemsize if rec.dtype_code in (0, 1) else 0
        rank, m, n = _u64(rec.plan.rank), _u64(rec.plan.m), _u64(rec.plan.n)
        need = {_lib.DT_WHAT_XF: m * rank * item, _lib.DT_WHAT_WF: rank * n * item,
                _lib.DT_WHAT_BIAS: _u64(rec.bias_len) * item}.get(err.what, need)
    return f"truncated while reading {what}: need {need} bytes, have {err.have}"


def deserialize(data: bytes) -> CompressedModel:
    """Parse a serialized model (reference model_io.py:141-210); a failure raises
    ModelFormatError carrying the exact failing byte offset."""
    data = bytes(data)
    hdr, metadata, index = _parse(data)
    layers, factors, biases, floors = [], [], [], []
    for name, rec in index:
        p = rec.plan
        plan = LayerPlan(q=p.q, r_dim=p.r_dim, rank=p.rank, m=p.m, n=p.n)
        dt = _STORED[rec.dtype_code]

        def view(offset, count):
            return np.frombuffer(data, dtype=dt, count=count, offset=offset).copy()

        xf = view(rec.xf_offset, plan.m * plan.rank).reshape(plan.m, plan.rank)
        wf = view(rec.wf_offset, plan.rank * plan.n).reshape(plan.rank, plan.n)
        layers.append((name, plan))
        factors.append(StoredFactors(xf=xf, wf=wf, plan=plan))
        biases.append(view(rec.bias_offset, rec.bias_len))
        if rec.floor_hit:
            floors.append(name)
    bias_total = sum(b.size for b in biases)
    stored = sum(p.compressed_elems for _, p in layers) + bias_total
    dense = sum(p.original_elems for _, p in layers) + bias_total
    plans = NetworkPlan(layers=tuple(layers), target_ratio=hdr.target_ratio,
                        achieved_total_ratio=float(Fraction(stored, dense)) if dense else 0.0,
                        floor_hits=tuple(floors), bias_counts=tuple(b.size for b in biases))
    model = CompressedModel(plans=plans, factors=factors, biases=biases, metadata=metadata,
                            format_version=hdr.version, _image=data,
                            _index=[rec for _, rec in index])
    model._stamp = model._snapshot()
    return model


def save_model(model: CompressedModel, path) -> int:
    """Write ``model`` to ``path``; returns the bytes written (reference model_io.py:213-218)."""
    data = serialize(model)
    with open(path, "wb") as fh:
        fh.write(data)
    return len(data)


def load_model(path) -> CompressedModel:
    """Read a file written by save_model (reference model_io.py:221-224)."""
    with open(path, "rb") as fh:
        return deserialize(fh.read())
