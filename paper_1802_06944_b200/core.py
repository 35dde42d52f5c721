"""Validation gate, deterministic seeding and parity metrics (reference core.py:21-95).

Seeding is host logic and reproduces the reference streams exactly
(SeedSequence → PCG64, scale-after-draw). Operands are moved to the current
CUDA device; there is no CPU compute path.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import ArgumentError, CudaError, DimensionError

FLOAT32 = np.float32
FLOAT64 = np.float64


def make_rng(seed: int) -> np.random.Generator:
    """core.py:39-41."""
    return np.random.default_rng(np.random.SeedSequence(seed))


def spawn_rngs(seed: int, count: int) -> list[np.random.Generator]:
    """core.py:44-51."""
    return [np.random.default_rng(c) for c in np.random.SeedSequence(seed).spawn(count)]


def sample_normal(rng: np.random.Generator, mean: float, stddev: float, shape) -> np.ndarray:
    """core.py:54-60."""
    if stddev < 0:
        raise ArgumentError(f"stddev must be >= 0, got {stddev}")
    return rng.standard_normal(shape) * stddev + mean


def _np(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().float().cpu().numpy() if a.dtype == torch.bfloat16 else a.detach().cpu().numpy()
    return np.asarray(a)


def max_abs_diff(a, b) -> float:
    """core.py:80-88."""
    a, b = _np(a), _np(b)
    if a.shape != b.shape:
        return float("inf")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a.astype(FLOAT64) - b.astype(FLOAT64))))


def rel_error(actual, expected) -> float:
    """core.py:91-95 — max|a-e| / max|e|, the parity metric."""
    e = _np(expected).astype(FLOAT64)
    scale = float(np.max(np.abs(e))) if e.size else 0.0
    return max_abs_diff(actual, e) / (scale if scale > 0 else 1.0)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise CudaError("no CUDA device visible: the DeepThin kernels are sm_100a-only "
                        "and there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_device_matrix(a, *, name: str = "matrix", check_finite: bool | None = None,
                     keep_bf16: bool = True) -> tuple[torch.Tensor, bool]:
    """Validate like core.as_matrix (2-D, finite, float) and return a contiguous CUDA tensor.

    numpy inputs are checked for non-finite entries (ArgumentError) as the
    reference does; CUDA tensors skip the scan unless ``check_finite`` (it would
    force a host sync). float64 is narrowed to float32 — the widest type the
    kernels compute in. Returns (tensor, came_from_numpy).
    """
    from_np = not isinstance(a, torch.Tensor)
    if from_np:
        arr = np.asarray(a)
        if arr.ndim != 2:
            raise DimensionError(f"{name} must be 2-D, got shape {arr.shape}")
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        if (check_finite is None or check_finite) and not np.all(np.isfinite(arr)):
            raise ArgumentError(f"{name} contains non-finite entries")
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32))
        return t.to(device(), non_blocking=False), True
    t = a
    if t.dim() != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {tuple(t.shape)}")
    if t.dtype not in (torch.float32, torch.bfloat16) or (t.dtype == torch.bfloat16 and not keep_bf16):
        t = t.float()
    if t.device.type != "cuda":
        t = t.to(device())
    t = t.contiguous()
    if check_finite and not bool(torch.isfinite(t).all()):
        raise ArgumentError(f"{name} contains non-finite entries")
    return t, False


def as_device_vector(a, length: int, name: str = "bias") -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a.detach().reshape(-1).float()
        t = t.to(device()) if t.device.type != "cuda" else t
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel(),
                                                  dtype=np.float32)).to(device())
    if t.numel() != length:
        raise DimensionError(f"{name} length {t.numel()} != output width {length}")
    return t.contiguous()


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())


def _operand_view(t: torch.Tensor):
    """(base tensor, pitch in elements, transposed?) of a 2-D CUDA view the tensor cores can read
    in place: row-major (stride (ld, 1)) or a transposed row-major view (stride (1, ld))."""
    if t.stride(1) == 1 and t.stride(0) >= max(1, t.shape[1]):
        return t, t.stride(0), False
    if t.stride(0) == 1 and t.stride(1) >= max(1, t.shape[0]):
        return t, t.stride(1), True
    t = t.contiguous()
    return t, t.shape[1], False


def matmul(a, b, *, mma: str = "tf32"):
    """core.py:63-77 matmul on the tcgen05 tensor cores (dt_matmul): 2-D operands, shape check
    with the reference's DimensionError text, fp32 accumulate. ``mma="tf32"`` multiplies in tf32
    (fp32 inputs), ``"bf16"`` in bf16. Transposed views (``x.t()``) are read in place — the
    backward's gᵀ·P and H'ᵀ·x' contractions need no transpose copy. numpy inputs return numpy
    (float32); CUDA tensors return a CUDA float32 tensor."""
    from . import _lib
    host = not isinstance(a, torch.Tensor) or not isinstance(b, torch.Tensor)
    at = a if isinstance(a, torch.Tensor) else as_device_matrix(a, name="left operand")[0]
    bt = b if isinstance(b, torch.Tensor) else as_device_matrix(b, name="right operand")[0]
    if at.dim() != 2 or bt.dim() != 2:
        raise DimensionError("matmul operands must be 2-D")
    if at.shape[1] != bt.shape[0]:
        raise DimensionError(f"cannot multiply {at.shape[0]}x{at.shape[1]} by "
                             f"{bt.shape[0]}x{bt.shape[1]}")
    if mma not in ("tf32", "bf16"):
        raise ArgumentError(f"mma must be 'tf32' or 'bf16', got {mma!r}")
    dt = torch.float32 if mma == "tf32" else torch.bfloat16
    code = _lib.DT_F32 if mma == "tf32" else _lib.DT_BF16
    at = at.to(device=device(), dtype=dt)
    bt = bt.to(device=device(), dtype=dt)
    M, K = at.shape
    N = bt.shape[1]
    av, lda, ta = _operand_view(at)
    bv, ldb, tb = _operand_view(bt)
    esz = 4 if mma == "tf32" else 2
    # TMA needs 16-byte pitches and bases: re-pack the rare operand that is not
    if (lda * esz) % 16 or av.data_ptr() % 16:
        av = _padded(at, esz)
        lda, ta = av.stride(0), False
    if (ldb * esz) % 16 or bv.data_ptr() % 16:
        bv = _padded(bt, esz)
        ldb, tb = bv.stride(0), False
    ldc = -(-N * 4 // 16) * 16 // 4
    c = torch.empty((M, ldc), dtype=torch.float32, device=device())
    lib = _lib.lib()
    ws = workspace(lib.dt_matmul_workspace_bytes(M, N, K, code))
    _lib.check(lib.dt_matmul(M, N, K, av.data_ptr(), lda, int(ta), bv.data_ptr(), ldb, int(tb), code,
                             c.data_ptr(), ldc, ws.data_ptr(), ws.numel(), stream_handle()))
    c = c[:, :N]
    return c.cpu().numpy() if host else c


def _padded(t: torch.Tensor, esz: int) -> torch.Tensor:
    """Row-major copy of t with a 16-byte-aligned pitch (zero padding)."""
    cols = -(-t.shape[1] * esz // 16) * 16 // esz
    out = torch.zeros((t.shape[0], cols), dtype=t.dtype, device=t.device)
    out[:, : t.shape[1]].copy_(t)
    return out
