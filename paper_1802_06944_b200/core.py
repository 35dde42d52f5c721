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
