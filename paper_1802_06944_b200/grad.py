"""Backward through a compressed layer on the GPU (reference grad.py:23-116).

``layer_backward`` mirrors grad.py:63-95: gradients w.r.t. both factors,
the input and the bias, through the activation, the contraction, the
inverse re-layout (the discarded tail gets zero gradient) and the factor
product — computed by dt_backward without materialising W.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import as_device_matrix, as_device_vector, device, stream_handle, workspace
from .errors import ArgumentError, DimensionError
from .factor import FactorPair
from .kernel import ACTIVATIONS, EXTRA_ACTIVATIONS, _act_code

LOSSES = ("mse", "softmax_cross_entropy")


@dataclass
class Gradients:
    """grad.py:23-28."""

    d_xf: object
    d_wf: object
    d_input: object
    d_bias: object


def backward_into(x: torch.Tensor, fp: FactorPair, bias, act: int, act_arg: float,
                  upstream: torch.Tensor, d_xf: torch.Tensor, d_wf: torch.Tensor,
                  d_bias: torch.Tensor | None, d_input: torch.Tensor | None, mma: int,
                  p_in: torch.Tensor | None = None) -> None:
    """Raw stream-ordered dt_backward(_ex) on device tensors; p_in: the P the forward kept."""
    p = fp.plan
    lib = _lib.lib()
    ps = _lib.plan_struct(p)
    batch = x.shape[0]
    ws = workspace(lib.dt_backward_workspace_bytes(C.byref(ps), batch, mma))
    _lib.check(lib.dt_backward_ex(
        C.byref(ps), batch, mma, x.data_ptr(),
        _lib.DT_BF16 if x.dtype == torch.bfloat16 else _lib.DT_F32,
        fp.xf.data_ptr(), fp.wf.data_ptr(), bias.data_ptr() if bias is not None else None,
        act, float(act_arg), upstream.data_ptr(), d_xf.data_ptr(), d_wf.data_ptr(),
        d_bias.data_ptr() if d_bias is not None else None,
        d_input.data_ptr() if d_input is not None else None,
        p_in.data_ptr() if p_in is not None else None,
        ws.data_ptr(), ws.numel(), stream_handle()))


def layer_backward(x, fp: FactorPair, bias, activation: str, upstream, *, act_arg: float = 20.0,
                   mma: str = "ffma", need_input_grad: bool = True) -> Gradients:
    """grad.py:63-95: Gradients(d_xf, d_wf, d_input, d_bias) of one compressed layer."""
    if activation not in ACTIVATIONS + EXTRA_ACTIVATIONS or activation == "softmax":
        raise ArgumentError(f"unknown activation {activation!r}")
    xt, host = as_device_matrix(x, name="input")
    up, _ = as_device_matrix(upstream, name="upstream", keep_bf16=False)
    p = fp.plan
    if xt.shape[1] != p.q:
        raise DimensionError(f"input width {xt.shape[1]} != layer input width {p.q}")
    if tuple(up.shape) != (xt.shape[0], p.r_dim):
        raise DimensionError(
            f"upstream shape {tuple(up.shape)} != layer output shape {(xt.shape[0], p.r_dim)}")
    b = as_device_vector(bias, p.r_dim)
    dev = device()
    d_xf = torch.empty((p.m, p.rank), dtype=torch.float32, device=dev)
    d_wf = torch.empty((p.rank, p.n), dtype=torch.float32, device=dev)
    d_b = torch.empty((p.r_dim,), dtype=torch.float32, device=dev)
    d_in = torch.empty((xt.shape[0], p.q), dtype=torch.float32, device=dev) if need_input_grad else None
    code = _lib.DT_MMA_BF16 if mma == "bf16" else _lib.DT_MMA_FFMA
    backward_into(xt, fp, b, _act_code(activation), act_arg, up, d_xf, d_wf, d_b, d_in, code)
    if host:
        cv = lambda t: None if t is None else t.cpu().numpy()
        return Gradients(cv(d_xf), cv(d_wf), cv(d_in), cv(d_b))
    return Gradients(d_xf, d_wf, d_in, d_b)


def mse_grad_into(y: torch.Tensor, target: torch.Tensor, grad: torch.Tensor,
                  norm_count: float, loss_sum: torch.Tensor | None = None) -> None:
    """grad.py:100-103 on device: grad = 2 (y - t) / norm_count; loss_sum = sum (y - t)^2 (fp64).

    ``norm_count`` is the GLOBAL y.size when the batch is sharded over ranks.
    """
    lib = _lib.lib()
    rows, cols = y.shape
    ws = workspace(lib.dt_mse_workspace_bytes(rows, cols))
    _lib.check(lib.dt_mse_grad(rows, cols, y.data_ptr(), target.data_ptr(), float(norm_count),
                               grad.data_ptr(),
                               loss_sum.data_ptr() if loss_sum is not None else None,
                               ws.data_ptr(), ws.numel(), stream_handle()))


def loss_and_grad(name: str, y, target):
    """grad.py:98-116: (scalar loss, dLoss/dY)."""
    if name == "mse":
        yt, host = as_device_matrix(y, name="y", keep_bf16=False)
        tt, _ = as_device_matrix(target, name="target", keep_bf16=False)
        if tt.shape != yt.shape:
            raise DimensionError(f"target shape {tuple(tt.shape)} != {tuple(yt.shape)}")
        g = torch.empty_like(yt)
        ls = torch.empty(1, dtype=torch.float64, device=yt.device)
        mse_grad_into(yt, tt, g, float(yt.numel()), ls)
        loss = float(ls.item()) / yt.numel()
        return loss, (g.cpu().numpy() if host else g)
    if name == "softmax_cross_entropy":
        # glue, not the hot path: plain torch ops on the device
        yt, host = as_device_matrix(y, name="y", keep_bf16=False)
        labels = torch.as_tensor(np.asarray(target) if not isinstance(target, torch.Tensor) else target,
                                 device=yt.device).long()
        z = yt - yt.max(dim=1, keepdim=True).values
        probs = torch.softmax(z, dim=1)
        batch = yt.shape[0]
        picked = probs[torch.arange(batch, device=yt.device), labels].clamp_min(1e-30)
        grad = probs.clone()
        grad[torch.arange(batch, device=yt.device), labels] -= 1.0
        grad /= batch
        loss = float(-torch.log(picked).mean())
        return loss, (grad.cpu().numpy() if host else grad)
    raise ArgumentError(f"loss must be one of {LOSSES}, got {name!r}")
