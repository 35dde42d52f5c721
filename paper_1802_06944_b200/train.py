"""Training step of a compressed layer on the GPU (reference train.py:86-117, 201-230, 305-357).

``DeepThinLayer`` holds fp32 master factors and bias and one flat fp32
gradient buffer [d_xf | d_wf | d_bias] so a data-parallel step needs a
single all-reduce. ``train_step`` is BASELINE config 5's step: forward,
MSE gradient normalised by the global element count, backward through the
inverse re-layout, all-reduce, SGD (train.py:107-111).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .core import as_device_vector, device, stream_handle
from .dist import allreduce_grads
from .factor import FactorPair
from .grad import backward_into, mse_grad_into
from .kernel import _act_code, forward_into
from .planner import LayerPlan


class DeepThinLayer:
    def __init__(self, plan: LayerPlan, xf, wf, bias=None, activation: str = "identity",
                 mma: str = "bf16", act_arg: float = 20.0):
        self.plan = plan
        self.fp = FactorPair(xf, wf, plan)
        self.bias = as_device_vector(np.zeros(plan.r_dim) if bias is None else bias, plan.r_dim).clone()
        self.activation = activation
        self.act = _act_code(activation)
        self.act_arg = act_arg
        self.mma = _lib.DT_MMA_BF16 if mma == "bf16" else _lib.DT_MMA_FFMA
        nx, nw = plan.m * plan.rank, plan.rank * plan.n
        self.grad_flat = torch.zeros(nx + nw + plan.r_dim, dtype=torch.float32, device=device())
        self.d_xf = self.grad_flat[:nx].view(plan.m, plan.rank)
        self.d_wf = self.grad_flat[nx:nx + nw].view(plan.rank, plan.n)
        self.d_bias = self.grad_flat[nx + nw:]
        self._x = None

    def forward(self, x: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
        self._x = x
        y = torch.empty((x.shape[0], self.plan.r_dim), dtype=out_dtype, device=x.device)
        forward_into(x, self.fp, self.bias, self.act, self.act_arg, y, self.mma)
        return y

    def forward_mse(self, x: torch.Tensor, target: torch.Tensor, norm_count: float,
                    loss_out: torch.Tensor) -> torch.Tensor:
        """Forward + MSE gradient in one pass (dt_forward_mse, identity activation, bf16 path):
        returns grad = 2 (y - target) / norm_count; loss_out[0] = sum (y - target)^2. y itself
        is never written (grad.py:98-103 fused into the contraction's epilogue)."""
        self._x = x
        lib = _lib.lib()
        ps = _lib.plan_struct(self.plan)
        batch = x.shape[0]
        from .core import workspace
        ws = workspace(lib.dt_forward_mse_workspace_bytes(C.byref(ps), batch))
        g = torch.empty((batch, self.plan.r_dim), dtype=torch.float32, device=x.device)
        tgt = target.contiguous().float()
        _lib.check(lib.dt_forward_mse(
            C.byref(ps), batch, x.data_ptr(), _lib.DT_BF16 if x.dtype == torch.bfloat16 else _lib.DT_F32,
            self.fp.xf.data_ptr(), self.fp.wf.data_ptr(), self.bias.data_ptr(), tgt.data_ptr(),
            float(norm_count), g.data_ptr(), loss_out.data_ptr(), ws.data_ptr(), ws.numel(),
            stream_handle()))
        return g

    def backward(self, upstream: torch.Tensor, need_input_grad: bool = False):
        d_in = (torch.empty((self._x.shape[0], self.plan.q), dtype=torch.float32, device=self._x.device)
                if need_input_grad else None)
        backward_into(self._x, self.fp, self.bias, self.act, self.act_arg, upstream, self.d_xf,
                      self.d_wf, self.d_bias, d_in, self.mma)
        return d_in

    def step(self, lr: float) -> None:
        """train.py:107-111 + :221: SGD on the fp32 masters, then refresh bf16 operand copies."""
        lib = _lib.lib()
        for p, g in ((self.fp.xf, self.d_xf), (self.fp.wf, self.d_wf), (self.bias, self.d_bias)):
            _lib.check(lib.dt_sgd_step(p.numel(), p.data_ptr(), g.data_ptr(), float(lr),
                                       stream_handle()))
        self.fp.refresh_derived()


def train_step(layer: DeepThinLayer, x: torch.Tensor, target: torch.Tensor, lr: float,
               global_rows: int | None = None, group=None, loss_out: torch.Tensor | None = None):
    """One SGD step on this rank's shard; returns the local sum of squared errors (fp64 device)."""
    rows = global_rows if global_rows is not None else x.shape[0]
    ls = loss_out if loss_out is not None else torch.empty(1, dtype=torch.float64, device=x.device)
    norm = float(rows * layer.plan.r_dim)
    if layer.mma == _lib.DT_MMA_BF16 and layer.activation == "identity":
        g = layer.forward_mse(x, target, norm, ls)   # MSE fused into the forward epilogue
    else:
        y = layer.forward(x)
        g = torch.empty_like(y)
        mse_grad_into(y, target, g, norm, ls)
    layer.backward(g)
    allreduce_grads(layer.grad_flat, group)
    layer.step(lr)
    return ls
