"""Training step of a compressed layer on the GPU (reference train.py:86-117, 201-230, 305-357).

``DeepThinLayer`` holds fp32 master factors and bias and one flat fp32
gradient buffer [d_xf | d_wf | d_bias] so a data-parallel step needs a
single all-reduce. ``train_step`` is BASELINE config 5's step: forward,
MSE gradient normalised by the global element count, backward through the
inverse re-layout, all-reduce, SGD (train.py:107-111).
"""

from __future__ import annotations

from ctypes import c_void_p as ctypes_void_p

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import as_device_vector, device, make_rng, stream_handle
from .errors import ArgumentError
from .dist import allreduce_grads
from .factor import FactorPair
from .grad import backward_into, loss_and_grad, mse_grad_into
from .kernel import _act_code, forward_into
from .planner import LayerPlan


class DeepThinLayer:
    def __init__(self, plan: LayerPlan, xf, wf, bias=None, activation: str = "identity",
                 mma: str = "bf16", act_arg: float = 20.0):
        self.plan = plan
        # fp32 masters in ONE flat buffer [xf | wf | bias] (256-byte aligned segments) laid out
        # like grad_flat, so the SGD step is a single launch over both flat buffers
        src = FactorPair(xf, wf, plan)
        nx, nw = plan.m * plan.rank, plan.rank * plan.n
        ox, ow, ob = 0, -(-nx // 64) * 64, 0
        ob = ow + -(-nw // 64) * 64
        total = ob + -(-plan.r_dim // 64) * 64
        self.param_flat = torch.zeros(total, dtype=torch.float32, device=device())
        self.grad_flat = torch.zeros(total, dtype=torch.float32, device=device())
        self.param_flat[ox:ox + nx].copy_(src.xf.reshape(-1))
        self.param_flat[ow:ow + nw].copy_(src.wf.reshape(-1))
        b = as_device_vector(np.zeros(plan.r_dim) if bias is None else bias, plan.r_dim)
        self.param_flat[ob:ob + plan.r_dim].copy_(b)
        self.fp = FactorPair.adopt(self.param_flat[ox:ox + nx].view(plan.m, plan.rank),
                                   self.param_flat[ow:ow + nw].view(plan.rank, plan.n), plan)
        # serialization keeps the source's dtype (and, until the first step, its exact values)
        self.fp._cache["source_dtype"] = src.source_dtype
        if "source64" in src._cache:
            self.fp._cache["source64"] = src._cache["source64"]
        self.bias = self.param_flat[ob:ob + plan.r_dim]
        self.d_xf = self.grad_flat[ox:ox + nx].view(plan.m, plan.rank)
        self.d_wf = self.grad_flat[ow:ow + nw].view(plan.rank, plan.n)
        self.d_bias = self.grad_flat[ob:ob + plan.r_dim]
        self.activation = activation
        self.act = _act_code(activation)
        self.act_arg = act_arg
        self.mma = _lib.DT_MMA_BF16 if mma == "bf16" else _lib.DT_MMA_FFMA
        self._x = None

    def forward(self, x: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
        self._x = x
        self._p = None
        y = torch.empty((x.shape[0], self.plan.r_dim), dtype=out_dtype, device=x.device)
        forward_into(x, self.fp, self.bias, self.act, self.act_arg, y, self.mma)
        return y

    def forward_mse(self, x: torch.Tensor, target: torch.Tensor, norm_count: float,
                    loss_out: torch.Tensor, keep_for_backward: bool = False) -> torch.Tensor:
        """Forward + MSE gradient in one pass (dt_forward_mse, identity activation, bf16 path):
        returns grad = 2 (y - target) / norm_count; loss_out[0] = sum (y - target)^2. y itself
        is never written (grad.py:98-103 fused into the contraction's epilogue).
        keep_for_backward (reuse geometries): the loss pass also produces d_bias (grad.py:85)
        and the forward's P is kept, so the next backward() skips both (dt_forward_mse_ex)."""
        self._x = x
        lib = _lib.lib()
        ps = _lib.plan_struct(self.plan)
        batch = x.shape[0]
        from .core import workspace
        ws = workspace(lib.dt_forward_mse_workspace_bytes(C.byref(ps), batch))
        g = torch.empty((batch, self.plan.r_dim), dtype=torch.float32, device=x.device)
        tgt = target.contiguous().float()
        self._p = None
        pbytes = lib.dt_forward_p_bytes(C.byref(ps), batch) if keep_for_backward else 0
        if pbytes:
            self._p = torch.empty(pbytes // 4, dtype=torch.float32, device=x.device)
        _lib.check(lib.dt_forward_mse_ex(
            C.byref(ps), batch, x.data_ptr(), _lib.DT_BF16 if x.dtype == torch.bfloat16 else _lib.DT_F32,
            self.fp.xf.data_ptr(), self.fp.wf.data_ptr(), self.bias.data_ptr(), tgt.data_ptr(),
            float(norm_count), g.data_ptr(), loss_out.data_ptr(),
            self.d_bias.data_ptr() if self._p is not None else None,
            self._p.data_ptr() if self._p is not None else None, ws.data_ptr(), ws.numel(),
            stream_handle()))
        return g

    def backward(self, upstream: torch.Tensor, need_input_grad: bool = False):
        d_in = (torch.empty((self._x.shape[0], self.plan.q), dtype=torch.float32, device=self._x.device)
                if need_input_grad else None)
        kept = getattr(self, "_p", None)  # forward_mse(keep_for_backward=True): P and d_bias done
        backward_into(self._x, self.fp, self.bias, self.act, self.act_arg, upstream, self.d_xf,
                      self.d_wf, None if kept is not None else self.d_bias, d_in, self.mma,
                      p_in=kept)
        self._p = None
        return d_in

    def reducer(self, group=None):
        """dist.GradReducer over grad_flat with buckets [d_xf] then [d_wf | d_bias] (the order
        the tensor-core backward finalises them), cached per process group."""
        from .dist import GradReducer
        key = id(group)
        cache = self.__dict__.setdefault("_reducers", {})
        if key not in cache:
            ow = -(-(self.plan.m * self.plan.rank) // 64) * 64
            cache[key] = GradReducer(self.grad_flat, [(0, ow), (ow, self.grad_flat.numel())], group)
        return cache[key]

    def grad_buffers(self):
        """train.py:226-227: the gradient buffers the global-norm clip sees."""
        return [self.d_xf, self.d_wf, self.d_bias]

    def step(self, lr: float) -> None:
        """train.py:107-111 + :221: SGD on the fp32 masters, then refresh bf16 operand copies."""
        lib = _lib.lib()
        _lib.check(lib.dt_sgd_step(self.param_flat.numel(), self.param_flat.data_ptr(),
                                   self.grad_flat.data_ptr(), float(lr), stream_handle()))
        self.fp.refresh_derived()


def train_step(layer: DeepThinLayer, x: torch.Tensor, target: torch.Tensor, lr: float,
               global_rows: int | None = None, group=None, loss_out: torch.Tensor | None = None):
    """One SGD step on this rank's shard; returns the local sum of squared errors (fp64 device)."""
    rows = global_rows if global_rows is not None else x.shape[0]
    ls = loss_out if loss_out is not None else torch.empty(1, dtype=torch.float64, device=x.device)
    norm = float(rows * layer.plan.r_dim)
    if layer.mma == _lib.DT_MMA_BF16 and layer.activation == "identity":
        # MSE fused into the forward; its loss pass also yields d_bias, and P is kept for the
        # backward (reuse geometries: config 5)
        g = layer.forward_mse(x, target, norm, ls, keep_for_backward=layer.plan.reuse_path)
    else:
        y = layer.forward(x)
        g = torch.empty_like(y)
        mse_grad_into(y, target, g, norm, ls)
    red = layer.reducer(group)
    if red.active:
        # d_xf is final after the backward's first GEMM: its all-reduce overlaps the rest
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())  # cudaEvent_t created; re-recorded in the backward
        _lib.check(_lib.lib().dt_set_backward_event(ctypes_void_p(ev.cuda_event)))
        layer.backward(g)
        red.launch(0, ev)
        red.launch(1)
        red.wait()
    else:
        layer.backward(g)
    layer.step(lr)
    return ls


# ---- multi-layer SGD trainer on the device (reference train.py:305-357) ----

LOSSES = ("mse", "softmax_cross_entropy")


@dataclass(frozen=True)
class TrainConfig:
    """grad.py:31-51: learning rate, epochs, batch size, shuffle seed, loss, global-norm clip."""

    learning_rate: float
    epochs: int
    batch_size: int
    seed: int
    loss: str = "mse"
    clip_norm: float | None = None

    def __post_init__(self):
        if not self.learning_rate > 0:
            raise ArgumentError(f"learning_rate must be > 0, got {self.learning_rate}")
        if self.epochs < 1 or self.batch_size < 1:
            raise ArgumentError("epochs and batch_size must be >= 1")
        if self.loss not in LOSSES:
            raise ArgumentError(f"loss must be one of {LOSSES}, got {self.loss!r}")
        if self.clip_norm is not None and not self.clip_norm > 0:
            raise ArgumentError(f"clip_norm must be > 0, got {self.clip_norm}")


def clip_gradients(layers, clip_norm) -> None:
    """train.py:318-327 on the device: global L2 norm over every layer's gradient buffers
    (fp64, fixed order), all buffers scaled by clip/norm when norm > clip and finite. No host
    synchronisation: the scale is computed and applied on the device."""
    if clip_norm is None:
        return
    bufs = [b for layer in layers for b in layer.grad_buffers()]
    total = torch.stack([(b.double() * b.double()).sum() for b in bufs]).sum()
    norm = torch.sqrt(total)
    scale = torch.where(torch.isfinite(norm) & (norm > clip_norm), clip_norm / norm,
                        torch.ones_like(norm)).float()
    for layer in layers:
        layer.grad_flat.mul_(scale)


def _forward_all(layers, x):
    for layer in layers:
        x = layer.forward(x)
    return x


def evaluate(layers, x, target, loss: str) -> float:
    """train.py:296-301: the validation loss of the chained layers."""
    return loss_and_grad(loss, _forward_all(layers, x), target)[0]


def sgd_train(layers, train_data, val_data, cfg: TrainConfig):
    """train.py:305-357 on the device: per epoch a seeded shuffle (make_rng(seed ^ 0x5DEE9),
    the reference's stream), minibatch forward through every DeepThinLayer, loss gradient,
    backward through the inverse re-layouts (input gradients chained), global-norm clip, SGD on
    the fp32 masters. Returns [(epoch, train_loss, val_loss)] with diverged losses as inf."""
    x_train, y_train = (torch.as_tensor(np.asarray(a, dtype=np.float32)).to(device())
                        if not isinstance(a, torch.Tensor) else a for a in train_data)
    x_val, y_val = (torch.as_tensor(np.asarray(a, dtype=np.float32)).to(device())
                    if not isinstance(a, torch.Tensor) else a for a in val_data)
    shuffle_rng = make_rng(cfg.seed ^ 0x5DEE9)
    history = []
    for epoch in range(1, cfg.epochs + 1):
        order = torch.as_tensor(shuffle_rng.permutation(len(x_train)), device=device())
        epoch_loss, batches = 0.0, 0
        for start in range(0, len(order), cfg.batch_size):
            idx = order[start:start + cfg.batch_size]
            out = _forward_all(layers, x_train[idx])
            loss, g = loss_and_grad(cfg.loss, out, y_train[idx])
            for i, layer in enumerate(reversed(layers)):
                g = layer.backward(g, need_input_grad=i + 1 < len(layers))
            clip_gradients(layers, cfg.clip_norm)
            for layer in layers:
                layer.step(cfg.learning_rate)
            epoch_loss += loss
            batches += 1
        train_loss = epoch_loss / batches
        val_loss = evaluate(layers, x_val, y_val, cfg.loss)
        history.append((epoch, train_loss if np.isfinite(train_loss) else float("inf"),
                        val_loss if np.isfinite(val_loss) else float("inf")))
    return history
