"""Batch-sharded data parallelism.

Rows of x (and of the target) are split contiguously across ranks; factors
and bias are replicated. The forward needs no communication. Training needs
exactly one reduction per step: a SUM all-reduce of the flat fp32 gradient
buffer [d_xf | d_wf | d_bias], with every rank's local gradient already
normalised by the GLOBAL element count (grad.py:100-103), so the reduced
buffer equals the full-batch gradient. torch.distributed carries it (NCCL
over NVLink on GPUs, gloo in the CPU tests).

``GradReducer`` overlaps that reduction with the backward: the buffer is split
into buckets in the order the backward finalises them (d_xf first: its GEMM
runs before H and d_wf), and each bucket's all-reduce is issued on a
communication stream that waits only on the CUDA event recorded when that
bucket is final (dt_set_backward_event), so NCCL moves d_xf over NVLink while
the tensor cores still compute d_wf.
"""

from __future__ import annotations

import torch
import torch.distributed as tdist


def world() -> tuple[int, int]:
    if tdist.is_available() and tdist.is_initialized():
        return tdist.get_rank(), tdist.get_world_size()
    return 0, 1


def shard_rows(total: int, rank: int, world_size: int) -> tuple[int, int]:
    """Rows [k*B/W, (k+1)*B/W) for rank k (balanced when W does not divide B)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank/world {rank}/{world_size}")
    start = (total * rank) // world_size
    stop = (total * (rank + 1)) // world_size
    return start, stop


def allreduce_grads(flat: torch.Tensor, group=None) -> torch.Tensor:
    """In-place SUM all-reduce of the flat gradient buffer (no-op on one rank)."""
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size(group) > 1:
        tdist.all_reduce(flat, op=tdist.ReduceOp.SUM, group=group)
    return flat


class GradReducer:
    """Bucketed, overlapped SUM all-reduce of a flat gradient buffer.

    buckets: (start, stop) element ranges of ``flat`` in the order they become final. Each
    ``launch(i, event)`` issues bucket i's all-reduce asynchronously — on CUDA tensors from a
    side stream that first waits on ``event`` (recorded on the compute stream when the bucket is
    final; None: the current stream's position) — and ``wait()`` orders the current stream
    after every launched reduction. A no-op on one rank. The result is the same element-wise
    SUM as one all-reduce of the whole buffer (NCCL / gloo reduce each element identically).
    """

    def __init__(self, flat: torch.Tensor, buckets, group=None):
        self.flat = flat
        self.buckets = [(int(a), int(b)) for a, b in buckets]
        self.group = group
        self.active = (tdist.is_available() and tdist.is_initialized()
                       and tdist.get_world_size(group) > 1)
        self.stream = torch.cuda.Stream(device=flat.device) if (self.active and flat.is_cuda) else None
        self._work = []

    def launch(self, i: int, event=None):
        if not self.active:
            return
        a, b = self.buckets[i]
        view = self.flat[a:b]
        if self.stream is None:
            self._work.append(tdist.all_reduce(view, op=tdist.ReduceOp.SUM, group=self.group,
                                               async_op=True))
            return
        if event is None:
            event = torch.cuda.Event()
            event.record(torch.cuda.current_stream(self.flat.device))
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(event)
            self._work.append(tdist.all_reduce(view, op=tdist.ReduceOp.SUM, group=self.group,
                                               async_op=True))

    def wait(self):
        for w in self._work:
            w.wait()  # CUDA: the current stream waits for the collective (no host block)
        self._work = []
