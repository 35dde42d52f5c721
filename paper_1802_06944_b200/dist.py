"""Batch-sharded data parallelism.

Rows of x (and of the target) are split contiguously across ranks; factors
and bias are replicated. The forward needs no communication. Training needs
exactly one collective per step: a SUM all-reduce of the flat fp32 gradient
buffer [d_xf | d_wf | d_bias], with every rank's local gradient already
normalised by the GLOBAL element count (grad.py:100-103), so the reduced
buffer equals the full-batch gradient. torch.distributed carries it (NCCL
over NVLink on GPUs, gloo in the CPU tests).
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
