"""World-size-2 gloo test of the batch-sharded data-parallel host logic.

Each rank takes its contiguous row shard, computes its local factor gradients
normalised by the GLOBAL element count (grad.py:100-103; the CPU oracle stands in
for the device kernels here), and all-reduces the flat [d_xf | d_wf | d_bias]
buffer through paper_1802_06944_b200.dist. The reduced buffer must equal the
full-batch gradient, and the forward needs no collective.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import deepthin_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_06944_b200.dist import allreduce_grads, shard_rows, world as dworld

    assert dworld() == (rank, world)
    plan = O.Plan(q=96, r_dim=64, rank=4, m=97, n=64)   # general path geometry, tail 64
    batch = 37                                          # does not divide by the world size
    d = O.baseline_inputs(plan, batch, seed=3)
    lo, hi = shard_rows(batch, rank, world)
    x, t = d["x"][lo:hi], d["target"][lo:hi]
    # forward on the shard: no communication
    y = O.layer_forward(x, d["xf"], d["wf"], plan, d["bias"], "identity")
    # local MSE gradient normalised by the global element count
    g = 2.0 * (y - t) / (batch * plan.r_dim)
    gr = O.layer_backward(x, d["xf"], d["wf"], plan, d["bias"], "identity", g)
    flat = torch.tensor(np.concatenate([gr.d_xf.ravel(), gr.d_wf.ravel(), gr.d_bias]))
    allreduce_grads(flat)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), flat.numpy())
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y)
    tdist.barrier()
    tdist.destroy_process_group()


def test_shard_rows_partition():
    from paper_1802_06944_b200.dist import shard_rows
    for total in (0, 1, 7, 37, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(10, 2, 2)


def test_allreduce_single_process_is_noop():
    from paper_1802_06944_b200.dist import allreduce_grads
    t = torch.arange(5.0)
    assert torch.equal(allreduce_grads(t.clone()), t)


def test_two_rank_gradient_allreduce_equals_full_batch(tmp_path):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    plan = O.Plan(q=96, r_dim=64, rank=4, m=97, n=64)
    batch = 37
    d = O.baseline_inputs(plan, batch, seed=3)
    y = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    _, g = O.loss_and_grad("mse", y, d["target"])
    gr = O.layer_backward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity", g)
    full = np.concatenate([gr.d_xf.ravel(), gr.d_wf.ravel(), gr.d_bias])
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.allclose(got, full, rtol=1e-10, atol=1e-14)
    # the sharded forward concatenates to the full-batch forward exactly
    ys = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    assert np.array_equal(ys, y)


def test_bench_self_launches_ranks_dry_run():
    """bench.py --gpus 2 without a torchrun environment launches two ranks itself
    (torch.distributed.run on 127.0.0.1); rank 0 reports n_gpus 2 and both ranks took part in
    a collective (rank_sum = 1 + 2)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--dry-run"], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["rank_sum"] == 3.0
    assert "world_size=2" in r.stderr


def _reducer_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_06944_b200.dist import GradReducer, allreduce_grads
    rng = np.random.default_rng(10 + rank)
    flat = torch.tensor(rng.standard_normal(1000))
    ref = flat.clone()
    allreduce_grads(ref)
    red = GradReducer(flat, [(0, 384), (384, 1000)])
    assert red.active
    red.launch(0)        # the d_xf bucket first (final before d_wf / d_bias)
    red.launch(1)
    red.wait()
    np.save(os.path.join(out_dir, f"red{rank}.npy"), flat.numpy())
    np.save(os.path.join(out_dir, f"ref{rank}.npy"), ref.numpy())
    tdist.barrier()
    tdist.destroy_process_group()


def test_bucketed_overlapped_reducer_equals_one_allreduce(tmp_path):
    """dist.GradReducer (bucketed, asynchronous; on GPUs each bucket waits only on the event the
    backward records when it is final) reduces to the same buffer as one all-reduce."""
    world = 2
    mp.spawn(_reducer_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"red{r}.npy"), np.load(tmp_path / f"ref{r}.npy"))


def test_reducer_single_process_is_noop():
    from paper_1802_06944_b200.dist import GradReducer
    t = torch.arange(6.0)
    red = GradReducer(t, [(0, 2), (2, 6)])
    assert not red.active
    red.launch(0)
    red.launch(1)
    red.wait()
    assert torch.equal(t, torch.arange(6.0))
