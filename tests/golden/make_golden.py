"""Generate golden vectors by importing the reference ``deepthin`` package.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz``. Every array is the reference's own output
on seeded inputs; ``tests/test_oracle_golden.py`` pins the oracle against it
and the GPU tests pin the CUDA path against the (pinned) oracle.
"""

from __future__ import annotations

import math
import os
import sys
import warnings

import numpy as np

REF = os.environ.get("DEEPTHIN_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from deepthin.core import make_rng, sample_normal, spawn_rngs  # noqa: E402
from deepthin.factor import (  # noqa: E402
    FactorPair, decompress, init_factors, phase, phase_count, relayout_index)
from deepthin.grad import layer_backward, loss_and_grad  # noqa: E402
from deepthin.kernel import ReuseTable, fused_matmul, layer_forward, predict_reuse  # noqa: E402
from deepthin.planner import LayerPlan  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def plan_of(q, r_dim, rank, n, m=None):
    m = m if m is not None else -(-(q * r_dim) // n)
    return LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)


def inputs(plan, batch, seed, bias_sd=0.01):
    """Same convention as oracle.baseline_inputs: children [xf, wf, bias, x, target]."""
    rx, rw, rb, ri, rt = spawn_rngs(seed, 5)
    sd = 1.0 / math.sqrt(plan.rank)
    return dict(
        xf=sample_normal(rx, 0.0, sd, (plan.m, plan.rank)),
        wf=sample_normal(rw, 0.0, sd, (plan.rank, plan.n)),
        bias=sample_normal(rb, 0.0, bias_sd, (plan.r_dim,)),
        x=sample_normal(ri, 0.0, 1.0, (batch, plan.q)),
        target=sample_normal(rt, 0.0, 1.0, (batch, plan.r_dim)))


def main():
    g: dict[str, np.ndarray] = {}
    warnings.simplefilter("ignore", RuntimeWarning)   # rank>1 fallback warning

    # --- seeding convention (core.py:39-60) -------------------------------
    g["rng_make7"] = make_rng(7).standard_normal(16)
    g["rng_spawn3"] = np.stack([r.standard_normal(8) for r in spawn_rngs(3, 4)])
    g["rng_sample"] = sample_normal(make_rng(11), 0.5, 0.25, (4, 5))

    # --- index laws (factor.py:74-110, kernel.py:184-205) -----------------
    rng = np.random.default_rng(100)
    idx_rows = []
    for _ in range(300):
        q = int(rng.integers(1, 400))
        r_dim = int(rng.integers(1, 300))
        n = int(rng.integers(1, min(q * r_dim, 5000) + 1))
        p = plan_of(q, r_dim, 1, n)
        cols = rng.integers(0, r_dim, 4)
        d, t = predict_reuse(p, 1)
        idx_rows.append([q, r_dim, n, p.m, phase_count(p), d, t,
                         *[phase(int(c), p) for c in cols], *cols.tolist()])
    g["index_laws"] = np.array(idx_rows, dtype=np.int64)
    p = plan_of(7, 5, 1, 5)
    g["relayout_7x5"] = np.array([relayout_index(k, p) for k in range(35)], dtype=np.int64)

    # --- decompress on random small plans, ranks 1-3 (factor.py:87-93) ----
    rng = np.random.default_rng(101)
    for i in range(24):
        q = int(rng.integers(1, 48))
        r_dim = int(rng.integers(1, 48))
        rank = int(rng.integers(1, 4))
        n = int(rng.integers(1, q * r_dim + 1))
        p = plan_of(q, r_dim, rank, n)
        fp = init_factors(p, 1.0, make_rng(1000 + i))
        g[f"dec{i}_plan"] = np.array([q, r_dim, rank, p.m, n])
        g[f"dec{i}_xf"] = np.asarray(fp.xf)
        g[f"dec{i}_wf"] = np.asarray(fp.wf)
        g[f"dec{i}_w"] = decompress(fp)

    # --- rank-1 fused_matmul with reuse accounting (kernel.py:222-293) ----
    rng = np.random.default_rng(102)
    for i in range(16):
        q = int(rng.integers(1, 80))
        r_dim = int(rng.integers(1, 80))
        n = int(rng.integers(1, q * r_dim + 1))
        p = plan_of(q, r_dim, 1, n)
        fp = init_factors(p, 1.0, make_rng(2000 + i))
        x = rng.standard_normal((int(rng.integers(1, 5)), q))
        table = ReuseTable()
        y, ops = fused_matmul(x, fp, reuse=table)
        g[f"fm{i}_plan"] = np.array([q, r_dim, 1, p.m, n])
        g[f"fm{i}_xf"] = np.asarray(fp.xf)
        g[f"fm{i}_wf"] = np.asarray(fp.wf)
        g[f"fm{i}_x"] = x
        g[f"fm{i}_y"] = y
        g[f"fm{i}_counts"] = np.array([table.hits, table.misses, ops.multiplies, ops.adds])
    # f32 route (output dtype f32, kernel.py:252,293)
    p = plan_of(64, 48, 1, 16)
    fp = init_factors(p, 1.0, make_rng(2100))
    fp32 = fp.with_values(np.asarray(fp.xf, np.float32), np.asarray(fp.wf, np.float32))
    x32 = np.random.default_rng(103).standard_normal((3, 64)).astype(np.float32)
    y32, _ = fused_matmul(x32, fp32)
    assert y32.dtype == np.float32
    g["fm32_xf"], g["fm32_wf"], g["fm32_x"], g["fm32_y"] = (
        np.asarray(fp32.xf), np.asarray(fp32.wf), x32, y32)

    # --- layer_forward: small plans x activations, + BASELINE geometries --
    rng = np.random.default_rng(104)
    acts = ("identity", "relu", "sigmoid", "tanh")
    for i in range(16):
        q = int(rng.integers(1, 64))
        r_dim = int(rng.integers(1, 64))
        rank = int(rng.integers(1, 4))
        n = int(rng.integers(1, q * r_dim + 1))
        p = plan_of(q, r_dim, rank, n)
        d = inputs(p, int(rng.integers(1, 6)), 3000 + i, bias_sd=0.3)
        fp = FactorPair(d["xf"], d["wf"], p)
        act = acts[i % 4]
        g[f"lf{i}_plan"] = np.array([q, r_dim, rank, p.m, n])
        g[f"lf{i}_act"] = np.array([i % 4])
        for k in ("xf", "wf", "bias", "x"):
            g[f"lf{i}_{k}"] = d[k]
        g[f"lf{i}_y"] = layer_forward(d["x"], fp, d["bias"], act)

    # BASELINE geometries (reference notation q, r_dim, rank, n, m), batch reduced.
    # inputs are rounded to the GPU I/O dtype first so the same arrays feed both sides
    geos = {
        "c1": (1024, 1024, 16, 256, 4096, 4, "f32"),    # config 1, reuse path
        "c2": (440, 2048, 24, 320, 2816, 4, "bf16"),     # config 2, general path
        "c4fc1": (494, 2048, 3, 320, 3162, 2, "bf16"),   # config 4 fc1: period 160, tail 128
        "c3l1": (2048, 2048, 3, 256, 16384, 2, "bf16"),  # config 3 hidden layer, reuse
    }
    for key, (q, r_dim, rank, n, m, batch, io) in geos.items():
        p = plan_of(q, r_dim, rank, n, m)
        d = inputs(p, batch, 0)
        for k in ("xf", "wf", "bias", "x"):
            a = d[k]
            if io == "f32":
                a = a.astype(np.float32).astype(np.float64)
            else:
                a = _bf16(a)
            d[k] = a
        fp = FactorPair(d["xf"], d["wf"], p)
        g[f"{key}_plan"] = np.array([q, r_dim, rank, m, n])
        g[f"{key}_x"] = d["x"]
        g[f"{key}_y"] = layer_forward(d["x"], fp, d["bias"], "identity")
        # sampled entries of W (too large to store whole)
        w = decompress(fp)
        srng = np.random.default_rng(5)
        ii = srng.integers(0, q, 2048)
        jj = srng.integers(0, r_dim, 2048)
        g[f"{key}_wsample"] = np.stack([ii, jj]).astype(np.int64)
        g[f"{key}_wvals"] = w[ii, jj]

    # --- layer_backward (grad.py:63-95) + loss_and_grad (grad.py:98-116) --
    rng = np.random.default_rng(105)
    for i in range(12):
        q = int(rng.integers(1, 40))
        r_dim = int(rng.integers(1, 40))
        rank = int(rng.integers(1, 4))
        n = int(rng.integers(1, q * r_dim + 1))
        p = plan_of(q, r_dim, rank, n)
        d = inputs(p, int(rng.integers(1, 6)), 4000 + i, bias_sd=0.3)
        fp = FactorPair(d["xf"], d["wf"], p)
        act = acts[i % 4]
        up = np.random.default_rng(4100 + i).standard_normal((d["x"].shape[0], r_dim))
        gr = layer_backward(d["x"], fp, d["bias"], act, up)
        g[f"lb{i}_plan"] = np.array([q, r_dim, rank, p.m, n])
        g[f"lb{i}_act"] = np.array([i % 4])
        for k in ("xf", "wf", "bias", "x"):
            g[f"lb{i}_{k}"] = d[k]
        g[f"lb{i}_up"] = up
        g[f"lb{i}_dxf"], g[f"lb{i}_dwf"] = gr.d_xf, gr.d_wf
        g[f"lb{i}_dx"], g[f"lb{i}_db"] = gr.d_input, gr.d_bias

    # training-step geometries: reuse (config-5 shape scaled down) and general (config 2)
    for key, (q, r_dim, rank, n, m, batch) in {
            "t5s": (512, 512, 8, 64, 4096, 8),
            "t2": (440, 2048, 24, 320, 2816, 3)}.items():
        p = plan_of(q, r_dim, rank, n, m)
        d = inputs(p, batch, 1)
        for k in ("xf", "wf", "bias", "x", "target"):
            d[k] = _bf16(d[k])
        fp = FactorPair(d["xf"], d["wf"], p)
        y = layer_forward(d["x"], fp, d["bias"], "identity")
        loss, dy = loss_and_grad("mse", y, d["target"])
        gr = layer_backward(d["x"], fp, d["bias"], "identity", dy)
        g[f"{key}_plan"] = np.array([q, r_dim, rank, m, n])
        g[f"{key}_loss"] = np.array([loss])
        g[f"{key}_dxf"], g[f"{key}_dwf"] = gr.d_xf, gr.d_wf
        g[f"{key}_dx"], g[f"{key}_db"] = gr.d_input, gr.d_bias

    yy = np.random.default_rng(106).standard_normal((5, 7))
    tt = np.random.default_rng(107).standard_normal((5, 7))
    l1, g1 = loss_and_grad("mse", yy, tt)
    l2, g2 = loss_and_grad("softmax_cross_entropy", yy, np.arange(5) % 7)
    g["loss_y"], g["loss_t"] = yy, tt
    g["loss_mse"], g["loss_mse_grad"] = np.array([l1]), g1
    g["loss_ce"], g["loss_ce_grad"] = np.array([l2]), g2

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


def _bf16(a):
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    u = a32.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


if __name__ == "__main__":
    main()
