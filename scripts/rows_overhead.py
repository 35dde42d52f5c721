"""Fixed per-launch cost of the row-tile kernel: prepared operands (no prep launch), batch sweep,
back-to-back launches timed with one event pair (config-3 hidden-layer geometry)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib
from paper_1802_06944_b200.kernel import forward_into, _act_code
plan = D.LayerPlan(q=2048, r_dim=2048, rank=3, m=16384, n=256)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (16384, 3)).astype(np.float32), rng.normal(0, .5, (3, 256)).astype(np.float32), plan)
b = torch.zeros(2048, device="cuda")
for B in (128, 1024, 4096, 16384, 65536):
    xs = [torch.randn(B, 2048, device="cuda").to(torch.bfloat16) for _ in range(2)]
    ys = [torch.empty(B, 2048, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    for cached in (True, False):
        f = lambda k: forward_into(xs[k % 2], fp, b, _act_code("sigmoid"), 0.0, ys[k % 2], _lib.DT_MMA_BF16, cached=cached)
        for k in range(3):
            f(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        e0.record()
        for k in range(K):
            f(k)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / K * 1e3
        print(f"B={B:6d} cached={cached}: {us:7.1f} us/launch, {4 * B * 2048 / us / 1e3:7.0f} GB/s")
