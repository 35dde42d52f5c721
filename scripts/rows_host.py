"""Host vs GPU cost of one row-tile forward (prepared operands): host enqueue time per call,
GPU time per call when the calls are replayed from a CUDA graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib
from paper_1802_06944_b200.kernel import forward_into, _act_code
plan = D.LayerPlan(q=2048, r_dim=2048, rank=3, m=16384, n=256)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (16384, 3)).astype(np.float32), rng.normal(0, .5, (3, 256)).astype(np.float32), plan)
b = torch.zeros(2048, device="cuda")
for B in (128, 4096, 16384):
    x = torch.randn(B, 2048, device="cuda").to(torch.bfloat16)
    y = torch.empty(B, 2048, device="cuda", dtype=torch.bfloat16)
    f = lambda: forward_into(x, fp, b, _act_code("sigmoid"), 0.0, y, _lib.DT_MMA_BF16, cached=True)
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host = (t1 - t0) / 50 * 1e6
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            f()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"B={B:6d}: host {host:6.1f} us/call, graph-replayed GPU {e0.elapsed_time(e1) / 50 * 1e3:6.1f} us/call")
