"""Config-3 layer 0 (440 -> 2048, general path, batch 16384) on the two-phase pair GEMM:
per-call time by output dtype and activation (isolates the epilogue's cost)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib
from paper_1802_06944_b200.kernel import forward_into, _act_code
B = 16384
plan = D.LayerPlan(q=440, r_dim=2048, rank=3, m=2816, n=320)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (2816, 3)).astype(np.float32), rng.normal(0, .5, (3, 320)).astype(np.float32), plan)
b = torch.zeros(2048, device="cuda")
xs = [torch.randn(B, 440, device="cuda").to(torch.bfloat16) for _ in range(2)]
import ctypes as C
ws = torch.empty(_lib.lib().dt_forward_workspace_bytes(C.byref(_lib.plan_struct(plan)), B, _lib.DT_MMA_BF16), dtype=torch.uint8, device="cuda")
for dt in (torch.float32, torch.bfloat16):
    ys = [torch.empty(B, 2048, device="cuda", dtype=dt) for _ in range(2)]
    for act in ("identity", "sigmoid"):
        f = lambda k: forward_into(xs[k % 2], fp, b, _act_code(act), 0.0, ys[k % 2], _lib.DT_MMA_BF16, ws=ws)
        for k in range(3): f(k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(20): f(k)
        e1.record(); torch.cuda.synchronize()
        print(f"{str(dt):15s} {act:9s}: {e0.elapsed_time(e1) / 20 * 1e3:6.1f} us")
