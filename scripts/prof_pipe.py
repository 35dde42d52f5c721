"""Config-2 forwards back to back with inference pipelining on (for DEEPTHIN_TC_TRACE runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1802_06944_b200 as D
q, r_dim, rank, n, m, batch = 440, 2048, 24, 320, 2816, 4096
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.standard_normal((m, rank)) / 5, rng.standard_normal((rank, n)) / 5, plan)
xs = [torch.randn(batch, q, device="cuda").to(torch.bfloat16) for _ in range(4)]
b = torch.zeros(r_dim, device="cuda")
with D.forward_pipeline(os.environ.get("PIPE", "1") == "1"):
    for it in range(int(os.environ.get("ITERS", "4"))):
        y = D.layer_forward(xs[it % 4], fp, b, mma="bf16")
torch.cuda.synchronize()
print("ok")
