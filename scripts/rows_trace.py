"""One traced launch of the row-tile reuse kernel at config-3 hidden-layer geometry."""
import os, sys
os.environ["DEEPTHIN_ROWS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1802_06944_b200 as D
B = int(os.environ.get("B", 16384)); q = int(os.environ.get("Q", 2048)); r_dim = int(os.environ.get("R", 2048))
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=3, m=q * r_dim // 256, n=256)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (plan.m, 3)).astype(np.float32), rng.normal(0, .5, (3, 256)).astype(np.float32), plan)
x = torch.randn(B, q, device="cuda").to(torch.bfloat16)
b = torch.zeros(r_dim, device="cuda")
for i in range(3):
    y = D.layer_forward(x, fp, b, os.environ.get("ACT", "sigmoid"), mma="bf16", out_dtype=torch.bfloat16)
torch.cuda.synchronize()
