"""ncu driver: a few config-1 forwards (reuse path, batch 64) on the FFMA path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1802_06944_b200 as D
plan = D.LayerPlan(q=1024, r_dim=1024, rank=16, m=4096, n=256)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.standard_normal((4096, 16)) / 4, rng.standard_normal((16, 256)) / 4, plan)
x = torch.randn(64, 1024, device="cuda")
b = torch.zeros(1024, device="cuda")
for _ in range(3):
    y = D.layer_forward(x, fp, b, mma="ffma")
torch.cuda.synchronize()
print("ok", float(y.abs().max()))
