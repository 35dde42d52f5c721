"""Traced launch of the config-3 layer-0 GEMM (timing build + DEEPTHIN_TC_TRACE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1802_06944_b200 as D
plan = D.LayerPlan(q=440, r_dim=2048, rank=3, m=2816, n=320)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.normal(0, .5, (2816, 3)), rng.normal(0, .5, (3, 320)), plan)
x = torch.randn(16384, 440, device="cuda").to(torch.bfloat16)
b = torch.zeros(2048, device="cuda")
for _ in range(2):
    y = D.layer_forward(x, fp, b, "sigmoid", mma="bf16", out_dtype=torch.bfloat16)
torch.cuda.synchronize()
