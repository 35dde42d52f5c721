"""Minimal driver for ncu: N forward launches of one BASELINE config (no timing logic)."""
import argparse
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib

GEO = {"c2": (440, 2048, 24, 320, 2816, 4096), "c1": (1024, 1024, 16, 256, 4096, 64)}
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--mma", default="bf16")
a = ap.parse_args()
q, r_dim, rank, n, m, batch = GEO[a.config]
batch = a.batch or batch
rng = np.random.default_rng(0)
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
fp = D.FactorPair(rng.standard_normal((m, rank)) / math.sqrt(rank),
                  rng.standard_normal((rank, n)) / math.sqrt(rank), plan)
x = torch.randn(batch, q, device="cuda").to(torch.bfloat16 if a.mma == "bf16" else torch.float32)
b = torch.zeros(r_dim, device="cuda")
for _ in range(a.iters):
    y = D.layer_forward(x, fp, b, mma=a.mma)
torch.cuda.synchronize()
print("ok", y.shape, float(y.abs().max()))
