"""Config-5 geometry (reuse path, q = r_dim = 8192, rank 64, n 1024, batch 8192 per GPU): time the
bf16 tensor-core forward (factored) and, for comparison, the two-phase dense form."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1802_06944_b200 as D

q = r_dim = 8192; rank = 64; n = 1024; m = 65536; batch = int(os.environ.get("C5_BATCH", 8192))
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
g = torch.Generator(device="cuda").manual_seed(0)
xf = (torch.randn(m, rank, device="cuda", generator=g) / 8).cpu().numpy()
wf = (torch.randn(rank, n, device="cuda", generator=g) / 8).cpu().numpy()
fp = D.FactorPair(xf, wf, plan)
x = torch.randn(batch, q, device="cuda", generator=g).to(torch.bfloat16)
b = torch.zeros(r_dim, device="cuda")
for mode in ("1", "0"):
    os.environ["DEEPTHIN_REUSE_FACTORED"] = mode
    for _ in range(3):
        y = D.layer_forward(x, fp, b, mma="bf16")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        y = D.layer_forward(x, fp, b, mma="bf16")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 2.0 * batch * q * r_dim
    print(f"factored={mode}: {ms * 1e3:.1f} us/forward, dense-equiv {flops / ms / 1e9:.0f} TFLOP/s, "
          f"{batch / ms * 1e3 / 1e6:.2f} M samples/s")
    if mode == "1":
        y1 = y.float()
    else:
        print("factored vs dense max rel diff", float((y.float() - y1).abs().max() / y1.abs().max()))
