"""Config-3 network: eager vs CUDA-graph DeviceModel.forward at the per-GPU batch of 1 and 8 GPUs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1802_06944_b200 import model_io as mi
import paper_1802_06944_b200 as D
layers, params, _ = bench.c3_params()
entries, factors, biases = [], [], []
for i, ((q, r, rk, n, m), (xf, wf, b)) in enumerate(zip(layers, params)):
    plan = D.LayerPlan(q=q, r_dim=r, rank=rk, m=m, n=n)
    entries.append((f"fc{i}", plan)); factors.append(mi.StoredFactors(xf, wf, plan)); biases.append(b)
model = mi.CompressedModel(plans=D.NetworkPlan(layers=tuple(entries), target_ratio=0.01, achieved_total_ratio=0.0, floor_hits=()), factors=factors, biases=biases)
dm = model.to_device(bench.C3_ACTS, mma="bf16")
for B in (16384, 2048):
    x = torch.randn(B, 440, device="cuda").to(torch.bfloat16)
    for graph in (False, True):
        for _ in range(3):
            dm.forward(x, out_dtype=torch.bfloat16, graph=graph)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dm.forward(x, out_dtype=torch.bfloat16, graph=graph)
        e1.record(); torch.cuda.synchronize()
        print(f"B={B:6d} graph={graph}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/forward")
