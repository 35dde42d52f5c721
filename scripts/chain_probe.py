"""Config-3 forward timed with the per-tile layer chaining of the clustered row-tile kernel
(DeviceModel.chain) off / on, eager and CUDA-graph: one GPU, CUDA events over 50 forwards."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_06944_b200 as D  # noqa: E402
from paper_1802_06944_b200 import model_io as mi  # noqa: E402


def main():
    layers, params, rx = bench.c3_params()
    entries, factors, biases = [], [], []
    for i, ((q, r_dim, rk, n, m), (xf, wf, b)) in enumerate(zip(layers, params)):
        plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rk, m=m, n=n)
        entries.append((f"fc{i}", plan))
        factors.append(mi.StoredFactors(xf, wf, plan))
        biases.append(b)
    model = mi.CompressedModel(plans=D.NetworkPlan(layers=tuple(entries), target_ratio=0.01,
                                                   achieved_total_ratio=0.0, floor_hits=()),
                               factors=factors, biases=biases)
    dm = model.to_device(bench.C3_ACTS, mma="bf16")
    B = int(os.environ.get("B", 16384))
    x = torch.randn(B, 440, device="cuda").to(torch.bfloat16)
    for chain in (False, True):
        for graph in (False, True):
            dm.chain = chain
            try:
                for _ in range(5):
                    y = dm.forward(x, out_dtype=torch.bfloat16, graph=graph)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(50):
                    y = dm.forward(x, out_dtype=torch.bfloat16, graph=graph)
                e1.record()
                torch.cuda.synchronize()
                print(f"chain={chain} graph={graph}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per forward")
            except Exception as ex:  # noqa: BLE001
                print(f"chain={chain} graph={graph}: {type(ex).__name__}: {ex}")
    dm.chain = False


if __name__ == "__main__":
    main()
