"""Per-kernel device-time table of one workload step, from CUPTI activity records (torch.profiler).

    python scripts/prof_kernels.py c5 [steps]      # config-5 training step (global batch 65536)
    python scripts/prof_kernels.py c3 [steps]      # config-3 network forward
    python scripts/prof_kernels.py c2 [steps]      # config-2 layer forward

Prints: kernel, launches, mean us, total us per step, share of the step's kernel time.
"""
import collections
import math
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_06944_b200 as D  # noqa: E402


def kname(full):
    """Short kernel name from a demangled signature: the k_* identifier with its template args."""
    import re
    m = re.search(r"(k_\w+)(<[^()]*>)?", full)
    return (m.group(1) + (m.group(2) or "")) if m else full.split("(")[0][-60:]


def c5_step(rows=65536):
    q = r_dim = 8192
    plan = D.LayerPlan(q=q, r_dim=r_dim, rank=64, m=65536, n=1024)
    g = torch.Generator(device="cuda").manual_seed(1234)
    xf = (torch.randn(65536, 64, device="cuda", generator=g) / 8).cpu().numpy()
    wf = (torch.randn(64, 1024, device="cuda", generator=g) / 8).cpu().numpy()
    bias = (torch.randn(r_dim, device="cuda", generator=g) * 0.01).cpu().numpy()
    layer = D.DeepThinLayer(plan, xf, wf, bias, mma="bf16")
    x = torch.randn(rows, q, device="cuda", generator=g).to(torch.bfloat16)
    t = torch.randn(rows, r_dim, device="cuda", generator=g)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    return lambda: D.train_step(layer, x, t, 1e-4, loss_out=loss)


def c3_step(rows=16384, graph=True):
    import numpy as np
    import bench
    from paper_1802_06944_b200 import model_io as mi
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
    x = torch.randn(rows, 440, device="cuda").to(torch.bfloat16)
    return lambda: dm.forward(x, out_dtype=torch.bfloat16, graph=graph)


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rows = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
    if key == "c5":
        step = c5_step(rows)
    elif key == "c3":
        step = c3_step(rows if len(sys.argv) > 3 else 16384)
    elif key == "c2":
        step = c2_step(rows if len(sys.argv) > 3 else 4096)
    else:
        raise SystemExit("configs: c5, c3, c2")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    agg = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            agg[kname(e.name)].append(e.time_range.end - e.time_range.start)
    tot = sum(sum(v) for v in agg.values()) / steps
    print(f"{key}: {ms * 1e3:.1f} us per step (events), kernels {tot:.1f} us per step")
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v) / steps:9.1f} us  {len(v) / steps:5.1f}x  {sum(v) / len(v):8.1f} us  "
              f"{sum(v) / steps / tot:6.1%}  {name}")



def c2_step(rows=4096):
    import numpy as np
    plan = D.LayerPlan(q=440, r_dim=2048, rank=24, m=2816, n=320)
    rng = np.random.default_rng(0)
    fp = D.FactorPair(rng.normal(0, 24 ** -0.5, (2816, 24)), rng.normal(0, 24 ** -0.5, (24, 320)), plan)
    b = torch.tensor(rng.normal(0, 0.01, 2048), dtype=torch.float32, device="cuda")
    xs = [torch.randn(rows, 440, device="cuda").to(torch.bfloat16) for _ in range(8)]
    from paper_1802_06944_b200.kernel import forward_pipeline
    it = [0]

    def step():
        with forward_pipeline(True, external_x=True):
            D.layer_forward(xs[it[0] % 8], fp, b, mma="bf16")
        it[0] += 1
    return step


if __name__ == "__main__":
    main()
