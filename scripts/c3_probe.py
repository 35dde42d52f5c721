"""Config-3 probe: the 7-layer acoustic-model network (440 -> 6x2048 sigmoid -> 3000 softmax, rank 3,
n_f 256 where it divides the input width else 320), batch 16384, bf16. Times the whole network and
each layer alone (CUDA events, warm), and prints the per-layer HBM-bound floor."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import model_io as mi

B = int(os.environ.get("C3_BATCH", 16384))
dims = [440] + [2048] * 6 + [3000]
rng = np.random.default_rng(0)
entries, factors, biases = [], [], []
for i in range(len(dims) - 1):
    q, r_dim = dims[i], dims[i + 1]
    n = 256 if q % 256 == 0 else 320
    m = -(-(q * r_dim) // n)
    plan = D.LayerPlan(q=q, r_dim=r_dim, rank=3, m=m, n=n)
    entries.append((f"fc{i}", plan))
    factors.append(mi.StoredFactors(rng.normal(0, 3 ** -0.5, (m, 3)).astype(np.float32),
                                    rng.normal(0, 3 ** -0.5, (3, n)).astype(np.float32), plan))
    biases.append(rng.normal(0, 0.01, r_dim).astype(np.float32))
model = mi.CompressedModel(plans=D.NetworkPlan(layers=tuple(entries), target_ratio=0.01,
                                               achieved_total_ratio=0.0, floor_hits=()),
                           factors=factors, biases=biases)
acts = ["sigmoid"] * 6 + ["softmax"]
dm = model.to_device(acts, mma="bf16")
xs = [torch.randn(B, 440, device="cuda").to(torch.bfloat16) for _ in range(4)]


def timeit(fn, k=20):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(k):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


t = timeit(lambda i: dm.forward(xs[i % 4], out_dtype=torch.bfloat16))
tot_bytes = 0
for i in range(7):
    q, r = dims[i], dims[i + 1]
    tot_bytes += 2 * B * (q + r)
print(f"network: {t:.1f} us/forward, {B / t:.2f} M samples/s, act bytes {tot_bytes / 1e6:.1f} MB "
      f"-> {tot_bytes / t / 1e3:.0f} GB/s")
for i, fp in enumerate(dm.factors):
    q, r = dims[i], dims[i + 1]
    xi = [torch.randn(B, q, device="cuda").to(torch.bfloat16) for _ in range(4)]
    yi = [torch.empty(B, r, device="cuda", dtype=torch.bfloat16) for _ in range(4)]
    bias = dm.biases[i]
    from paper_1802_06944_b200.kernel import forward_into, _act_code
    code = D._lib.DT_MMA_BF16
    import ctypes as C
    lib = D._lib.lib()
    need = lib.dt_forward_workspace_bytes(C.byref(D._lib.plan_struct(fp.plan)), B, code)
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device="cuda")
    tl = timeit(lambda k: forward_into(xi[k % 4], fp, bias, _act_code(os.environ.get("LACT", "sigmoid")), 20.0, yi[k % 4],
                                       code, ws=ws))
    by = 2 * B * (q + r)
    print(f"layer {i} {q}->{r} reuse={fp.plan.reuse_path}: {tl:.1f} us, {by / tl / 1e3:.0f} GB/s "
          f"(floor {by / 6546e3:.1f} us)")
