"""Config-5 training step (reuse path, bf16 tensor cores): forward + MSE gradient + backward +
SGD on one GPU's 8192-row shard. Prints us/step and the breakdown."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1802_06944_b200 as D

q = r_dim = 8192; rank = 64; n = 1024; m = 65536; batch = int(os.environ.get("C5_BATCH", 8192))
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
g = torch.Generator(device="cuda").manual_seed(0)
xf = (torch.randn(m, rank, device="cuda", generator=g) / 8).cpu().numpy()
wf = (torch.randn(rank, n, device="cuda", generator=g) / 8).cpu().numpy()
layer = D.DeepThinLayer(plan, xf, wf, mma=os.environ.get("MMA", "bf16"))
x = torch.randn(batch, q, device="cuda", generator=g).to(torch.bfloat16)
t = torch.randn(batch, r_dim, device="cuda", generator=g)
for _ in range(3):
    D.train_step(layer, x, t, 1e-3)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
K = int(os.environ.get("K", 10))
tot = [0.0] * 4
for _ in range(K):
    e[0].record()
    y = layer.forward(x)
    e[1].record()
    gy = torch.empty_like(y)
    ls = torch.empty(1, dtype=torch.float64, device="cuda")
    from paper_1802_06944_b200.grad import mse_grad_into
    mse_grad_into(y, t, gy, float(batch * r_dim), ls)
    e[2].record()
    layer.backward(gy)
    e[3].record()
    layer.step(1e-3)
    e[4].record()
    torch.cuda.synchronize()
    for i in range(4):
        tot[i] += e[i].elapsed_time(e[i + 1]) / K
print(f"step {sum(tot) * 1e3:.1f} us: forward {tot[0] * 1e3:.1f}, mse {tot[1] * 1e3:.1f}, "
      f"backward {tot[2] * 1e3:.1f}, sgd {tot[3] * 1e3:.1f}; {batch / sum(tot) * 1e3 / 1e6:.2f} M samples/s")
