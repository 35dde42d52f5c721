"""Host cost of one dt_forward call (config 2, two-phase) vs its GPU time."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib

import os
q, r_dim, rank, n, m, batch = (1024, 1024, 16, 256, 4096, 64) if os.environ.get("HO_C1") else (440, 2048, 24, 320, 2816, 4096)
MMA = _lib.DT_MMA_FFMA if os.environ.get("HO_FFMA") else _lib.DT_MMA_BF16
plan = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
rng = np.random.default_rng(0)
fp = D.FactorPair(rng.standard_normal((m, rank)) / 5, rng.standard_normal((rank, n)) / 5, plan)
x = torch.randn(batch, q, device="cuda").to(torch.float32 if MMA == _lib.DT_MMA_FFMA else torch.bfloat16)
y = torch.empty(batch, r_dim, device="cuda")
b = torch.zeros(r_dim, device="cuda")
lib = _lib.lib()
ps = _lib.plan_struct(plan)
ws = torch.empty(lib.dt_forward_workspace_bytes(C.byref(ps), batch, MMA), dtype=torch.uint8,
                 device="cuda")
sh = torch.cuda.current_stream().cuda_stream


def call():
    lib.dt_forward(C.byref(ps), batch, MMA, x.data_ptr(), _lib.DT_F32 if MMA == _lib.DT_MMA_FFMA else _lib.DT_BF16, fp.xf.data_ptr(),
                   fp.wf.data_ptr(), _lib.DT_F32, b.data_ptr(), 0, 0.0, y.data_ptr(), _lib.DT_F32,
                   ws.data_ptr(), ws.numel(), sh)


for _ in range(20):
    call()
torch.cuda.synchronize()
N = 400
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(N):
    call()
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host {1e6 * (t1 - t0) / N:.2f} us/call, gpu {1e3 * e0.elapsed_time(e1) / N:.2f} us/call")
# GPU-only: the same calls captured in a CUDA graph
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    call_s = s.cuda_stream
    g_ok = True
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            lib.dt_forward(C.byref(ps), batch, MMA, x.data_ptr(), _lib.DT_F32 if MMA == _lib.DT_MMA_FFMA else _lib.DT_BF16,
                           fp.xf.data_ptr(), fp.wf.data_ptr(), _lib.DT_F32, b.data_ptr(), 0, 0.0,
                           y.data_ptr(), _lib.DT_F32, ws.data_ptr(), ws.numel(), s.cuda_stream)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(40):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph-replayed: gpu {1e3 * e0.elapsed_time(e1) / 400:.2f} us/call")
