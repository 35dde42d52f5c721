"""Time dt_matmul for the same shape under each operand order (tf32 and bf16)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1802_06944_b200.core import matmul

def op(rows, cols, trans, dt):
    if trans:
        return torch.randn(cols, rows, device="cuda").to(dt).t()
    return torch.randn(rows, cols, device="cuda").to(dt)

for mma, dt in (("tf32", torch.float32), ("bf16", torch.bfloat16)):
    for (M, N, K) in ((8192, 512, 65536), (65536, 512, 8192), (16384, 8192, 512)):
        for ta, tb in ((0, 1), (1, 0), (0, 0), (1, 1)):
            a, b = op(M, K, ta, dt), op(K, N, tb, dt)
            for _ in range(2):
                matmul(a, b, mma=mma)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                matmul(a, b, mma=mma)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            tf = 2 * M * N * K / (ms * 1e-3) / 1e12
            print(f"{mma} M{M} N{N} K{K} a_{'MN' if ta else 'K'} b_{'K' if tb else 'MN'}: {ms*1e3:8.1f} us {tf:6.1f} TFLOP/s")
