"""Pure-write, pure-read and copy HBM bandwidth on this GPU (torch fill_ / sum / copy_ over 2 GiB,
CUDA events, best of 10) — the directional rooflines beside MEASURED_PEAKS.json's copy figure."""
import json
import torch

n = 1 << 30  # bf16 elements (2 GiB)
a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
af = a.view(torch.float32)


def best(fn, bytes_, reps=10):
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1))
    return bytes_ / (min(t) * 1e-3) / 1e9


out = {
    "write_gbs_fill": round(best(lambda: a.fill_(1.0), 2 * n), 1),
    "write_gbs_memset": round(best(lambda: a.zero_(), 2 * n), 1),
    "read_gbs_sum": round(best(lambda: af.sum(), 2 * n), 1),
    "copy_gbs": round(best(lambda: b.copy_(a), 4 * n), 1),
}
# a smaller write burst into an L2 full of other dirty lines (config 2's y: 33.5 MB per call)
y = torch.empty(8, 4096 * 2048, dtype=torch.float32, device="cuda")
i = [0]
def burst():
    y[i[0] % 8].fill_(1.0)
    i[0] += 1
out["write_gbs_33MB_rotating"] = round(best(burst, 4096 * 2048 * 4, reps=32), 1)
print(json.dumps(out))
