"""Config-4 probe: SpeechRNN forward at T=500, B=64; per-part timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1802_06944_b200.speech import SpeechRNN
T, B = int(os.environ.get("T", 500)), int(os.environ.get("B", 64))
m = SpeechRNN.random(0)
x = torch.randn(T, B, 494, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = m.forward(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    y = m.forward(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"forward T={T} B={B}: {ms:.2f} ms, {T * B / ms * 1e3 / 1e6:.3f} M frames/s")
y2 = m.forward(x, persistent=False)
torch.cuda.synchronize()
print("persistent == graph:", bool(torch.equal(y, y2)))
st = m._graphs[(T, B)]
e0.record()
for _ in range(3):
    st["graph"].replay()
e1.record(); torch.cuda.synchronize()
print(f"recurrence graph replay: {e0.elapsed_time(e1) / 3:.2f} ms ({e0.elapsed_time(e1) / 3 / T * 1e3:.1f} us/step)")
