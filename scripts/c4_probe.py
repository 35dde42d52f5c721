"""Config-4 speech model at a short sequence (T env, default 8; B = 64): one warm forward and one
measured forward — the command the LSTM ncu captures run (k_lstm_seq is one launch per forward)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_06944_b200.speech import SpeechRNN  # noqa: E402

T, B = int(os.environ.get("T", 8)), 64
m = SpeechRNN.random(0)
x = torch.randn(T, B, 494, device="cuda").to(torch.bfloat16)
for _ in range(2):
    y = m.forward(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
y = m.forward(x)
e1.record()
torch.cuda.synchronize()
print(f"T={T} B={B}: {e0.elapsed_time(e1) * 1e3:.1f} us per forward, logits {tuple(y.shape)}")
