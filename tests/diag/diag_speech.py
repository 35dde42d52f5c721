"""Stage-by-stage comparison of SpeechRNN against the f64 contract emulation (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import deepthin_oracle as O
from test_gpu_speech import build, contract_layer
from paper_1802_06944_b200.speech import GATES
m, orc = build()
T, B = 3, 3
x = O.round_bf16(np.random.default_rng(1).standard_normal((T, B, 494)))
xt = torch.tensor(x, dtype=torch.bfloat16, device="cuda").reshape(T * B, 494)
h = xt; he = x.reshape(T * B, 494)
def cmp(tag, dev, emu):
    d = dev.double().cpu().numpy()
    print(f"{tag:8s} rel {O.rel_error(d, emu):.3e}  max|e| {np.max(np.abs(emu)):.3g}")
for name in ("fc1", "fc2", "fc3"):
    h = m._dense(name, h, "clipped_relu")
    xf, wf, p, b = orc[name]
    he = O.round_bf16(O.apply_activation("clipped_relu", contract_layer(name, he, xf, wf, p, b)))
    cmp(name, h, he)
    he = h.double().cpu().numpy()  # continue from the device values
gx = [m._dense(f"x_{g}", h, "identity") for g in GATES]
gxe = []
for g, t in zip(GATES, gx):
    xf, wf, p, b = orc[f"x_{g}"]
    e = O.round_bf16(contract_layer(f"x_{g}", he, xf, wf, p, b)); gxe.append(e)
    cmp(f"x_{g}", t, e)
# one recurrent layer at a random h
hp = np.random.default_rng(2).standard_normal((B, 2048)) * 0.5
hpt = torch.tensor(hp, dtype=torch.float32, device="cuda")
import paper_1802_06944_b200 as D
for g in GATES:
    fp, b = m.layers[f"h_{g}"]
    y = D.layer_forward(hpt, fp, b, mma="ffma")
    xf, wf, p, bb = orc[f"h_{g}"]
    cmp(f"h_{g}", y, O.layer_forward(hp.astype(np.float32).astype(np.float64), xf, wf, p, bb))
seq = m._recurrence([t.clone() for t in gx], T, B, graph=False)
gxd = [t.double().cpu().numpy() for t in gx]
hp = np.zeros((B, 2048)); c = np.zeros((B, 2048)); se = np.zeros((T * B, 2048))
for t in range(T):
    gh = [contract_layer(f"h_{g}", hp, *orc[f"h_{g}"][:3], orc[f"h_{g}"][3]) for g in GATES]
    hp, c = O.lstm_cell([a[t * B:(t + 1) * B] for a in gxd], gh, c)
    se[t * B:(t + 1) * B] = O.round_bf16(hp)
cmp("seq", seq, se)
y4 = m._dense("fc4", seq, "clipped_relu")
xf, wf, p, b = orc["fc4"]
cmp("fc4", y4, O.round_bf16(O.apply_activation("clipped_relu", contract_layer("fc4", seq.double().cpu().numpy(), xf, wf, p, b))))
yo = m._dense("out", y4, "identity", out_dtype=torch.float32)
xf, wf, p, b = orc["out"]
cmp("out", yo, contract_layer("out", y4.double().cpu().numpy(), xf, wf, p, b))
