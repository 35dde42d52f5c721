"""Per-layer bf16 error of the device network chain vs the bf16 contract (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from oracle import deepthin_oracle as O
import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import model_io as mi
from test_gpu_forward import bf16_contract, bf16_emulated
from test_gpu_model import config3_like, oplan, f32

g = np.load("tests/golden/dthn.npz")
for label, model, acts, x in (
        ("golden", mi.deserialize(g["f64_bytes"].tobytes()), ["tanh", "relu", "identity"],
         O.round_bf16(np.random.default_rng(4).standard_normal((300, 12)))),
        ("c3like", mi.deserialize(mi.serialize(config3_like())), ["sigmoid"] * 3 + ["identity"],
         O.round_bf16(np.random.default_rng(5).standard_normal((512, 440))))):
    dm = model.to_device(acts, mma="bf16")
    h = x
    for i, ((_, p), fp, b) in enumerate(zip(model.plans.layers, model.factors, model.biases)):
        d = {"x": h, "xf": f32(fp.xf), "wf": f32(fp.wf)}
        bias = f32(b)
        pre_want = bf16_contract(d, oplan(p), bias)
        pre_w = bf16_emulated(d, oplan(p), bias)
        pre_exact = h @ O.decompress(d["xf"], d["wf"], oplan(p)) + bias
        y = D.layer_forward(torch.tensor(h, dtype=torch.bfloat16, device="cuda"), dm.factors[i],
                            dm.biases[i], "identity", mma="bf16").double().cpu().numpy()
        print(label, i, p, "dev-vs-contract %.3e dev-vs-exact %.3e contract-vs-exact %.3e Wemul-vs-exact %.3e"
              % (O.rel_error(y, pre_want), O.rel_error(y, pre_exact), O.rel_error(pre_want, pre_exact),
                 O.rel_error(pre_w, pre_exact)), "max|y|", np.abs(pre_exact).max())
        h = O.round_bf16(O.apply_activation(acts[i], pre_want))
