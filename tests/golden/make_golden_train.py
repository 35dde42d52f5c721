"""Golden sgd_train run of the reference (train.py:305-357) on a tiny 2-layer DeepThin network.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_train.py

Writes tests/golden/train.npz: the data, the initial factors/biases, the per-epoch
(train_loss, val_loss) history and the final factors, for two configurations (with and
without the global-norm clip).
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("DEEPTHIN_REF_SRC", "/root/reference/pkg/src"))
from deepthin.core import make_rng  # noqa: E402
from deepthin.grad import TrainConfig  # noqa: E402
from deepthin.planner import LayerPlan  # noqa: E402
from deepthin.train import DeepThinWeights, TrainLayer, sgd_train  # noqa: E402

PLANS = [LayerPlan(q=12, r_dim=20, rank=2, m=35, n=7), LayerPlan(q=20, r_dim=4, rank=1, m=20, n=4)]
ACTS = ["tanh", "identity"]


def main():
    out = {}
    rng = make_rng(3)
    x = rng.standard_normal((96, 12))
    w_true = rng.standard_normal((12, 4)) / 3
    y = np.tanh(x @ w_true) + 0.05 * rng.standard_normal((96, 4))
    out["x"], out["y"] = x, y
    for tag, clip in (("noclip", None), ("clip", 0.5)):
        init = make_rng(11)
        layers = []
        for i, (p, a) in enumerate(zip(PLANS, ACTS)):
            w = DeepThinWeights(p, 0.3, init)
            b = 0.01 * init.standard_normal(p.r_dim)
            out[f"{tag}_xf{i}"], out[f"{tag}_wf{i}"], out[f"{tag}_b{i}"] = w.xf.copy(), w.wf.copy(), b.copy()
            layers.append(TrainLayer(w, b, a))
        cfg = TrainConfig(learning_rate=0.05, epochs=3, batch_size=16, seed=7, loss="mse", clip_norm=clip)
        hist = sgd_train(layers, (x[:64], y[:64]), (x[64:], y[64:]), cfg)
        out[f"{tag}_hist"] = np.array([[e, tr, va] for e, tr, va in hist])
        for i, l in enumerate(layers):
            out[f"{tag}_xf{i}_final"], out[f"{tag}_wf{i}_final"] = l.weights.xf, l.weights.wf
            out[f"{tag}_b{i}_final"] = l.bias
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "train.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
