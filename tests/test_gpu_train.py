"""The device SGD trainer (train.py sgd_train mirror) against the reference's
own sgd_train run (tests/golden/train.npz from tests/golden/make_golden_train.py): a 2-layer
DeepThin network (tanh general-path layer -> identity reuse layer), MSE, 3 epochs, with and
without the global-norm clip. The device path runs the exact fp32 FFMA kernels, so the loss
history and the trained factors match the reference's float64 run to ~1e-5 relative."""

import os

import numpy as np
import pytest
import torch

import paper_1802_06944_b200 as D

pytestmark = pytest.mark.gpu

PLANS = [(12, 20, 2, 35, 7), (20, 4, 1, 20, 4)]
ACTS = ["tanh", "identity"]


@pytest.mark.parametrize("tag,clip", [("noclip", None), ("clip", 0.5)])
def test_sgd_train_matches_reference(tag, clip):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "train.npz"))
    layers = []
    for i, ((q, r, rk, m, n), act) in enumerate(zip(PLANS, ACTS)):
        plan = D.LayerPlan(q=q, r_dim=r, rank=rk, m=m, n=n)
        layers.append(D.DeepThinLayer(plan, g[f"{tag}_xf{i}"], g[f"{tag}_wf{i}"], g[f"{tag}_b{i}"],
                                      activation=act, mma="ffma"))
    cfg = D.TrainConfig(learning_rate=0.05, epochs=3, batch_size=16, seed=7, loss="mse", clip_norm=clip)
    x, y = g["x"], g["y"]
    hist = D.sgd_train(layers, (x[:64], y[:64]), (x[64:], y[64:]), cfg)
    np.testing.assert_allclose(np.array(hist), g[f"{tag}_hist"], rtol=2e-5, atol=0)
    for i, layer in enumerate(layers):
        for got, key in ((layer.fp.xf, "xf"), (layer.fp.wf, "wf"), (layer.bias, "b")):
            want = g[f"{tag}_{key}{i}_final"]
            err = np.max(np.abs(got.double().cpu().numpy() - want)) / np.max(np.abs(want))
            assert err <= 2e-5, (tag, i, key, err)


def test_train_config_validation():
    with pytest.raises(D.ArgumentError):
        D.TrainConfig(learning_rate=0.0, epochs=1, batch_size=1, seed=0)
    with pytest.raises(D.ArgumentError):
        D.TrainConfig(learning_rate=0.1, epochs=1, batch_size=1, seed=0, loss="l1")
    with pytest.raises(D.ArgumentError):
        D.TrainConfig(learning_rate=0.1, epochs=1, batch_size=1, seed=0, clip_norm=-1.0)
