"""GPU parity of the backward path (dt_backward), the MSE gradient and the SGD step."""

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D

pytestmark = pytest.mark.gpu

ACTS = ("identity", "relu", "sigmoid", "tanh")
F32_TOL = 1e-5


def plan_of(arr):
    q, r_dim, rank, m, n = (int(v) for v in arr)
    return O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n), D.LayerPlan(q=q, r_dim=r_dim, rank=rank,
                                                                       m=m, n=n)


def test_backward_matches_reference_golden(golden):
    for i in range(12):
        _, p = plan_of(golden[f"lb{i}_plan"])
        act = ACTS[int(golden[f"lb{i}_act"][0])]
        fp = D.FactorPair(golden[f"lb{i}_xf"], golden[f"lb{i}_wf"], p)
        gr = D.layer_backward(golden[f"lb{i}_x"], fp, golden[f"lb{i}_bias"], act,
                              golden[f"lb{i}_up"])
        for mine, key in ((gr.d_xf, "dxf"), (gr.d_wf, "dwf"), (gr.d_input, "dx"), (gr.d_bias, "db")):
            assert O.rel_error(mine, golden[f"lb{i}_{key}"]) <= F32_TOL, (i, key)


@pytest.mark.parametrize("key", ["t5s", "t2"])
def test_training_geometry_gradients(golden, key):
    op, p = plan_of(golden[f"{key}_plan"])
    batch = golden[f"{key}_dx"].shape[0]
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=1).items()}
    fp = D.FactorPair(d["xf"], d["wf"], p)
    y = D.layer_forward(d["x"], fp, d["bias"], mma="ffma")
    loss, dy = D.loss_and_grad("mse", y, d["target"])
    assert loss == pytest.approx(float(golden[f"{key}_loss"][0]), rel=1e-5)
    gr = D.layer_backward(d["x"], fp, d["bias"], "identity", dy)
    for mine, k in ((gr.d_xf, "dxf"), (gr.d_wf, "dwf"), (gr.d_input, "dx"), (gr.d_bias, "db")):
        assert O.rel_error(mine, golden[f"{key}_{k}"]) <= F32_TOL, k


def test_discarded_tail_gets_zero_gradient():
    # pkg/tests/test_grad.py:63-79 — m*n - q*r_dim = 2 tail elements
    op = O.Plan(q=5, r_dim=2, rank=1, m=3, n=4)
    xf, wf = O.init_factors(op, 0.7, O.make_rng(5))
    x = O.make_rng(6).standard_normal((3, 5))
    up = O.make_rng(7).standard_normal((3, 2))
    fp = D.FactorPair(xf, wf, D.LayerPlan(q=5, r_dim=2, rank=1, m=3, n=4))
    gr = D.layer_backward(x, fp, np.zeros(2), "identity", up)
    d_aux = np.concatenate([(x.T @ up).T.ravel(), np.zeros(2)]).reshape(3, 4)
    assert np.allclose(gr.d_xf, d_aux @ wf.T, atol=1e-5)
    assert np.allclose(gr.d_wf, xf.T @ d_aux, atol=1e-5)


def test_zero_upstream_and_shape_errors():
    op = O.Plan(q=6, r_dim=5, rank=2, m=8, n=4)
    xf, wf = O.init_factors(op, 0.7, O.make_rng(0))
    fp = D.FactorPair(xf, wf, D.LayerPlan(q=6, r_dim=5, rank=2, m=8, n=4))
    x = O.make_rng(1).standard_normal((3, 6))
    gr = D.layer_backward(x, fp, np.zeros(5), "tanh", np.zeros((3, 5)))
    for g in (gr.d_xf, gr.d_wf, gr.d_input, gr.d_bias):
        assert not np.any(g)
    with pytest.raises(D.DimensionError):
        D.layer_backward(np.zeros((2, 6)), fp, np.zeros(5), "relu", np.zeros((3, 5)))


def test_backward_deterministic():
    op = O.Plan(q=440, r_dim=2048, rank=24, m=2816, n=320)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, 300, seed=4).items()}
    fp = D.FactorPair(d["xf"], d["wf"], D.LayerPlan(q=440, r_dim=2048, rank=24, m=2816, n=320))
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda")
    up = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    g1 = D.layer_backward(x, fp, d["bias"], "sigmoid", up)
    g2 = D.layer_backward(x, fp, d["bias"], "sigmoid", up)
    for a, b in ((g1.d_xf, g2.d_xf), (g1.d_wf, g2.d_wf), (g1.d_input, g2.d_input), (g1.d_bias, g2.d_bias)):
        assert torch.equal(a, b)


def test_train_step_update_matches_oracle():
    # config-5-shaped reuse layer scaled down; one SGD step at lr 1e-3 (train.py:107-111)
    op = O.Plan(q=512, r_dim=512, rank=8, m=4096, n=64)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, 64, seed=2).items()}
    layer = D.DeepThinLayer(D.LayerPlan(q=512, r_dim=512, rank=8, m=4096, n=64), d["xf"], d["wf"],
                            d["bias"], mma="ffma")
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda")
    t = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    xf0, wf0, b0 = layer.fp.xf.clone(), layer.fp.wf.clone(), layer.bias.clone()
    lsum = D.train_step(layer, x, t, lr=1e-3)
    y = O.layer_forward(d["x"], d["xf"], d["wf"], op, d["bias"])
    loss, dy = O.loss_and_grad("mse", y, d["target"])
    gr = O.layer_backward(d["x"], d["xf"], d["wf"], op, d["bias"], "identity", dy)
    assert float(lsum.item()) / y.size == pytest.approx(loss, rel=1e-5)
    # check the gradients that drove the step (the post-step factors would pass trivially,
    # SURVEY.md §7 hard part 6), then that the step applied exactly p - lr * g in fp32
    assert O.rel_error(layer.d_xf, gr.d_xf) <= F32_TOL
    assert O.rel_error(layer.d_wf, gr.d_wf) <= F32_TOL
    assert O.rel_error(layer.d_bias, gr.d_bias) <= F32_TOL
    for p0, p1, g in ((xf0, layer.fp.xf, layer.d_xf), (wf0, layer.fp.wf, layer.d_wf),
                      (b0, layer.bias, layer.d_bias)):
        assert torch.allclose(p1, p0 - 1e-3 * g, rtol=1e-6, atol=1e-12)


BF16_TOL = 2e-3


@pytest.mark.parametrize("geo", [
    (1024, 1024, 16, 256, 4096, 512),   # config 1 geometry (reuse)
    (512, 1536, 64, 128, 6144, 300),    # config-5-like rank 64, ragged batch
    (2048, 2048, 3, 256, 16384, 128),   # config 3 hidden layer (rank 3, s*rank = 24)
    (96, 130, 4, 32, 400, 70),          # discarded tail (m*n > q*r_dim), s*rank = 12
])
@pytest.mark.parametrize("act", ["identity", "tanh"])
def test_tc_backward_reuse_factored(geo, act):
    # the tensor-core backward of reuse geometries (k_train.cu: our tcgen05 GEMMs over the
    # transposed views, tf32 / bf16 hi+lo; rank % 4 != 0 or unaligned widths take the exact FFMA
    # backward) against the oracle fed the same bf16-rounded inputs
    q, r_dim, rank, n, m, batch = geo
    op = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=4, bias_sd=0.3).items()}
    fp = D.FactorPair(d["xf"], d["wf"], D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
    up = O.round_bf16(O.make_rng(9).standard_normal((batch, r_dim)))
    ref = O.layer_backward(d["x"], d["xf"], d["wf"], op, d["bias"], act, up)
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda").to(torch.bfloat16)
    gr = D.layer_backward(x, fp, d["bias"], act, up, mma="bf16")
    for mine, want, k in ((gr.d_xf, ref.d_xf, "dxf"), (gr.d_wf, ref.d_wf, "dwf"),
                          (gr.d_input, ref.d_input, "dx"), (gr.d_bias, ref.d_bias, "db")):
        assert O.rel_error(mine, want) <= BF16_TOL, (k, O.rel_error(mine, want))
    # the discarded tail of I (rows >= r_dim*s of xf) receives exactly zero gradient
    s = q // n
    assert not torch.any(gr.d_xf[r_dim * s:]).item()


@pytest.mark.parametrize("geo", [
    (8192 // 8, 1024, 16, 128, 8192, 700),   # reuse (k_train.cu: tcgen05 GEMM, MSE epilogue)
    (440, 2048, 24, 320, 2816, 600),         # general (two-phase GEMM epilogue)
])
def test_forward_mse_fused_matches_separate(geo):
    # dt_forward_mse: the MSE gradient in the final GEMM's epilogue. Its pre-image z = g N/2 + t
    # is the layer's output: <= 2e-3 against the oracle on the same bf16 inputs (the general
    # path also equals forward + mse_grad to fp32 rounding), and the fp64 loss is the sum of the
    # same fp32 differences
    q, r_dim, rank, n, m, batch = geo
    op = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=8).items()}
    p = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    layer = D.DeepThinLayer(p, d["xf"], d["wf"], d["bias"], mma="bf16")
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda").to(torch.bfloat16)
    t = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    norm = float(batch * r_dim)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    g = layer.forward_mse(x, t, norm, loss)
    z = g.double() * (norm / 2.0) + t.double()
    want = O.layer_forward(d["x"], d["xf"], d["wf"], op, d["bias"])
    assert O.rel_error(z.cpu().numpy(), want) <= 2e-3
    if not p.reuse_path:  # the general MSE forward rounds W once to bf16 (pair kernel)
        from test_gpu_forward import bf16_emulated
        assert O.rel_error(z.cpu().numpy(), bf16_emulated(d, op, d["bias"])) <= 1e-3
    own = float(((g.double() * norm / 2.0) ** 2).sum())
    assert float(loss.item()) == pytest.approx(own, rel=1e-5)  # fp32 chunk sums


def test_forward_mse_tcgen05_epilogue_large():
    """Config-5-like factored geometry (s*rank = 512): the MSE is the epilogue of our tf32
    tcgen05 GEMM (k_tc_xgemm.cu XE_MSE: target TMA-staged, fp64 loss partials per warp).
    Checked against the oracle's forward on the same bf16 inputs (tf32 contract 2e-3 on the
    gradient's pre-image) and against its own loss definition."""
    q = r_dim = 2048; rank = 64; n = 256; m = q * r_dim // n; batch = 1024
    op = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=3).items()}
    p = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    layer = D.DeepThinLayer(p, d["xf"], d["wf"], d["bias"], mma="bf16")
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda").to(torch.bfloat16)
    t = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    norm = float(batch * r_dim)
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    g = layer.forward_mse(x, t, norm, loss)
    z = O.layer_forward(d["x"], d["xf"], d["wf"], op, d["bias"])
    got_z = g.double().cpu().numpy() * norm / 2.0 + d["target"]
    assert O.rel_error(got_z, z) <= 2e-3
    want_loss = float(((g.double() * norm / 2.0) ** 2).sum())
    assert float(loss.item()) == pytest.approx(want_loss, rel=1e-5)
    assert float(loss.item()) == pytest.approx(float(((z - d["target"]) ** 2).sum()), rel=2e-3)


@pytest.mark.parametrize("geo", [
    (2048, 2048, 64, 256, 16384, 1024),   # config-5-like: MSE epilogue with fused column sums
    (1024, 1024, 16, 128, 8192, 300),     # factored path, our GEMM-2 MSE epilogue
])
def test_forward_mse_keep_for_backward_is_exact(geo):
    """dt_forward_mse_ex keeps P and produces d_bias in the MSE epilogue; dt_backward_ex reuses
    them: d_xf / d_wf equal the recomputing path's bits (same GEMMs on the same P), d_bias agrees
    to fp32 summation order (epilogue column sums vs the separate column-sum kernel), the loss
    is the same fixed-order sum."""
    q, r_dim, rank, n, m, batch = geo
    op = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=5).items()}
    p = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda").to(torch.bfloat16)
    t = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    out = []
    for keep in (False, True):
        layer = D.DeepThinLayer(p, d["xf"], d["wf"], d["bias"], mma="bf16")
        loss = torch.empty(1, dtype=torch.float64, device="cuda")
        g = layer.forward_mse(x, t, float(batch * r_dim), loss, keep_for_backward=keep)
        layer.backward(g)
        out.append((g.clone(), layer.grad_flat.clone(), float(loss.item())))
    assert torch.equal(out[0][0], out[1][0])
    # grad_flat = [d_xf | d_wf | d_bias], 64-element-aligned segments (train.py DeepThinLayer)
    ob = -(-(p.m * p.rank) // 64) * 64 + -(-(p.rank * p.n) // 64) * 64
    assert torch.equal(out[0][1][:ob], out[1][1][:ob])
    db0, db1 = out[0][1][ob:ob + r_dim], out[1][1][ob:ob + r_dim]
    assert torch.allclose(db0, db1, rtol=1e-5, atol=1e-6 * float(db0.abs().max()))
    assert out[1][2] == pytest.approx(out[0][2], rel=1e-12)


@pytest.mark.parametrize("geo", [
    (440, 2048, 24, 320, 2816, 512),    # config 2 geometry (straddling rows, period 8)
    (96, 136, 4, 40, 327, 70),          # discarded tail (m*n > q*r_dim), ragged batch
    (1000, 512, 8, 384, 1334, 200),     # q % 8 == 0, q not a multiple of n
])
@pytest.mark.parametrize("act", ["identity", "tanh"])
def test_tc_backward_general_geometry(geo, act):
    """the tensor-core backward of straddling geometries (k_train.cu xback_general:
    d_W^T = g^T x on tcgen05 with g split bf16 hi | lo, the flat inverse re-layout as a view,
    d_xf / d_wf / d_input as tf32 GEMMs) against the oracle's layer_backward (grad.py:63-95) on
    the same bf16-rounded inputs: <= 2e-3; bitwise repeatable (fixed-order split-K)."""
    q, r_dim, rank, n, m, batch = geo
    op = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    assert q % n != 0
    d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(op, batch, seed=6, bias_sd=0.3).items()}
    fp = D.FactorPair(d["xf"], d["wf"], D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
    up = O.round_bf16(O.make_rng(3).standard_normal((batch, r_dim)))
    ref = O.layer_backward(d["x"], d["xf"], d["wf"], op, d["bias"], act, up)
    x = torch.tensor(d["x"], dtype=torch.float32, device="cuda").to(torch.bfloat16)
    gr = D.layer_backward(x, fp, d["bias"], act, up, mma="bf16")
    for mine, want, k in ((gr.d_xf, ref.d_xf, "dxf"), (gr.d_wf, ref.d_wf, "dwf"),
                          (gr.d_input, ref.d_input, "dx"), (gr.d_bias, ref.d_bias, "db")):
        assert O.rel_error(mine, want) <= BF16_TOL, (k, O.rel_error(mine, want))
    gr2 = D.layer_backward(x, fp, d["bias"], act, up, mma="bf16")
    for a, b in ((gr.d_xf, gr2.d_xf), (gr.d_wf, gr2.d_wf), (gr.d_input, gr2.d_input)):
        assert np.array_equal(np.asarray(a.cpu() if hasattr(a, "cpu") else a),
                              np.asarray(b.cpu() if hasattr(b, "cpu") else b))
