"""GPU parity of the .dthn loader → device-resident network.

The network is the reference-serialized golden model (tests/golden/dthn.npz: fc0 12→40 rank 2
general path, fc1 40→40 rank 3 reuse path, out 40→9 rank 1 reuse path) plus a BASELINE-config-3
shaped network built here. Checks:
  * decoding on the device is exact: fp32 masters == the stored values rounded by numpy
    (float64 → float32 RNE), bf16 copies == RNE of those;
  * FFMA network forward vs the oracle's layer chain (kernel.py:296-320 per layer, f64) on the
    fp32-rounded factors: rel_error <= 1e-5;
  * bf16 network forward vs the bf16 contract per layer, emulated in f64 with bf16
    intermediates (what the device chain stores between layers): rel_error <= 4e-3 for the
    3-layer chain (2e-3 per layer, north_star; an intermediate that lands on the other side of
    a bf16 rounding boundary carries one bf16 ulp into the next layer);
  * pipelined (PDL) and serial chains agree bit for bit.
"""

import os

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import model_io as mi
from test_gpu_forward import bf16_contract

pytestmark = pytest.mark.gpu

ACTS = ["tanh", "relu", "identity"]


@pytest.fixture(scope="module")
def dthn():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "dthn.npz"))


def oplan(p):
    return O.Plan(q=p.q, r_dim=p.r_dim, rank=p.rank, m=p.m, n=p.n)


def oracle_chain(model, x, acts, *, factor_round, inter_round=None, contract=None):
    h = x
    last = len(model.factors) - 1
    for i, ((_, p), fp, b) in enumerate(zip(model.plans.layers, model.factors, model.biases)):
        d = {"x": h, "xf": factor_round(fp.xf), "wf": factor_round(fp.wf)}
        bias = np.asarray(b, dtype=np.float32).astype(np.float64)
        if contract is None:
            h = O.layer_forward(h, d["xf"], d["wf"], oplan(p), bias, acts[i])
        else:  # intermediates are stored bf16 on the device, the last layer's output fp32
            ydt = torch.float32 if i == last or inter_round is None else torch.bfloat16
            h = O.apply_activation(acts[i], contract(d, oplan(p), bias, ydt))
        if inter_round is not None and i + 1 < len(model.factors):
            h = inter_round(h)
    return h


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_device_decode_is_exact(dthn, tag):
    model = mi.deserialize(dthn[f"{tag}_bytes"].tobytes())
    dm = model.to_device(ACTS, mma="bf16")
    assert dm.h2d_bytes == len(dthn[f"{tag}_bytes"])
    for fp, dfp, b, db in zip(model.factors, dm.factors, model.biases, dm.biases):
        for host, dev in ((fp.xf, dfp.xf), (fp.wf, dfp.wf), (b, db)):
            want = np.asarray(host).astype(np.float32)
            assert np.array_equal(dev.cpu().numpy(), want.reshape(dev.shape))
        for dev, dev16 in zip((dfp.xf, dfp.wf), dfp.bf16()):
            assert torch.equal(dev16, dev.to(torch.bfloat16))


@pytest.mark.parametrize("tag", ["f32", "f64"])
def test_ffma_network_matches_oracle_chain(dthn, tag):
    model = mi.deserialize(dthn[f"{tag}_bytes"].tobytes())
    dm = model.to_device(ACTS, mma="ffma")
    x = np.random.default_rng(3).standard_normal((200, 12))
    y = dm.forward(x)
    assert isinstance(y, np.ndarray) and y.shape == (200, 9)
    want = oracle_chain(model, f32(x), ACTS, factor_round=f32)
    assert O.rel_error(y, want) <= 1e-5


def test_bf16_network_matches_contract_chain(dthn):
    model = mi.deserialize(dthn["f64_bytes"].tobytes())
    dm = model.to_device(ACTS, mma="bf16")
    x = O.round_bf16(np.random.default_rng(4).standard_normal((300, 12)))
    y = dm.forward(torch.tensor(x, dtype=torch.bfloat16, device="cuda"))
    assert y.dtype == torch.float32 and tuple(y.shape) == (300, 9)
    # every golden layer takes the two-phase path: W regenerated from the fp32 masters, then
    # rounded once to bf16 for the bf16 intermediates (bf16_contract, y_dtype bf16); the
    # factors themselves stay fp32
    want = oracle_chain(model, x, ACTS, factor_round=f32, inter_round=O.round_bf16,
                        contract=bf16_contract)
    assert O.rel_error(y.double().cpu().numpy(), want) <= 4e-3


def config3_like(scale_out=3000, hidden=2048, layers=3, seed=0):
    """BASELINE config 3's layer geometry (440 → hidden sigmoid ... → 3000 softmax, n_f = 256
    where it divides the input width else 320, rank 3), fewer hidden layers."""
    rng = np.random.default_rng(seed)
    dims = [440] + [hidden] * layers + [scale_out]
    entries, factors, biases = [], [], []
    for i in range(len(dims) - 1):
        q, r_dim = dims[i], dims[i + 1]
        n = 256 if q % 256 == 0 else 320
        m = -(-(q * r_dim) // n)
        plan = D.LayerPlan(q=q, r_dim=r_dim, rank=3, m=m, n=n)
        entries.append((f"fc{i}", plan))
        # bf16-valued factors: the factored reuse layers read wf as bf16 and xf as tf32, so
        # the contract emulation needs no extra factor rounding
        factors.append(mi.StoredFactors(
            O.round_bf16(rng.normal(0, 3 ** -0.5, (m, 3))).astype(np.float32),
            O.round_bf16(rng.normal(0, 3 ** -0.5, (3, n))).astype(np.float32), plan))
        biases.append(rng.normal(0, 0.01, r_dim).astype(np.float32))
    plans = D.NetworkPlan(layers=tuple(entries), target_ratio=0.01, achieved_total_ratio=0.0,
                          floor_hits=())
    return mi.CompressedModel(plans=plans, factors=factors, biases=biases)


def test_config3_shaped_network_bf16_and_pipeline():
    """Parity on the logits (identity head); the softmax head separately. Softmax turns an
    absolute logit error into a relative probability error (dp/p = dz), so a relative-to-max
    bound on probabilities would measure the logits' magnitude, not the kernels."""
    model = mi.deserialize(mi.serialize(config3_like()))
    x = O.round_bf16(np.random.default_rng(5).standard_normal((512, 440)))
    xt = torch.tensor(x, dtype=torch.bfloat16, device="cuda")
    logits_acts = ["sigmoid"] * 3 + ["identity"]
    serial = model.to_device(logits_acts, mma="bf16", pipeline=False)
    piped = model.to_device(logits_acts, mma="bf16")
    y0 = serial.forward(xt)
    y1 = piped.forward(xt)
    y2 = piped.forward(xt)  # second call: the first layer's W^T slot alternates
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(y1, y2)
    logits = y0.double().cpu().numpy()
    want = oracle_chain(model, x, logits_acts, factor_round=f32, inter_round=O.round_bf16,
                        contract=bf16_contract)
    assert O.rel_error(logits, want) <= 4e-3
    probs = model.to_device(["sigmoid"] * 3 + ["softmax"], mma="bf16").forward(xt)
    got = probs.double().cpu().numpy()
    assert np.allclose(got.sum(axis=1), 1.0, atol=1e-5)
    assert np.max(np.abs(got - O.apply_activation("softmax", logits))) <= 1e-6


@pytest.mark.parametrize("rows,chunks", [(1000, 3), (4096, 4), (100, 4)])
def test_forward_host_pipeline_equals_device_forward(rows, chunks):
    """forward_host (row blocks pipelined over copy / compute / copy streams) returns the bits
    of one forward over the whole batch, also when its static buffers are reused by a second
    call on other inputs and when the last block is ragged."""
    model = config3_like(layers=2)
    dm = model.to_device(["sigmoid"] * 2 + ["softmax"], mma="bf16")
    g = torch.Generator().manual_seed(rows)
    hy = None
    for call in range(2):
        hx = torch.randn(rows, 440, generator=g).to(torch.bfloat16).pin_memory()
        want = dm.forward(hx.cuda(), out_dtype=torch.bfloat16).cpu()
        hy = dm.forward_host(hx, hy, chunks=chunks)
        assert hy.dtype == torch.bfloat16 and tuple(hy.shape) == (rows, 3000)
        assert torch.equal(hy, want), call
    with pytest.raises(D.DimensionError):
        dm.forward_host(torch.zeros(4, 441, dtype=torch.bfloat16))


def test_chain_and_argument_errors(dthn):
    model = mi.deserialize(dthn["f32_bytes"].tobytes())
    with pytest.raises(D.ArgumentError):
        model.to_device(["relu"], mma="bf16")
    with pytest.raises(D.ArgumentError):
        model.to_device(ACTS, mma="tf32")
    broken = mi.CompressedModel(plans=D.NetworkPlan(
        layers=(model.plans.layers[1], model.plans.layers[0]), target_ratio=0.5,
        achieved_total_ratio=0.0, floor_hits=()),  # 40 -> 40 then a 12-input layer
        factors=[model.factors[1], model.factors[0]], biases=[model.biases[1], model.biases[0]])
    with pytest.raises(D.DimensionError):
        broken.to_device("relu")
    dm = model.to_device(ACTS, mma="ffma")
    with pytest.raises(D.DimensionError):
        dm.forward(np.zeros((4, 13)))


def test_row_tile_layer_chaining_is_exact(monkeypatch):
    """Chained row-tile layers (per-tile flags, dt_rows_chain, three rotating activation
    buffers) give the unchained chain's bits, across repeated forwards (monotone flag epochs)
    and a second batch size. Chaining is a feature of the clustered row-tile kernel: the
    unchained run uses it too (the slab kernel's softmax rounds its partial sums in another
    order)."""
    monkeypatch.setenv("DEEPTHIN_ROWS_SLAB", "0")
    model = mi.deserialize(mi.serialize(config3_like(layers=4)))
    acts = ["sigmoid"] * 4 + ["softmax"]
    dm = model.to_device(acts, mma="bf16")
    for rows in (1000, 384):
        x = torch.randn(rows, 440, device="cuda").to(torch.bfloat16)
        dm.chain = False
        want = dm.forward(x, out_dtype=torch.bfloat16).clone()
        dm.chain = True
        for _ in range(3):
            got = dm.forward(x, out_dtype=torch.bfloat16)
            torch.cuda.synchronize()
            assert torch.equal(got, want)
        dm.chain = False


def test_graph_forward_equals_eager():
    """DeviceModel.forward(graph=True): the captured layer chain replays the eager bits."""
    model = mi.deserialize(mi.serialize(config3_like(layers=3)))
    dm = model.to_device(["sigmoid"] * 3 + ["softmax"], mma="bf16")
    x = torch.randn(700, 440, device="cuda").to(torch.bfloat16)
    want = dm.forward(x, out_dtype=torch.bfloat16).clone()
    for _ in range(3):
        got = dm.forward(x, out_dtype=torch.bfloat16, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(got, want)
    x.copy_(torch.randn(700, 440, device="cuda").to(torch.bfloat16))  # same buffer, new data
    want2 = dm.forward(x, out_dtype=torch.bfloat16)
    assert torch.equal(dm.forward(x, out_dtype=torch.bfloat16, graph=True), want2)


def chain_model(dims, ns, seed=7):
    rng = np.random.default_rng(seed)
    entries, factors, biases = [], [], []
    for i, n in enumerate(ns):
        q, r_dim = dims[i], dims[i + 1]
        m = -(-(q * r_dim) // n)
        plan = D.LayerPlan(q=q, r_dim=r_dim, rank=3, m=m, n=n)
        entries.append((f"fc{i}", plan))
        factors.append(mi.StoredFactors(rng.normal(0, 3 ** -0.5, (m, 3)).astype(np.float32),
                                        rng.normal(0, 3 ** -0.5, (3, n)).astype(np.float32), plan))
        biases.append(rng.normal(0, 0.01, r_dim).astype(np.float32))
    plans = D.NetworkPlan(layers=tuple(entries), target_ratio=0.01, achieved_total_ratio=0.0,
                          floor_hits=())
    return mi.CompressedModel(plans=plans, factors=factors, biases=biases)


@pytest.mark.parametrize("rows", [300, 8192])
def test_pipelined_chain_with_back_to_back_general_layers_is_exact(rows):
    """with inference pipelining a layer's GEMM signals its dependents right
    after its prologue, so the next layer (W regeneration, then its GEMM) starts while the
    current one still writes its output. A general-path GEMM whose x is that output must wait
    before loading x. Chain: general -> general -> row-tile reuse -> general, pipelined vs
    serial, bit for bit, repeated (a race shows up as a mismatch on some call)."""
    model = chain_model([440, 560, 2048, 2048, 1000], [320, 320, 256, 320])
    assert [p.reuse_path for _, p in model.plans.layers] == [False, False, True, False]
    acts = ["sigmoid", "tanh", "sigmoid", "identity"]
    serial = model.to_device(acts, mma="bf16", pipeline=False)
    piped = model.to_device(acts, mma="bf16", pipeline=True)
    x = torch.randn(rows, 440, device="cuda").to(torch.bfloat16)
    want = serial.forward(x)
    for _ in range(6):
        got = piped.forward(x)
        torch.cuda.synchronize()
        assert torch.equal(got, want)
    for _ in range(3):  # graph replay of the pipelined chain
        got = piped.forward(x, graph=True)
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_external_x_pipeline_mode_matches_serial():
    """DT_PIPELINE_EXTERNAL_X (independent inputs, the bench's mode): back-to-back forwards of
    one layer over rotating buffers give the serial bits."""
    plan = D.LayerPlan(q=440, r_dim=2048, rank=24, m=2816, n=320)
    rng = np.random.default_rng(1)
    fp = D.FactorPair(rng.normal(0, 0.2, (2816, 24)), rng.normal(0, 0.2, (24, 320)), plan)
    bias = rng.normal(0, 0.01, 2048)
    xs = [torch.randn(4096, 440, device="cuda").to(torch.bfloat16) for _ in range(3)]
    want = [D.layer_forward(x, fp, bias, mma="bf16") for x in xs]
    from paper_1802_06944_b200.kernel import forward_pipeline
    with forward_pipeline(True, external_x=True):
        got = [D.layer_forward(x, fp, bias, mma="bf16") for x in xs * 3]
    torch.cuda.synchronize()
    for k, g in enumerate(got):
        assert torch.equal(g, want[k % 3])


def test_gpu_factor_pair_float64_round_trips_through_dthn():
    """a model whose layers are device FactorPairs built from float64
    factors serializes them as float64 (dtype code 1), bit-exact, like the reference
    (model_io.py:100-110); after an SGD step the file carries the updated values, not a
    stale image."""
    rng = np.random.default_rng(11)
    plan = D.LayerPlan(q=12, r_dim=40, rank=2, m=40, n=12)
    xf, wf = rng.standard_normal((40, 2)), rng.standard_normal((2, 12))
    fp = D.FactorPair(xf, wf, plan)
    assert fp.source_dtype == np.float64
    bias = rng.standard_normal(40)
    model = mi.CompressedModel(plans=D.NetworkPlan(layers=(("fc0", plan),), target_ratio=1.0,
                                                   achieved_total_ratio=0.0, floor_hits=()),
                               factors=[fp], biases=[bias])
    back = mi.deserialize(mi.serialize(model))
    assert back.factors[0].xf.dtype == np.float64
    assert np.array_equal(back.factors[0].xf, xf) and np.array_equal(back.factors[0].wf, wf)
    assert mi.expected_file_size(model) == len(mi.serialize(model))
    img0 = model.image()[0]
    layer = D.DeepThinLayer(plan, xf, wf, bias, mma="ffma")
    model2 = mi.CompressedModel(plans=model.plans, factors=[layer.fp], biases=[bias])
    img_a = model2.image()[0]
    x = torch.randn(8, 12, device="cuda")
    t = torch.randn(8, 40, device="cuda")
    D.train_step(layer, x, t, 0.1)
    torch.cuda.synchronize()
    img_b = model2.image()[0]
    assert img_a == img0 and img_b != img_a
    moved = mi.deserialize(img_b).factors[0]
    assert moved.xf.dtype == np.float64
    assert np.array_equal(moved.xf, layer.fp.xf.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("rows", [1000, 4096, 128])
def test_fused_layer_chain_matches_layer_by_layer(rows):
    """dt_chain_forward (k_tc_chain.cu): the config-3 hidden layers + output layer as ONE kernel
    with the activations kept in shared memory give the bits of the layer-by-layer row-tile
    kernels (same per-layer arithmetic and summation order), with bf16 output (the chain runs
    through the identity head) and fp32 output (the last layer runs on its own). A softmax head
    is never chained: the row-tile kernel fuses it on the fp32 logits."""
    model = mi.deserialize(mi.serialize(config3_like(layers=5)))
    acts = ["sigmoid"] * 5 + ["identity"]
    dm = model.to_device(acts, mma="bf16")
    x = torch.randn(rows, 440, device="cuda").to(torch.bfloat16)
    assert dm._fused_runs(torch.bfloat16) == {1: 5}
    assert dm._fused_runs(torch.float32) == {}  # layers 1-4: the run would end on a sigmoid
    assert model.to_device(["sigmoid"] * 5 + ["softmax"], mma="bf16")._fused_runs(torch.bfloat16) == {}
    for out in (torch.bfloat16, torch.float32):
        dm.fuse = False
        want = dm.forward(x, out_dtype=out).clone()
        dm.fuse = True
        got = dm.forward(x, out_dtype=out)
        torch.cuda.synchronize()
        assert torch.equal(got, want), (out, (got.float() - want.float()).abs().max().item())
    got = dm.forward(x, out_dtype=torch.bfloat16, graph=True)
    torch.cuda.synchronize()
    dm.fuse = False
    assert torch.equal(got, dm.forward(x, out_dtype=torch.bfloat16))
