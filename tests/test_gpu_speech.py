"""GPU parity of BASELINE config 4 (speech-RNN-shaped model, paper_1802_06944_b200/speech.py).

Every contraction is a DeepThin layer checked elsewhere against the pinned oracle; here the
whole model (fc1-3 -> LSTM with 8 compressed gate matrices -> fc4 -> out) is compared with
oracle.speech_forward in f64:
  * against the device contract emulated in f64 (bf16 stored activations, W rounded to bf16 on
    the general-path fc1, factored reuse layers exact on bf16-valued factors, the recurrence in
    fp32): rel_error <= 1e-2 on the logits — six stored bf16 stages in series (fc1-3, the gate
    inputs, the sequence, fc4), each able to differ from the emulation by one bf16 ulp (2^-8
    relative, 2 across a binade boundary) where the two round independently;
  * against the unrounded f64 oracle: rel_error <= 2e-2 (bf16 activations everywhere);
  * the CUDA-graph replay equals eager execution bit for bit, and repeats are deterministic.
"""

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D
from paper_1802_06944_b200.speech import GATES, SpeechRNN, compressed_plan

pytestmark = pytest.mark.gpu


def build(seed=3, n_in=494, hidden=2048, n_out=29):
    rng = np.random.default_rng(seed)
    shapes = {"fc1": (n_in, hidden, 3), "fc2": (hidden, hidden, 3), "fc3": (hidden, hidden, 3),
              "fc4": (hidden, hidden, 3), "out": (hidden, n_out, 1)}
    for g in GATES:
        shapes[f"x_{g}"] = (hidden, hidden, 32)
        shapes[f"h_{g}"] = (hidden, hidden, 32)
    dev, orc = {}, {}
    for name in SpeechRNN.NAMES:
        q, r_dim, rank = shapes[name]
        p = compressed_plan(q, r_dim, rank)
        sd = (rank * q) ** -0.25  # variance-preserving (speech.py SpeechRNN.random)
        xf = O.round_bf16(rng.normal(0, sd, (p.m, rank)))
        wf = O.round_bf16(rng.normal(0, sd, (rank, p.n)))
        b = rng.normal(0, 0.01, r_dim)
        dev[name] = (D.FactorPair(xf.astype(np.float32), wf.astype(np.float32), p), b.astype(np.float32))
        orc[name] = (xf, wf, O.Plan(q=p.q, r_dim=p.r_dim, rank=p.rank, m=p.m, n=p.n),
                     b.astype(np.float32).astype(np.float64))
    return SpeechRNN(dev), orc


def contract_layer(name, h, xf, wf, plan, b):
    if name.startswith("h_"):                      # recurrence: exact fp32 FFMA
        return O.layer_forward(h, xf, wf, plan, b)
    if plan.q % plan.n:                            # general path: W^T regenerated in bf16
        return h @ O.round_bf16(O.decompress(xf, wf, plan)) + b
    s = plan.q // plan.n                           # factored reuse path
    p = (h.reshape(h.shape[0] * s, plan.n) @ wf.T).reshape(h.shape[0], s * plan.rank)
    return p @ xf[: plan.r_dim * s].reshape(plan.r_dim, s * plan.rank).T + b


@pytest.fixture(scope="module")
def model():
    return build()


def test_speech_forward_matches_oracle(model):
    m, orc = model
    T, B = 5, 3
    x = O.round_bf16(np.random.default_rng(1).standard_normal((T, B, 494)))
    y = m.forward(torch.tensor(x, dtype=torch.bfloat16, device="cuda"))
    assert y.shape == (T, B, 29) and y.dtype == torch.float32
    got = y.double().cpu().numpy()
    want = O.speech_forward(x, orc, layer=contract_layer, store=O.round_bf16)
    assert O.rel_error(got, want) <= 1e-2
    assert O.rel_error(got, O.speech_forward(x, orc)) <= 2e-2


def test_speech_graph_equals_eager_and_repeats(model):
    m, _ = model
    T, B = 7, 4
    x = torch.randn(T, B, 494, device="cuda").to(torch.bfloat16)
    y1 = m.forward(x, graph=True, persistent=False)
    y2 = m.forward(x, graph=True, persistent=False)   # replay of the captured recurrence
    y3 = m.forward(x, graph=False, persistent=False)
    y4 = m.forward(x)                                 # the persistent one-kernel recurrence
    y5 = m.forward(x)
    assert torch.equal(y1, y2) and torch.equal(y1, y3)
    assert torch.equal(y4, y5)
    # same arithmetic and summation order as the per-step kernels
    assert torch.equal(y1, y4)


def test_lstm_gates_match_oracle(model):
    """dt_lstm_gates (the four recurrent contractions of one step, 3xTF32 tensor-core tiles,
    ~fp32 accuracy) against the oracle's layer_forward per gate: rel_error <= 1e-5."""
    import ctypes as C
    from paper_1802_06944_b200 import _lib
    m, orc = model
    lib = _lib.lib()
    hl = [m.layers[f"h_{g}"] for g in GATES]
    for B in (1, 64, 100):
        h = np.random.default_rng(B).standard_normal((B, 2048)).astype(np.float32)
        ht = torch.tensor(h, device="cuda")
        gh = [torch.empty((B, 2048), device="cuda") for _ in GATES]
        ps = _lib.plan_struct(hl[0][0].plan)
        ws = torch.empty(lib.dt_lstm_gates_workspace_bytes(C.byref(ps), B), dtype=torch.uint8,
                         device="cuda")
        P = lambda ts: (C.c_void_p * 4)(*[t.data_ptr() for t in ts])
        _lib.check(lib.dt_lstm_gates(C.byref(ps), B, ht.data_ptr(), P([fp.xf for fp, _ in hl]),
                                     P([fp.wf for fp, _ in hl]), P([b for _, b in hl]), P(gh),
                                     ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
        for g, gate in enumerate(GATES):
            xf, wf, p, b = orc[f"h_{gate}"]
            want = O.layer_forward(h.astype(np.float64), xf, wf, p, b)
            assert O.rel_error(gh[g].double().cpu().numpy(), want) <= 1e-5, (B, gate)


def test_speech_shape_errors(model):
    m, _ = model
    with pytest.raises(D.DimensionError):
        m.forward(torch.zeros(3, 2, 100, device="cuda"))


@pytest.mark.parametrize("H,n,R,B,T", [(300, 60, 8, 5, 6), (256, 128, 4, 33, 4), (96, 12, 2, 64, 5),
                                       (512, 256, 12, 17, 3)])
def test_lstm_padded_geometries(H, n, R, B, T):
    """Gate geometries off config 4's shape: n % 8 != 0 (segment dots padded to n8 with zeros),
    rank % 8 != 0 (the P tile's rank rows padded), odd batch. Per gate against the oracle
    (<= 1e-5), and the persistent recurrence (dt_lstm_sequence) bit-equal to the per-step form
    (dt_lstm_gates + dt_lstm_cell) and within 1e-4 of the f64 cell recursion on its own gx."""
    import ctypes as C
    from paper_1802_06944_b200 import _lib
    from test_gpu_forward import make_case
    lib = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    cases = [make_case(H, H, R, n, H * H // n, 1, seed=40 + g, bias_sd=0.1) for g in range(4)]
    ps = _lib.plan_struct(cases[0][2].plan)
    P = lambda ts: (C.c_void_p * 4)(*[t.data_ptr() for t in ts])
    xfs, wfs = P([c[2].xf for c in cases]), P([c[2].wf for c in cases])
    bs_t = [torch.tensor(c[1]["bias"], dtype=torch.float32, device="cuda") for c in cases]
    bs = P(bs_t)
    rng = np.random.default_rng(H + B)
    # gates of one step
    h = rng.standard_normal((B, H)).astype(np.float32)
    ht = torch.tensor(h, device="cuda")
    gh = [torch.empty((B, H), device="cuda") for _ in range(4)]
    wsg = torch.empty(lib.dt_lstm_gates_workspace_bytes(C.byref(ps), B), dtype=torch.uint8, device="cuda")
    _lib.check(lib.dt_lstm_gates(C.byref(ps), B, ht.data_ptr(), xfs, wfs, bs, P(gh), wsg.data_ptr(),
                                 wsg.numel(), st))
    for g, (plan, d, _) in enumerate(cases):
        want = O.layer_forward(h.astype(np.float64), d["xf"], d["wf"], plan, d["bias"])
        assert O.rel_error(gh[g].double().cpu().numpy(), want) <= 1e-5, g
    # the recurrence: persistent kernel vs per-step kernels vs f64
    gx = [torch.tensor(O.round_bf16(rng.standard_normal((T * B, H))), dtype=torch.float32,
                       device="cuda").to(torch.bfloat16) for _ in range(4)]
    need = lib.dt_lstm_sequence_workspace_bytes(C.byref(ps), B)
    assert need > 0
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    out = torch.empty((T * B, H), dtype=torch.bfloat16, device="cuda")
    _lib.check(lib.dt_lstm_sequence(C.byref(ps), T, B, P(gx), xfs, wfs, bs, out.data_ptr(),
                                    ws.data_ptr(), ws.numel(), st))
    c = torch.zeros((B, H), device="cuda")
    h32 = torch.zeros((B, H), device="cuda")
    steps = torch.empty_like(out)
    for t in range(T):
        _lib.check(lib.dt_lstm_gates(C.byref(ps), B, h32.data_ptr(), xfs, wfs, bs, P(gh),
                                     wsg.data_ptr(), wsg.numel(), st))
        _lib.check(lib.dt_lstm_cell(B, H, P([x[t * B:(t + 1) * B] for x in gx]), H, P(gh),
                                    c.data_ptr(), h32.data_ptr(), steps[t * B:].data_ptr(), st))
    torch.cuda.synchronize()
    assert torch.equal(out, steps)
    hh, cc = np.zeros((B, H)), np.zeros((B, H))
    gxn = [x.double().cpu().numpy() for x in gx]
    for t in range(T):
        ghh = [O.layer_forward(hh, d["xf"], d["wf"], plan, d["bias"]) for plan, d, _ in cases]
        hh, cc = O.lstm_cell([x[t * B:(t + 1) * B] for x in gxn], ghh, cc)
        got = out[t * B:(t + 1) * B].double().cpu().numpy()
        assert np.max(np.abs(got - hh)) <= 2 ** -8 + 1e-4, t  # bf16 output rounding


@pytest.mark.parametrize("H,n,R,B,T", [(512, 256, 12, 17, 4), (1024, 256, 8, 64, 3)])
def test_lstm_sequence_fused_gate_clusters_equal_three_phase_form(H, n, R, B, T, monkeypatch):
    """The fused gate-cluster recurrence (four gates of a 64-column block in a cluster of four,
    DSMEM scatter, cell state in registers, two grid barriers per step: the default when the
    geometry allows) gives the bits of the three-phase form (DEEPTHIN_LSTM_FUSED=0), also with
    ragged batch rows and when called twice on the same workspace."""
    import ctypes as C
    from paper_1802_06944_b200 import _lib
    from test_gpu_forward import make_case
    lib = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    cases = [make_case(H, H, R, n, H * H // n, 1, seed=70 + g, bias_sd=0.1) for g in range(4)]
    ps = _lib.plan_struct(cases[0][2].plan)
    P = lambda ts: (C.c_void_p * 4)(*[t.data_ptr() for t in ts])
    xfs, wfs = P([c[2].xf for c in cases]), P([c[2].wf for c in cases])
    bs_t = [torch.tensor(c[1]["bias"], dtype=torch.float32, device="cuda") for c in cases]
    bs = P(bs_t)
    rng = np.random.default_rng(H + B)
    gx = [torch.tensor(rng.standard_normal((T * B, H)), dtype=torch.float32,
                       device="cuda").to(torch.bfloat16) for _ in range(4)]
    ws = torch.empty(lib.dt_lstm_sequence_workspace_bytes(C.byref(ps), B), dtype=torch.uint8,
                     device="cuda")
    outs = {}
    for mode in ("0", "1", "1"):
        monkeypatch.setenv("DEEPTHIN_LSTM_FUSED", mode)
        out = torch.empty((T * B, H), dtype=torch.bfloat16, device="cuda")
        _lib.check(lib.dt_lstm_sequence(C.byref(ps), T, B, P(gx), xfs, wfs, bs, out.data_ptr(),
                                        ws.data_ptr(), ws.numel(), st))
        torch.cuda.synchronize()
        if mode in outs:
            assert torch.equal(out, outs[mode])
        outs[mode] = out
    assert torch.equal(outs["0"], outs["1"])
    assert float(outs["1"].float().abs().max()) > 0.05
