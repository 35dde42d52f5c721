"""GPU parity of the row-tile reuse kernel (k_tc_rows.cu): the factored DeepThin layer in one
persistent tcgen05 kernel (P = x_seg @ wf^T in TMEM -> tf32 A operand -> y = act(P XF2^T + b),
TMA-stored). It serves bf16 inputs on reuse geometries (n | q) with n % 64 == 0 and
s * rank <= 32 — BASELINE config 3's hidden/output layers and config 4's FC layers.

Bounds (rel_error = max|a-e| / max|e|, core.py:91-95):
  * <= 1e-3 against the factored bf16 contract emulated in f64 (the only rounding left is P's
    and xf's tf32 truncation);
  * <= 2e-3 against the oracle's layer_forward (kernel.py:296-320) on the same bf16 inputs;
  * activations on the kernel's own logits (fp32 output): |act - oracle act(logits)| <= 1e-6
    (sigmoid/tanh from MUFU ex2 + rcp, act.cuh act_fast).
"""

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D
from test_gpu_forward import bf16_factored_emulated, gpu_x, make_case, rows_path

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["slab", "cluster"])
def rows_kernel(request, monkeypatch):
    """Every test here runs on both row kernels: the slab kernel (k_tc_slab.cu, the default
    where s is a power of two) and the clustered row-tile kernel (DEEPTHIN_ROWS_SLAB=0)."""
    monkeypatch.setenv("DEEPTHIN_ROWS_SLAB", "1" if request.param == "slab" else "0")
    return request.param

GEOS = [
    # q, r_dim, rank, n, m, batch
    (2048, 2048, 3, 256, 16384, 1000),   # config 3 hidden layer, ragged batch
    (2048, 3000, 3, 256, 24000, 300),    # config 3 output layer (3000 = 23.4 chunks)
    (512, 640, 4, 64, 5120, 129),        # s * rank = 32 (full tf32 atom)
    (128, 96, 2, 64, 192, 77),           # s * rank = 4 -> K padded to 8
    (2048, 2048, 1, 256, 16384, 5),      # rank 1 (the reference's fused_matmul case)
]


@pytest.mark.parametrize("geo", GEOS)
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_rows_reuse_matches_contract_and_oracle(geo, out):
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=21, rnd=O.round_bf16, bias_sd=0.1)
    y = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma="bf16", out_dtype=out)
    assert y.dtype == out
    got = y.double().cpu().numpy()
    extra = 2 ** -8 if out == torch.bfloat16 else 0.0
    assert O.rel_error(got, bf16_factored_emulated(d, plan, d["bias"])) <= 1e-3 + extra
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    assert O.rel_error(got, ref) <= 2e-3 + extra


@pytest.mark.parametrize("act", ["relu", "sigmoid", "tanh", "clipped_relu", "softmax"])
def test_rows_activations(act):
    plan, d, fp = make_case(2048, 2048, 3, 256, 16384, 256, seed=4, rnd=O.round_bf16, bias_sd=0.5)
    x = gpu_x(d["x"], torch.bfloat16)
    pre = D.layer_forward(x, fp, d["bias"], "identity", mma="bf16")
    y = D.layer_forward(x, fp, d["bias"], act, mma="bf16", act_arg=2.0)
    want = O.apply_activation(act, pre.double().cpu().numpy(), 2.0)
    err = np.max(np.abs(y.double().cpu().numpy() - want))
    assert err <= 1e-6, (act, err)


def test_rows_deterministic_and_shard_invariant():
    plan, d, fp = make_case(2048, 2048, 3, 256, 16384, 2048, seed=5, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    y1 = D.layer_forward(x, fp, d["bias"], "sigmoid", mma="bf16", out_dtype=torch.bfloat16)
    y2 = D.layer_forward(x, fp, d["bias"], "sigmoid", mma="bf16", out_dtype=torch.bfloat16)
    assert torch.equal(y1, y2)
    for lo, hi in ((0, 128), (128, 1024), (1000, 2048), (77, 300)):
        ys = D.layer_forward(x[lo:hi].contiguous(), fp, d["bias"], "sigmoid", mma="bf16",
                             out_dtype=torch.bfloat16)
        assert torch.equal(ys, y1[lo:hi]), (lo, hi)


def test_rows_large_batch_persistent_tiles():
    # more 128-row tiles than SMs: every CTA loops over several tiles (ring/TMEM phase reuse)
    plan, d, fp = make_case(512, 640, 4, 64, 5120, 148 * 128 * 2 + 50, seed=6, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    pre = D.layer_forward(x, fp, d["bias"], "identity", mma="bf16")
    assert O.rel_error(pre, bf16_factored_emulated(d, plan, d["bias"])) <= 1e-3
    y = D.layer_forward(x, fp, d["bias"], "tanh", mma="bf16")
    assert np.max(np.abs(y.double().cpu().numpy() - np.tanh(pre.double().cpu().numpy()))) <= 1e-6


@pytest.mark.parametrize("act,out", [("sigmoid", torch.bfloat16), ("identity", torch.float32),
                                     ("tanh", torch.bfloat16)])
def test_rows_prepared_operands_equal_per_call(act, out):
    """dt_rows_prepare + dt_forward(DT_FACTORS_ROWS) (operands derived once per pair) gives the
    per-call path's bits; refresh_derived picks up changed factors."""
    from paper_1802_06944_b200 import _lib
    from paper_1802_06944_b200.kernel import _act_code, forward_into
    plan, d, fp = make_case(2048, 2048, 3, 256, 16384, 300, seed=8, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    b = torch.tensor(d["bias"], dtype=torch.float32, device="cuda")
    y0 = torch.empty((300, 2048), dtype=out, device="cuda")
    y1 = torch.empty_like(y0)
    forward_into(x, fp, b, _act_code(act), 20.0, y0, _lib.DT_MMA_BF16)
    forward_into(x, fp, b, _act_code(act), 20.0, y1, _lib.DT_MMA_BF16, cached=True)
    assert fp.rows_prepared(b, _act_code(act), _lib.DT_BF16 if out == torch.bfloat16 else _lib.DT_F32) is not None
    assert torch.equal(y0, y1)
    fp.xf.mul_(0.5)
    fp.refresh_derived()
    forward_into(x, fp, b, _act_code(act), 20.0, y0, _lib.DT_MMA_BF16)
    forward_into(x, fp, b, _act_code(act), 20.0, y1, _lib.DT_MMA_BF16, cached=True)
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_rows_fused_softmax_output_layer(out, fused, monkeypatch):
    """Config 3's output layer (2048 -> 3000, 6 chunks per cluster CTA): the row softmax runs in
    the epilogue in two passes (cluster-wide (max, sum) of the fp32 logits, then the recomputed
    chunks normalised) — or, DEEPTHIN_ROWS_SOFTMAX=0, logits then the separate row kernel.
    Checked against the oracle's softmax of the kernel's own logits (identity launch of the
    same kernel), ragged batch."""
    monkeypatch.setenv("DEEPTHIN_ROWS_SOFTMAX", fused)  # fused epilogue / separate row kernel
    plan, d, fp = make_case(2048, 3000, 3, 256, 24000, 333, seed=12, rnd=O.round_bf16, bias_sd=0.5)
    x = gpu_x(d["x"], torch.bfloat16)
    logits = D.layer_forward(x, fp, d["bias"], "identity", mma="bf16").double().cpu().numpy()
    y = D.layer_forward(x, fp, d["bias"], "softmax", mma="bf16", out_dtype=out)
    got = y.double().cpu().numpy()
    # the fused epilogue works on the fp32 logits; the separate row pass with bf16 output reads
    # bf16 logits back
    oks = []
    for lg in (logits, O.round_bf16(logits)):
        want = O.apply_activation("softmax", lg)
        tol = 1e-6 + (2 ** -8 * want if out == torch.bfloat16 else 2e-6 * want)
        oks.append(bool(np.all(np.abs(got - want) <= tol)))
    assert oks[0] or (out == torch.bfloat16 and oks[1] and fused == "0")
    assert np.allclose(got.sum(axis=1), 1.0, atol=1e-5 if out == torch.float32 else 2e-2)
    y2 = D.layer_forward(x, fp, d["bias"], "softmax", mma="bf16", out_dtype=out)
    assert torch.equal(y, y2)


def test_prepared_path_launches_only_the_row_kernel():
    """cached=True really takes the prepared-operand route: one launch per call (no prep)."""
    from paper_1802_06944_b200 import _lib
    from paper_1802_06944_b200.kernel import _act_code, forward_into
    plan, d, fp = make_case(2048, 2048, 3, 256, 16384, 256, seed=2, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    b = torch.tensor(d["bias"], dtype=torch.float32, device="cuda")
    y = torch.empty((256, 2048), dtype=torch.bfloat16, device="cuda")
    lib = _lib.lib()
    forward_into(x, fp, b, _act_code("sigmoid"), 0.0, y, _lib.DT_MMA_BF16, cached=True)  # prepares
    n0 = lib.dt_launch_counter()
    forward_into(x, fp, b, _act_code("sigmoid"), 0.0, y, _lib.DT_MMA_BF16, cached=True)
    assert lib.dt_launch_counter() - n0 == 1
    n0 = lib.dt_launch_counter()
    forward_into(x, fp, b, _act_code("sigmoid"), 0.0, y, _lib.DT_MMA_BF16)
    assert lib.dt_launch_counter() - n0 == 2   # per-call prep + the row kernel


def _random_rows_geometries(count=10, seed=2024):
    """Seeded random reuse geometries inside the row-tile envelope: n in {64, 128, 256, 320},
    s * round_up(rank, 4) <= 32, r_dim a multiple of 8 (16-byte bf16 rows), ragged batch."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        n = int(rng.choice([64, 128, 256, 320]))
        rank = int(rng.integers(1, 9))
        rp = -(-rank // 4) * 4
        s = int(rng.choice([s for s in (1, 2, 4, 8) if s * rp <= 32]))
        q, r_dim = s * n, 8 * int(rng.integers(1, 400))
        m = -(-(q * r_dim) // n) + int(rng.integers(0, 5))   # sometimes a discarded tail
        out.append((q, r_dim, rank, n, m, int(rng.integers(1, 700))))
    return out


@pytest.mark.parametrize("geo", _random_rows_geometries())
def test_rows_random_geometries(geo):
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=3, rnd=O.round_bf16, bias_sd=0.2)
    x = gpu_x(d["x"], torch.bfloat16)
    for out in (torch.float32, torch.bfloat16):
        assert rows_path(plan, out), geo  # s * rank % 4 != 0 included: rank padded per segment
        y = D.layer_forward(x, fp, d["bias"], mma="bf16", out_dtype=out).double().cpu().numpy()
        extra = 2 ** -8 if out == torch.bfloat16 else 0.0
        assert O.rel_error(y, bf16_factored_emulated(d, plan, d["bias"])) <= 1e-3 + extra, geo


@pytest.mark.parametrize("geo", [(2048, 2048, 3, 256, 16384, 16384 + 40), (2048, 3000, 3, 256, 24000, 2500),
                                 (512, 640, 4, 64, 5120, 4099), (256, 512, 5, 128, 1024, 700),
                                 (256, 384, 9, 256, 384, 333)])
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_slab_kernel_bits_equal_cluster_kernel(geo, out, monkeypatch):
    """The slab kernel performs the clustered kernel's arithmetic row by row (same MMA shapes
    along K, same hi + lo sum, same epilogue): the outputs are bit-identical (the fused softmax
    to rounding: its partials combine in another order), at slab sizes with partial groups and
    16-row tails."""
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=8, rnd=O.round_bf16, bias_sd=0.2)
    x = gpu_x(d["x"], torch.bfloat16)
    for act in ("identity", "sigmoid", "softmax"):
        ys = {}
        for k in ("1", "0"):
            monkeypatch.setenv("DEEPTHIN_ROWS_SLAB", k)
            ys[k] = D.layer_forward(x, fp, d["bias"], act, mma="bf16", out_dtype=out)
        if act == "softmax":  # the partial (max, sum) pairs combine in a different fixed order
            rtol = 1e-5 if out == torch.float32 else 2.0 ** -7
            assert torch.allclose(ys["1"].float(), ys["0"].float(), rtol=rtol, atol=1e-30), (geo, act)
        else:
            assert torch.equal(ys["1"], ys["0"]), (geo, act)
