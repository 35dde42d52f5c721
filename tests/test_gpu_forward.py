"""GPU parity of the forward path (dt_forward) against the pinned oracle and golden vectors.

Tolerances (BASELINE.json north_star), in the reference's metric rel_error =
max|a-e| / max|e| (core.py:91-95):
  * FFMA fp32 path            rel_error <= 1e-5
  * bf16 tcgen05 path (fp32 accumulate) rel_error <= 2e-3, oracle fed the SAME
    bf16-rounded inputs.
"""

import numpy as np
import pytest
import torch

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D

pytestmark = pytest.mark.gpu

ACTS = ("identity", "relu", "sigmoid", "tanh")
F32_TOL = 1e-5
BF16_TOL = 2e-3


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def make_case(q, r_dim, rank, n, m, batch, seed=0, rnd=f32, bias_sd=0.01):
    plan = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: rnd(v) for k, v in O.baseline_inputs(plan, batch, seed=seed, bias_sd=bias_sd).items()}
    fp = D.FactorPair(d["xf"], d["wf"], D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
    return plan, d, fp


def gpu_x(a, dtype):
    return torch.tensor(a, dtype=torch.float32, device="cuda").to(dtype)


def bf16_emulated(d, plan, bias):
    """The single-bf16 contract emulated in f64: W rounded to bf16 (RNE), exact sums — the
    fused kernel (mma="bf16_fused") and the general-geometry MSE forward.

    The kernel must match this up to fp32 accumulation order and the occasional
    one-ulp bf16 double-rounding of a regenerated element."""
    w = O.round_bf16(O.decompress(d["xf"], d["wf"], plan))
    return d["x"] @ w + bias


def bf16_hilo_emulated(d, plan, bias):
    """The two-phase contract (k_regen_wt hi | lo + the any-major GEMM): W carried as a bf16
    hi + lo pair (~16 significant bits), bf16 x exact, fp32 accumulate."""
    w = O.decompress(d["xf"], d["wf"], plan)
    hi = O.round_bf16(w)
    return d["x"] @ (hi + O.round_bf16(w - hi)) + bias


def path_contract(path, d, plan, bias):
    return bf16_emulated(d, plan, bias) if path == "bf16_fused" else bf16_contract(d, plan, bias)


def factored_path(plan, y_dtype=torch.float32):
    """The bf16 tensor-core path computes reuse geometries in factored form: the row-tile kernel
    (k_tc_rows.cu) or the two-GEMM factored form (dt_forward_path)."""
    return D.forward_path(plan, "bf16", torch.bfloat16, y_dtype) in ("rows", "factored")


def rows_path(plan, y_dtype=torch.float32):
    return D.forward_path(plan, "bf16", torch.bfloat16, y_dtype) == "rows"


def bf16_factored_emulated(d, plan, bias):
    """The factored reuse contract in f64: P = x.view(B*s, n) @ wf^T (bf16 operands, fp32 P),
    then y = P.view(B, s*rank) @ XF2^T + bias on tf32 products, XF2 = xf.view(r_dim, s*rank).
    With bf16-valued inputs the only rounding left is P's tf32 rounding (2^-11 relative)."""
    x, xf, wf = d["x"], d["xf"], d["wf"]
    s = plan.q // plan.n
    b = x.shape[0]
    p = (x.reshape(b * s, plan.n) @ wf.T).reshape(b, s * plan.rank)
    xf2 = xf[: plan.r_dim * s].reshape(plan.r_dim, s * plan.rank)
    return p @ xf2.T + bias


def bf16_contract(d, plan, bias, y_dtype=torch.float32):
    """Reuse geometries: the factored contract. Straddling geometries: the memoized runs and the
    fp32-output two-phase form carry wf / W as bf16 hi + lo (the runs' tf32 rounding of P and xf,
    2^-11 relative, is inside the bound); the bf16-output two-phase form rounds W once to bf16
    (k_tc_gemm.cu tc_forward_impl, dt_forward_path)."""
    path = D.forward_path(plan, "bf16", torch.bfloat16, y_dtype)
    if path in ("rows", "factored"):
        return bf16_factored_emulated(d, plan, bias)
    if path == "pair":
        return bf16_emulated(d, plan, bias)
    return bf16_hilo_emulated(d, plan, bias)


def check_activation(y_act, y_pre, act, arg=20.0):
    """The fused activation epilogue, checked on the kernel's own pre-activations."""
    pre = y_pre.detach().double().cpu().numpy() if hasattr(y_pre, "detach") else y_pre
    want = O.apply_activation(act, pre, arg)
    got = y_act.detach().double().cpu().numpy() if hasattr(y_act, "detach") else y_act
    assert np.max(np.abs(got - want)) <= 1e-6 * max(1.0, np.max(np.abs(want))), act


# ---- FFMA fp32 path -----------------------------------------------------------------

def test_ffma_matches_reference_golden_small_plans(golden):
    for i in range(16):
        q, r_dim, rank, m, n = (int(v) for v in golden[f"lf{i}_plan"])
        act = ACTS[int(golden[f"lf{i}_act"][0])]
        fp = D.FactorPair(golden[f"lf{i}_xf"], golden[f"lf{i}_wf"],
                          D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
        y = D.layer_forward(golden[f"lf{i}_x"], fp, golden[f"lf{i}_bias"], act, mma="ffma")
        assert isinstance(y, np.ndarray)
        assert O.rel_error(y, golden[f"lf{i}_y"]) <= F32_TOL, (i, q, r_dim, rank, n)


def test_ffma_fused_matmul_golden_rank1(golden):
    for i in range(16):
        q, r_dim, rank, m, n = (int(v) for v in golden[f"fm{i}_plan"])
        fp = D.FactorPair(golden[f"fm{i}_xf"], golden[f"fm{i}_wf"],
                          D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
        table = D.ReuseTable()
        y, ops = D.fused_matmul(golden[f"fm{i}_x"], fp, reuse=table)
        assert O.rel_error(y, golden[f"fm{i}_y"]) <= F32_TOL
        hits, misses, mul, add = (int(v) for v in golden[f"fm{i}_counts"])
        assert (table.hits, table.misses, ops.multiplies, ops.adds) == (hits, misses, mul, add)


@pytest.mark.parametrize("key", ["c1", "c2", "c4fc1", "c3l1"])
def test_baseline_geometries_vs_reference_golden(golden, key):
    q, r_dim, rank, m, n = (int(v) for v in golden[f"{key}_plan"])
    rnd = f32 if key == "c1" else O.round_bf16
    plan = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
    d = {k: rnd(v) for k, v in O.baseline_inputs(plan, golden[f"{key}_x"].shape[0], 0).items()}
    fp = D.FactorPair(d["xf"], d["wf"], D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
    y = D.layer_forward(d["x"], fp, d["bias"], "identity", mma="ffma")
    assert O.rel_error(y, golden[f"{key}_y"]) <= F32_TOL


def test_ffma_config1_full_batch():
    # BASELINE config 1: q=r_dim=1024, m=4096, n=256, rank 16, batch 64 (reuse path), fp32
    plan, d, fp = make_case(1024, 1024, 16, 256, 4096, 64)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(torch.tensor(d["x"], dtype=torch.float32, device="cuda"), fp, d["bias"],
                        mma="ffma")
    assert y.dtype == torch.float32 and y.shape == (64, 1024)
    assert O.rel_error(y, ref) <= F32_TOL


@pytest.mark.parametrize("geo", [(440, 2048, 24, 320, 2816, 256), (494, 2048, 3, 320, 3162, 100),
                                 (300, 257, 2, 41, 1881, 37)])
def test_ffma_general_path(geo):
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=3)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(d["x"], fp, d["bias"], "identity", mma="ffma")
    assert O.rel_error(y, ref) <= F32_TOL
    # bounded activations shrink max|e| and would inflate rel_error; |act'| <= 1 so
    # the absolute error stays within the pre-activation bound
    for act in ("relu", "tanh", "sigmoid"):
        ya = D.layer_forward(d["x"], fp, d["bias"], act, mma="ffma")
        want = O.apply_activation(act, ref)
        assert np.max(np.abs(ya - want)) <= F32_TOL * np.max(np.abs(ref)), act
        check_activation(ya, y, act)


def test_ffma_bf16_input_exact_products():
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 64, rnd=O.round_bf16)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma="ffma")
    assert O.rel_error(y, ref) <= F32_TOL


# ---- bf16 tcgen05 paths ----------------------------------------------------------------
# "bf16": two-phase (W^T regenerated into L2-resident workspace, then the tcgen05 GEMM), any
# geometry. "bf16_fused": the single kernel regenerating W blocks in shared memory (general
# geometries only).
TC_PATHS = ["bf16", "bf16_fused"]


@pytest.mark.parametrize("path", TC_PATHS)
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_tc_config2_full_batch(seed, path):
    # BASELINE config 2: in 440 -> out 2048, m_f 2816, n_f 320, rank 24, batch 4096
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 4096, seed=seed, rnd=O.round_bf16)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma=path)
    err = O.rel_error(y, ref)
    assert err <= BF16_TOL, err
    assert O.rel_error(y, path_contract(path, d, plan, d["bias"])) <= 1e-3
    if path == "bf16":  # W as bf16 hi + lo: the oracle itself to ~1e-5 (<= 5e-4)
        assert err <= 5e-5, err


GENERAL_GEOS = [
    (494, 2048, 3, 320, 3162, 300),    # config 4 fc1: period 160, tail 128, q % 8 != 0
    (440, 2048, 3, 320, 2816, 1000),   # config 3 layer 0 (rank 3)
    (300, 257, 2, 41, 1881, 129),      # odd everything, ragged r_dim and batch
    (200, 100, 5, 7, 2858, 1),         # n odd (scalar scatter path), batch 1
    (64, 600, 40, 48, 800, 260),       # rank 40 -> padded K of 48
]


@pytest.mark.parametrize("path", TC_PATHS)
@pytest.mark.parametrize("geo", GENERAL_GEOS)
def test_tc_general_geometries(geo, path):
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=5, rnd=O.round_bf16)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma=path)
    # kernel correctness: tight against the path's contract (bf16 hi + lo W for "bf16", the
    # bf16-rounded W for the fused kernel)
    assert O.rel_error(y, path_contract(path, d, plan, d["bias"])) <= 1e-3
    # the contract tolerance is a statistic over many outputs; a 100-output row can
    # exceed it by chance from W's bf16 rounding alone
    if batch * r_dim >= 10_000:
        assert O.rel_error(y, ref) <= BF16_TOL


@pytest.mark.parametrize("geo", [
    (1024, 1024, 16, 256, 4096, 512),  # BASELINE config 1 (reuse: n | q)
    (1024, 1024, 16, 256, 4096, 1),    # config 1, batch 1
    (512, 1536, 72, 128, 6144, 700),   # reuse, rank 72 > 64 (two-phase only)
    (96, 130, 4, 32, 390, 257),        # reuse, ragged r_dim / batch, q % 64 != 0
    (1000, 300, 8, 125, 2400, 33),     # reuse with n % 8 != 0 (scalar W^T stores)
    (13, 17, 3, 5, 45, 9),             # tiny: q < 16, K padded by TMA zero fill
])
def test_tc_reuse_and_edge_geometries(geo):
    # reuse geometries with aligned views take the factored two-GEMM form, the rest two-phase
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=11, rnd=O.round_bf16)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma="bf16")
    assert O.rel_error(y, bf16_contract(d, plan, d["bias"])) <= 1e-3
    if batch * r_dim >= 10_000:
        assert O.rel_error(y, ref) <= BF16_TOL


@pytest.mark.parametrize("path", TC_PATHS)
@pytest.mark.parametrize("act", ["relu", "sigmoid", "tanh", "clipped_relu", "softmax"])
def test_tc_fused_activations(act, path):
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 384, seed=7, rnd=O.round_bf16, bias_sd=0.5)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    x = gpu_x(d["x"], torch.bfloat16)
    pre = D.layer_forward(x, fp, d["bias"], "identity", mma=path)
    assert O.rel_error(pre, ref) <= BF16_TOL          # the contraction (deterministic kernel)
    y = D.layer_forward(x, fp, d["bias"], act, mma=path, act_arg=2.0)
    check_activation(y, pre, act, 2.0)                # the fused epilogue on the same logits


@pytest.mark.parametrize("path", TC_PATHS)
def test_tc_fp32_input_and_bf16_output(path):
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 512, seed=2, rnd=O.round_bf16)
    ref = O.layer_forward(d["x"], d["xf"], d["wf"], plan, d["bias"], "identity")
    y = D.layer_forward(gpu_x(d["x"], torch.float32), fp, d["bias"], mma=path)
    assert O.rel_error(y, ref) <= BF16_TOL
    yb = D.layer_forward(gpu_x(d["x"], torch.bfloat16), fp, d["bias"], mma=path,
                         out_dtype=torch.bfloat16)
    assert yb.dtype == torch.bfloat16
    # bf16 output adds <= 2^-8 relative rounding on top of the operand rounding
    assert O.rel_error(yb.float(), ref) <= BF16_TOL + 2 ** -8


def test_tc_two_phase_agrees_with_fused():
    # The two-phase path carries W as bf16 hi + lo, the fused kernel rounds W once to bf16:
    # each within its own contract, and the two within the single rounding's 2e-3 of each other
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 1024, seed=3, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    a = D.layer_forward(x, fp, d["bias"], mma="bf16")
    b = D.layer_forward(x, fp, d["bias"], mma="bf16_fused")
    assert O.rel_error(a, bf16_hilo_emulated(d, plan, d["bias"])) <= 1e-4
    assert O.rel_error(b, bf16_emulated(d, plan, d["bias"])) <= 1e-3
    assert O.rel_error(a, b.double().cpu().numpy()) <= BF16_TOL


@pytest.mark.parametrize("path", TC_PATHS)
def test_tc_deterministic_and_shard_invariant(path):
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 4096, seed=9, rnd=O.round_bf16)
    x = gpu_x(d["x"], torch.bfloat16)
    b = d["bias"]
    y1 = D.layer_forward(x, fp, b, mma=path)
    y2 = D.layer_forward(x, fp, b, mma=path)
    assert torch.equal(y1, y2)
    # batch sharding (multi-GPU DP) must not change any row's bits
    for lo, hi in ((0, 1024), (1024, 2048), (2048, 4096), (100, 357)):
        ys = D.layer_forward(x[lo:hi].contiguous(), fp, b, mma=path)
        assert torch.equal(ys, y1[lo:hi]), (lo, hi)


def test_empty_batch_and_errors():
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 4, rnd=O.round_bf16)
    for mma in ("ffma", "bf16", "bf16_fused"):
        y = D.layer_forward(torch.zeros((0, 440), device="cuda", dtype=torch.bfloat16), fp, d["bias"],
                            mma=mma)
        assert y.shape == (0, 2048)
    with pytest.raises(D.DimensionError):
        D.layer_forward(torch.zeros((2, 441), device="cuda"), fp, d["bias"])
    with pytest.raises(D.DimensionError):
        D.layer_forward(torch.zeros((2, 440), device="cuda"), fp, np.zeros(7))
    with pytest.raises(D.ArgumentError):
        D.layer_forward(torch.zeros((2, 440), device="cuda"), fp, d["bias"], "gelu")
    with pytest.raises(D.ArgumentError):
        D.layer_forward(np.full((2, 440), np.nan), fp, d["bias"])


def test_decompress_matches_oracle(golden):
    for i in range(24):
        q, r_dim, rank, m, n = (int(v) for v in golden[f"dec{i}_plan"])
        fp = D.FactorPair(golden[f"dec{i}_xf"], golden[f"dec{i}_wf"],
                          D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n))
        w = D.decompress(fp)
        assert O.rel_error(w, golden[f"dec{i}_w"]) <= F32_TOL


def test_session_host_buffers_match_device_path():
    # dt_session_forward (host buffers, chunked over two streams, ragged last chunk) against
    # the device-pointer path on the same inputs
    import ctypes as C
    from paper_1802_06944_b200 import _lib
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 2500, seed=4, rnd=O.round_bf16)
    lib = _lib.lib()
    ps = _lib.plan_struct(fp.plan)
    host = {k: np.ascontiguousarray(d[k], dtype=np.float32) for k in ("xf", "wf", "bias", "x")}
    for mma, code in (("bf16", _lib.DT_MMA_BF16), ("ffma", _lib.DT_MMA_FFMA)):
        sess = C.c_void_p()
        _lib.check(lib.dt_session_create(C.byref(ps), code, host["xf"].ctypes.data,
                                         host["wf"].ctypes.data, host["bias"].ctypes.data,
                                         C.byref(sess)))
        try:
            y = np.empty((2500, 2048), dtype=np.float32)
            h2d, d2h = C.c_int64(), C.c_int64()
            _lib.check(lib.dt_session_forward(sess, 2500, host["x"].ctypes.data, 0, 0.0,
                                              y.ctypes.data, C.byref(h2d), C.byref(d2h)))
            assert h2d.value == 2500 * 440 * 4 and d2h.value == 2500 * 2048 * 4
        finally:
            lib.dt_session_destroy(sess)
        ref = D.layer_forward(gpu_x(d["x"], torch.float32), fp, d["bias"], mma=mma)
        ref = ref.cpu().numpy()
        if mma == "bf16":   # row results do not depend on the batch split
            assert np.array_equal(y, ref)
        else:               # split-K partitioning follows the chunk shape
            assert O.rel_error(y, ref) <= 1e-6


@pytest.mark.parametrize("variant", ["DEEPTHIN_GEMM_WGEN", "DEEPTHIN_GEMM_FUSED"])
def test_tc_alternative_pair_schedules(variant, monkeypatch):
    # the in-CTA W generation (no W^T outside the SM) and the cooperative fused phase 1 are
    # opt-in schedules of the pair kernel that carries the general-geometry forward + MSE
    # (single bf16 W): the gradient's pre-image z = g N / 2 + t within that contract
    monkeypatch.setenv(variant, "1")
    for geo in [(440, 2048, 24, 320, 2816, 1024), (494, 2048, 3, 320, 3162, 300),
                (300, 257, 2, 41, 1881, 129)]:
        q, r_dim, rank, n, m, batch = geo
        plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=6, rnd=O.round_bf16)
        layer = D.DeepThinLayer(D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n), d["xf"],
                                d["wf"], d["bias"], mma="bf16")
        t = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
        norm = float(batch * r_dim)
        loss = torch.empty(1, dtype=torch.float64, device="cuda")
        g = layer.forward_mse(gpu_x(d["x"], torch.bfloat16), t, norm, loss)
        z = (g.double() * (norm / 2.0) + t.double()).cpu().numpy()
        assert O.rel_error(z, bf16_emulated(d, plan, d["bias"])) <= 1e-3, geo


def test_tc_forward_pipeline_matches_serial():
    # pipelined consecutive forwards (phase 1 of call i+1 overlapping the GEMM of call i, W^T
    # slots alternating) give the same bits as serial calls, also when y buffers are reused
    plan, d, fp = make_case(440, 2048, 24, 320, 2816, 1024, seed=12, rnd=O.round_bf16)
    xs = [gpu_x(d["x"], torch.bfloat16)]
    g = torch.Generator(device="cuda").manual_seed(3)
    xs += [torch.randn(1024, 440, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4)]
    b = torch.tensor(d["bias"], dtype=torch.float32, device="cuda")
    serial = [D.layer_forward(x, fp, b, mma="bf16") for x in xs]
    with D.forward_pipeline():
        piped = [D.layer_forward(x, fp, b, mma="bf16") for x in xs for _ in range(2)]
    torch.cuda.synchronize()
    for k, x in enumerate(xs):
        assert torch.equal(piped[2 * k], serial[k]) and torch.equal(piped[2 * k + 1], serial[k]), k


@pytest.mark.parametrize("geo", [
    (440, 2048, 3, 320, 2816, 1000),    # config 3 layer 0: period 8, 18 distinct runs
    (440, 2048, 3, 320, 2816, 5),       # fewer rows than one tile
    (120, 200, 2, 48, 503, 300),        # period 2, discarded tail rows
    (64, 96, 5, 40, 157, 70),           # rank 5, 12 runs, ragged batch
    (256, 1024, 1, 96, 2734, 129),      # rank 1 (the reference's own fused_matmul case)
    (16, 64, 3, 24, 46, 33),            # q below one K block
])
@pytest.mark.parametrize("act", ["identity", "sigmoid", "relu"])
def test_runs_path_low_rank_general_bf16(geo, act):
    """k_tc_runs.cu: low-rank straddling layers with bf16 in/out as the reference's memoized
    runs (kernel.py:99-164) — x . Wruns^T (wf hi + lo) then the tiny per-column combine with xf
    (tf32) — against the oracle on the same bf16 inputs: logits <= 2e-3 + one bf16 ulp; the
    fused activation on those logits."""
    q, r_dim, rank, n, m, batch = geo
    plan, d, fp = make_case(q, r_dim, rank, n, m, batch, seed=13, bias_sd=0.3)
    assert D.forward_path(fp.plan, "bf16", torch.bfloat16, torch.bfloat16) == "runs"
    x = gpu_x(O.round_bf16(d["x"]), torch.bfloat16)
    ref = O.layer_forward(O.round_bf16(d["x"]), d["xf"], d["wf"], plan, d["bias"], "identity")
    z = D.layer_forward(x, fp, d["bias"], "identity", mma="bf16", out_dtype=torch.bfloat16)
    assert O.rel_error(z.double().cpu().numpy(), ref) <= BF16_TOL + 2 ** -8
    y = D.layer_forward(x, fp, d["bias"], act, mma="bf16", out_dtype=torch.bfloat16)
    want = O.apply_activation(act, ref)
    tol = 2 ** -8 * max(1.0, float(np.max(np.abs(want)))) + (0.25 if act == "sigmoid" else 1.0) * \
        BF16_TOL * float(np.max(np.abs(ref)))
    assert np.max(np.abs(y.double().cpu().numpy() - want)) <= tol
