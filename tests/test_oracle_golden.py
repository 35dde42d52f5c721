"""Pin the CPU oracle against the reference's own outputs (golden.npz) and known answers.

CPU-only. The golden vectors were produced by importing the reference package
(tests/golden/make_golden.py); the known answers are the ones the reference's
test-suite freezes (pkg/tests/test_factor.py:47-52, :141-149,
test_kernel.py:133-150, :250-262, test_grad.py:28-79).
"""

import math

import numpy as np
import pytest

from oracle import deepthin_oracle as O

ACTS = ("identity", "relu", "sigmoid", "tanh")


def plan_from(arr):
    q, r_dim, rank, m, n = (int(v) for v in arr)
    return O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)


class TestSeeding:
    def test_make_rng_stream(self, golden):
        assert np.array_equal(O.make_rng(7).standard_normal(16), golden["rng_make7"])

    def test_spawn_streams(self, golden):
        got = np.stack([r.standard_normal(8) for r in O.spawn_rngs(3, 4)])
        assert np.array_equal(got, golden["rng_spawn3"])

    def test_sample_normal(self, golden):
        assert np.array_equal(O.sample_normal(O.make_rng(11), 0.5, 0.25, (4, 5)),
                              golden["rng_sample"])


class TestIndexLaws:
    def test_phase_phasecount_predict_reuse(self, golden):
        for row in golden["index_laws"]:
            q, r_dim, n, m, pc, d, t = (int(v) for v in row[:7])
            phases = row[7:11]
            cols = row[11:15]
            p = O.Plan(q=q, r_dim=r_dim, rank=1, m=m, n=n)
            assert O.phase_count(p) == pc
            assert O.predict_reuse(p) == (d, t)
            assert [O.phase(int(c), p) for c in cols] == phases.tolist()

    def test_relayout(self, golden):
        p = O.Plan(q=7, r_dim=5, rank=1, m=7, n=5)
        got = np.array([O.relayout_index(k, p) for k in range(35)])
        assert np.array_equal(got, golden["relayout_7x5"])

    def test_frozen_2x3_layout(self):
        # pkg/tests/test_factor.py:47-52
        p = O.Plan(q=3, r_dim=2, rank=1, m=2, n=3)
        want = {0: (0, 0), 1: (1, 0), 2: (2, 0), 3: (0, 1), 4: (1, 1), 5: (2, 1)}
        for k, rc in want.items():
            assert O.relayout_index(k, p) == rc
        with pytest.raises(O.ArgumentError):
            O.relayout_index(6, p)

    def test_frozen_phases(self):
        # pkg/tests/test_factor.py:141-149
        p = O.Plan(q=3, r_dim=4, rank=1, m=3, n=4)
        assert [O.phase(c, p) for c in range(4)] == [0, 3, 2, 1]
        assert O.phase_count(p) == 4
        p = O.Plan(q=12, r_dim=6, rank=1, m=18, n=4)
        assert O.phase_count(p) == 1 and O.is_reuse_path(p)

    def test_frozen_reuse_predictions(self):
        # pkg/tests/test_kernel.py:133-150
        assert O.predict_reuse(O.Plan(q=12, r_dim=30, rank=1, m=30, n=12)) == (1, 30)
        one = O.predict_reuse(O.Plan(q=10, r_dim=7, rank=1, m=10, n=7))
        three = O.predict_reuse(O.Plan(q=10, r_dim=21, rank=1, m=30, n=7))
        assert three[0] == one[0] and three[1] == 3 * one[1]

    def test_plan_validation(self):
        with pytest.raises(O.ArgumentError):
            O.Plan(q=4, r_dim=4, rank=1, m=3, n=5)   # m*n < q*r_dim
        with pytest.raises(O.ArgumentError):
            O.Plan(q=0, r_dim=4, rank=1, m=3, n=5)


class TestDecompress:
    def test_bit_identical_to_reference(self, golden):
        for i in range(24):
            p = plan_from(golden[f"dec{i}_plan"])
            xf, wf = golden[f"dec{i}_xf"], golden[f"dec{i}_wf"]
            assert np.array_equal(O.decompress(xf, wf, p), golden[f"dec{i}_w"])
            assert np.array_equal(O.scatter_decompress(xf, wf, p), golden[f"dec{i}_w"])

    @pytest.mark.parametrize("key", ["c1", "c2", "c4fc1", "c3l1"])
    def test_baseline_geometry_samples(self, golden, key):
        p = plan_from(golden[f"{key}_plan"])
        d = O.baseline_inputs(p, 1, seed=0)
        rnd = (lambda a: a.astype(np.float32).astype(np.float64)) if key == "c1" else O.round_bf16
        w = O.decompress(rnd(d["xf"]), rnd(d["wf"]), p)
        ii, jj = golden[f"{key}_wsample"]
        assert np.array_equal(w[ii, jj], golden[f"{key}_wvals"])

    def test_all_ones_and_zero(self):
        # pkg/tests/test_factor.py:79-89
        p = O.Plan(q=6, r_dim=4, rank=1, m=6, n=4)
        xf, wf = O.init_factors(p, 1.0, O.make_rng(1))
        w = O.decompress(np.ones_like(xf), wf, p)
        assert np.array_equal(w.T.ravel(), np.tile(wf.ravel(), p.m)[:24])
        assert not O.decompress(np.zeros_like(xf), wf, p).any()


class TestForward:
    def test_fused_rank1_values_and_counts(self, golden):
        for i in range(16):
            p = plan_from(golden[f"fm{i}_plan"])
            x = golden[f"fm{i}_x"]
            table = O.ReuseTable()
            y, ops = O.fused_matmul(x, golden[f"fm{i}_xf"], golden[f"fm{i}_wf"], p, reuse=table)
            assert O.rel_error(y, golden[f"fm{i}_y"]) <= 1e-12
            hits, misses, mul, add = golden[f"fm{i}_counts"]
            assert (table.hits, table.misses, ops.multiplies, ops.adds) == (hits, misses, mul, add)

    def test_fused_f32_route(self, golden):
        p = O.Plan(q=64, r_dim=48, rank=1, m=192, n=16)
        y, _ = O.fused_matmul(golden["fm32_x"], golden["fm32_xf"], golden["fm32_wf"], p)
        assert y.dtype == np.float32
        assert O.rel_error(y, golden["fm32_y"]) <= 1e-6

    def test_fused_rank_r_superposition(self):
        # the rank-r extension equals decompress + matmul
        rng = np.random.default_rng(0)
        for _ in range(30):
            q, r_dim = int(rng.integers(1, 60)), int(rng.integers(1, 60))
            n = int(rng.integers(1, q * r_dim + 1))
            p = O.Plan(q=q, r_dim=r_dim, rank=int(rng.integers(1, 5)), m=-(-(q * r_dim) // n), n=n)
            xf, wf = O.init_factors(p, 1.0, O.make_rng(int(rng.integers(1 << 30))))
            x = rng.standard_normal((3, q))
            y, _ = O.fused_matmul(x, xf, wf, p)
            assert O.rel_error(y, x @ O.decompress(xf, wf, p)) <= 1e-10

    def test_layer_forward_small(self, golden):
        for i in range(16):
            p = plan_from(golden[f"lf{i}_plan"])
            act = ACTS[int(golden[f"lf{i}_act"][0])]
            y = O.layer_forward(golden[f"lf{i}_x"], golden[f"lf{i}_xf"], golden[f"lf{i}_wf"], p,
                                golden[f"lf{i}_bias"], act)
            assert O.rel_error(y, golden[f"lf{i}_y"]) <= 1e-12

    @pytest.mark.parametrize("key", ["c1", "c2", "c4fc1", "c3l1"])
    def test_layer_forward_baseline_geometry(self, golden, key):
        p = plan_from(golden[f"{key}_plan"])
        batch = golden[f"{key}_x"].shape[0]
        d = O.baseline_inputs(p, batch, seed=0)
        rnd = (lambda a: a.astype(np.float32).astype(np.float64)) if key == "c1" else O.round_bf16
        d = {k: rnd(v) for k, v in d.items()}
        assert np.array_equal(d["x"], golden[f"{key}_x"])
        y = O.layer_forward(d["x"], d["xf"], d["wf"], p, d["bias"], "identity")
        assert O.rel_error(y, golden[f"{key}_y"]) <= 1e-12

    def test_known_activation_answers(self):
        # pkg/tests/test_kernel.py:250-262
        p = O.Plan(q=4, r_dim=4, rank=1, m=4, n=4)
        xf, wf = O.init_factors(p, 1.0, O.make_rng(1))
        out = O.layer_forward(np.ones((2, 4)), np.zeros_like(xf), wf, p, -np.ones(4), "relu")
        assert not out.any()
        out = O.layer_forward(np.ones((2, 4)), np.zeros_like(xf), wf, p, np.zeros(4), "sigmoid")
        assert np.all(out == 0.5)

    def test_errors(self):
        p = O.Plan(q=6, r_dim=6, rank=1, m=9, n=4)
        xf, wf = O.init_factors(p, 1.0, O.make_rng(0))
        with pytest.raises(O.DimensionError):
            O.fused_matmul(np.zeros((2, 7)), xf, wf, p)
        with pytest.raises(O.DimensionError):
            O.layer_forward(np.zeros((1, 6)), xf, wf, p, np.zeros(5))
        with pytest.raises(O.ArgumentError):
            O.as_matrix(np.array([[np.nan]]))


class TestBackward:
    def test_layer_backward_small(self, golden):
        for i in range(12):
            p = plan_from(golden[f"lb{i}_plan"])
            act = ACTS[int(golden[f"lb{i}_act"][0])]
            gr = O.layer_backward(golden[f"lb{i}_x"], golden[f"lb{i}_xf"], golden[f"lb{i}_wf"], p,
                                  golden[f"lb{i}_bias"], act, golden[f"lb{i}_up"])
            for mine, key in ((gr.d_xf, "dxf"), (gr.d_wf, "dwf"), (gr.d_input, "dx"),
                              (gr.d_bias, "db")):
                assert O.rel_error(mine, golden[f"lb{i}_{key}"]) <= 1e-12, (i, key)

    @pytest.mark.parametrize("key", ["t5s", "t2"])
    def test_training_geometry(self, golden, key):
        p = plan_from(golden[f"{key}_plan"])
        batch = golden[f"{key}_dx"].shape[0]
        d = {k: O.round_bf16(v) for k, v in O.baseline_inputs(p, batch, seed=1).items()}
        y = O.layer_forward(d["x"], d["xf"], d["wf"], p, d["bias"], "identity")
        loss, dy = O.loss_and_grad("mse", y, d["target"])
        assert loss == pytest.approx(float(golden[f"{key}_loss"][0]), rel=1e-12)
        gr = O.layer_backward(d["x"], d["xf"], d["wf"], p, d["bias"], "identity", dy)
        for mine, k in ((gr.d_xf, "dxf"), (gr.d_wf, "dwf"), (gr.d_input, "dx"), (gr.d_bias, "db")):
            assert O.rel_error(mine, golden[f"{key}_{k}"]) <= 1e-10, k

    def test_losses(self, golden):
        l1, g1 = O.loss_and_grad("mse", golden["loss_y"], golden["loss_t"])
        assert l1 == pytest.approx(float(golden["loss_mse"][0]), rel=1e-14)
        assert np.allclose(g1, golden["loss_mse_grad"], rtol=0, atol=1e-15)
        l2, g2 = O.loss_and_grad("softmax_cross_entropy", golden["loss_y"], np.arange(5) % 7)
        assert l2 == pytest.approx(float(golden["loss_ce"][0]), rel=1e-14)
        assert np.allclose(g2, golden["loss_ce_grad"], rtol=0, atol=1e-15)

    def test_discarded_tail_zero_gradient(self):
        # pkg/tests/test_grad.py:63-79: m*n - q*r_dim = 2 tail elements
        p = O.Plan(q=5, r_dim=2, rank=1, m=3, n=4)
        xf, wf = O.init_factors(p, 0.7, O.make_rng(5))
        x = O.make_rng(6).standard_normal((3, 5))
        up = O.make_rng(7).standard_normal((3, 2))
        gr = O.layer_backward(x, xf, wf, p, np.zeros(2), "identity", up)
        d_aux = np.concatenate([(x.T @ up).T.ravel(), np.zeros(2)]).reshape(3, 4)
        assert np.allclose(gr.d_xf, d_aux @ wf.T, atol=1e-12)

    def test_finite_difference(self):
        # central differences on the 3x2 worked layout (pkg/tests/test_grad.py:44-61)
        p = O.Plan(q=3, r_dim=2, rank=1, m=2, n=3)
        xf, wf = O.init_factors(p, 0.7, O.make_rng(3))
        rng = O.make_rng(4)
        x, bias, up = rng.standard_normal((1, 3)), rng.standard_normal(2), rng.standard_normal((1, 2))
        gr = O.layer_backward(x, xf, wf, p, bias, "identity", up)
        eps = 1e-6
        num = np.zeros(xf.size)
        for i in range(xf.size):
            d = np.zeros(xf.size)
            d[i] = eps
            f = lambda xv: float(((x @ O.decompress(xv.reshape(xf.shape), wf, p) + bias) * up).sum())
            num[i] = (f(xf.ravel() + d) - f(xf.ravel() - d)) / (2 * eps)
        assert np.abs(gr.d_xf.ravel() - num).max() / max(np.abs(num).max(), 1e-12) <= 1e-6


def test_bf16_rounding_is_rne():
    vals = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 1e-3])
    got = O.round_bf16(vals)
    assert got[0] == 1.0 and got[1] == 1.0 and got[2] == 1.0 + 2 ** -6
    assert got[3] == -2.5
    assert abs(got[4] - 1e-3) <= 1e-3 * 2 ** -8
    assert math.isclose(O.round_bf16(np.array([3.0]))[0], 3.0)


def test_oracle_lstm_cell_known_answer():
    """oracle.lstm_cell (config 4, unpinned by the reference): gate order i, f, g, o; with all
    pre-activations 0: i = f = o = 1/2, g = 0 -> c' = c/2, h' = tanh(c/2)/2."""
    z = [np.zeros((2, 3))] * 4
    c = np.array([[1.0, -2.0, 0.5], [0.0, 4.0, -1.0]])
    h, cn = O.lstm_cell(z, z, c)
    assert np.allclose(cn, c / 2) and np.allclose(h, np.tanh(c / 2) / 2)
    # saturated gates: i = o = 1, f = 0, g = tanh(large) = 1 -> c' = 1, h' = tanh(1)
    big = [np.full((1, 1), 50.0), np.full((1, 1), -50.0), np.full((1, 1), 50.0), np.full((1, 1), 50.0)]
    h, cn = O.lstm_cell(big, [np.zeros((1, 1))] * 4, np.full((1, 1), 7.0))
    assert np.allclose(cn, 1.0) and np.allclose(h, np.tanh(1.0))


def test_oracle_speech_forward_is_layer_forward_chain():
    """speech_forward with T = 1 and zero initial state equals the explicit chain of
    layer_forward calls (kernel.py:296-320) and one cell step."""
    rng = np.random.default_rng(0)
    def lay(q, r_dim, rank, n):
        m = -(-(q * r_dim) // n)
        p = O.Plan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
        return (rng.normal(0, 0.5, (m, rank)), rng.normal(0, 0.5, (rank, n)), p, rng.normal(0, 0.1, r_dim))
    layers = {"fc1": lay(6, 8, 2, 3), "fc2": lay(8, 8, 1, 4), "fc3": lay(8, 8, 1, 4),
              "fc4": lay(8, 8, 1, 4), "out": lay(8, 5, 1, 4)}
    for g in "ifgo":
        layers[f"x_{g}"] = lay(8, 8, 2, 4)
        layers[f"h_{g}"] = lay(8, 8, 2, 4)
    x = rng.standard_normal((1, 3, 6))
    y = O.speech_forward(x, layers, clip=1.5)
    lf = lambda name, h: O.layer_forward(h, *layers[name])
    h = x[0]
    for name in ("fc1", "fc2", "fc3"):
        h = O.apply_activation("clipped_relu", lf(name, h), 1.5)
    gx = [lf(f"x_{g}", h) for g in "ifgo"]
    gh = [lf(f"h_{g}", np.zeros((3, 8))) for g in "ifgo"]
    hs, _ = O.lstm_cell(gx, gh, np.zeros((3, 8)))
    want = lf("out", O.apply_activation("clipped_relu", lf("fc4", hs), 1.5))
    assert np.allclose(y[0], want, rtol=0, atol=1e-12)
