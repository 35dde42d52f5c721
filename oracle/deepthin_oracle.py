"""CPU oracle for the DeepThin compressed-layer hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``deepthin``
(``/root/reference/pkg/src/deepthin``) for the functions on the hot path
(SURVEY.md §8(a) rows a1-a14). It exists to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
  ``--impl reference`` leg may import it;
* the product package ``paper_1802_06944_b200`` never imports it and has no CPU
  fallback.

Parity status: PINNED. ``tests/test_oracle_golden.py`` checks every function
here against golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``) and against the
reference test-suite's known answers (``pkg/tests/test_factor.py:47-52``,
``:141-144``, ``test_kernel.py:250-262`` …).

Notation is the reference's: a layer maps ``q`` inputs to
``r_dim`` outputs; its weight ``W`` (q × r_dim) is the column-major refill of
``v = (xf @ wf).ravel()`` with ``xf`` m × rank and ``wf`` rank × n.

Activations the reference does not define (``clipped_relu``, ``softmax``; used
by BASELINE configs 3/4) are stated here and are *unpinned* by the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FLOAT32 = np.float32
FLOAT64 = np.float64
_ALLOWED = (np.dtype(np.float32), np.dtype(np.float64))


class OracleError(ValueError):
    """Base of the oracle's error classes (mirrors deepthin/errors.py:6-43)."""


class DimensionError(OracleError):
    pass


class ArgumentError(OracleError):
    pass


class UnsupportedConfigurationError(OracleError):
    pass


# --------------------------------------------------------------------------
# core.py
# --------------------------------------------------------------------------

def as_matrix(a, *, dtype=None, name="matrix"):
    """Validation gate — restates core.py:21-36 (2-D, C-contiguous, f32/f64, finite)."""
    arr = np.asarray(a)
    if arr.ndim != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {arr.shape}")
    if dtype is None:
        dtype = arr.dtype if arr.dtype in _ALLOWED else FLOAT64
    arr = np.ascontiguousarray(arr, dtype=dtype)
    if not np.all(np.isfinite(arr)):
        raise ArgumentError(f"{name} contains non-finite entries")
    return arr


def make_rng(seed):
    """core.py:39-41 — SeedSequence → PCG64."""
    return np.random.default_rng(np.random.SeedSequence(seed))


def spawn_rngs(seed, count):
    """core.py:44-51 — independent children of one SeedSequence."""
    return [np.random.default_rng(c) for c in np.random.SeedSequence(seed).spawn(count)]


def sample_normal(rng, mean, stddev, shape):
    """core.py:54-60 — scale-after-draw normal samples."""
    if stddev < 0:
        raise ArgumentError(f"stddev must be >= 0, got {stddev}")
    return rng.standard_normal(shape) * stddev + mean


def matmul(a, b):
    """core.py:63-77 — shape-checked product in the promoted dtype."""
    am = as_matrix(a, name="left operand")
    bm = as_matrix(b, name="right operand")
    if am.shape[1] != bm.shape[0]:
        raise DimensionError(
            f"cannot multiply {am.shape[0]}x{am.shape[1]} by {bm.shape[0]}x{bm.shape[1]}")
    dt = np.result_type(am.dtype, bm.dtype)
    return np.matmul(am.astype(dt, copy=False), bm.astype(dt, copy=False))


def _host(a):
    """Accept device tensors from the code under test (copied to host, widened)."""
    if hasattr(a, "detach"):
        return a.detach().float().cpu().numpy()
    return np.asarray(a)


def max_abs_diff(a, b):
    """core.py:80-88."""
    a = _host(a)
    b = _host(b)
    if a.shape != b.shape:
        return float("inf")
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a.astype(FLOAT64) - b.astype(FLOAT64))))


def rel_error(actual, expected):
    """core.py:91-95 — max|a-e| / max|e| (the parity metric everywhere)."""
    expected = np.asarray(expected, dtype=FLOAT64)
    scale = float(np.max(np.abs(expected))) if expected.size else 0.0
    return max_abs_diff(actual, expected) / (scale if scale > 0 else 1.0)


# --------------------------------------------------------------------------
# planner.py (LayerPlan only) and factor.py
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Plan:
    """Geometry of one compressed matrix — restates planner.py:27-60 (validation only)."""

    q: int
    r_dim: int
    rank: int
    m: int
    n: int

    def __post_init__(self):
        for label in ("q", "r_dim", "rank", "m", "n"):
            if getattr(self, label) < 1:
                raise ArgumentError(f"{label} must be >= 1, got {getattr(self, label)}")
        if self.m * self.n < self.q * self.r_dim:
            raise ArgumentError(
                f"m*n = {self.m * self.n} must cover q*r_dim = {self.q * self.r_dim}")


def check_factors(xf, wf, plan):
    """factor.py:36-41 — the FactorPair shape check."""
    xf = as_matrix(xf, name="xf")
    wf = as_matrix(wf, name="wf")
    if xf.shape != (plan.m, plan.rank):
        raise DimensionError(f"xf must be {plan.m}x{plan.rank}, got {xf.shape}")
    if wf.shape != (plan.rank, plan.n):
        raise DimensionError(f"wf must be {plan.rank}x{plan.n}, got {wf.shape}")
    return xf, wf


def init_factors(plan, sigma, rng):
    """factor.py:60-71 — xf ~ N(0, sigma²), wf ~ N(0, 1/rank)."""
    if not sigma > 0:
        raise ArgumentError(f"sigma must be > 0, got {sigma}")
    xf = sample_normal(rng, 0.0, sigma, (plan.m, plan.rank))
    wf = sample_normal(rng, 0.0, 1.0 / math.sqrt(plan.rank), (plan.rank, plan.n))
    return xf, wf


def relayout_index(flat, plan):
    """factor.py:74-84 — v[flat] lands at W[flat % q, flat // q]."""
    if not 0 <= flat < plan.q * plan.r_dim:
        raise ArgumentError(f"flat index {flat} out of range for {plan.q}x{plan.r_dim}")
    return flat % plan.q, flat // plan.q


def decompress(xf, wf, plan):
    """factor.py:87-93 — dense q × r_dim W; the m·n − q·r_dim tail is discarded."""
    v = np.matmul(xf, wf).ravel()
    qr = plan.q * plan.r_dim
    return np.ascontiguousarray(v[:qr].reshape(plan.r_dim, plan.q).T)


def scatter_decompress(xf, wf, plan):
    """Element-wise restatement of the same law (pkg/tests/oracles.py:79-86 style)."""
    v = np.matmul(xf, wf).ravel()
    out = np.zeros((plan.q, plan.r_dim), dtype=v.dtype)
    k = np.arange(plan.q * plan.r_dim)
    out[k % plan.q, k // plan.q] = v[k]
    return out


def phase(col, plan):
    """factor.py:96-105 — wf offset at which output column ``col`` starts."""
    if not 0 <= col < plan.r_dim:
        raise ArgumentError(f"col {col} out of range for r_dim {plan.r_dim}")
    return (col * plan.q) % plan.n


def phase_count(plan):
    """factor.py:108-110 — n / gcd(n, q), capped by r_dim."""
    return min(plan.n // math.gcd(plan.n, plan.q), plan.r_dim)


def is_reuse_path(plan):
    """Path (a) of BASELINE.json: n | q ⇔ one phase."""
    return plan.q % plan.n == 0


# --------------------------------------------------------------------------
# kernel.py
# --------------------------------------------------------------------------

ACTIVATIONS = ("identity", "relu", "sigmoid", "tanh")
EXTRA_ACTIVATIONS = ("clipped_relu", "softmax")   # not in the reference: unpinned


def apply_activation(name, z, arg=20.0):
    """kernel.py:39-48 (+ clipped_relu / row softmax, unpinned)."""
    if name == "identity":
        return z
    if name == "relu":
        return np.maximum(z, 0.0)
    if name == "sigmoid":
        return 1.0 / (1.0 + np.exp(-z))
    if name == "tanh":
        return np.tanh(z)
    if name == "clipped_relu":
        return np.minimum(np.maximum(z, 0.0), arg)
    if name == "softmax":
        e = np.exp(z - z.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)
    raise ArgumentError(f"unknown activation {name!r}")


def activation_grad(name, z, arg=20.0):
    """kernel.py:51-62 (relu'(0) = 0); clipped_relu'(z) = 1 on (0, arg)."""
    if name == "identity":
        return np.ones_like(z)
    if name == "relu":
        return (z > 0).astype(z.dtype)
    if name == "sigmoid":
        s = 1.0 / (1.0 + np.exp(-z))
        return s * (1.0 - s)
    if name == "tanh":
        return 1.0 - np.tanh(z) ** 2
    if name == "clipped_relu":
        return ((z > 0) & (z < arg)).astype(z.dtype)
    raise ArgumentError(f"unknown activation {name!r}")


@dataclass
class OpCount:
    """kernel.py:65-77."""

    multiplies: int = 0
    adds: int = 0


@dataclass
class ReuseTable:
    """kernel.py:80-96 (counts only; entries recorded on request)."""

    hits: int = 0
    misses: int = 0
    record_entries: bool = False
    entries: dict = field(default_factory=dict)


def runs_of_phase(t, plan):
    """The runs of a column in phase slot ``t`` — restates _Layout (kernel.py:107-121).

    Returns (wf_offset, input_start, length, aux_row_in_period) arrays for the
    column ``t`` (columns t, t+period, … repeat it shifted by q/gcd aux rows).
    """
    q, n = plan.q, plan.n
    p = (t * q) % n
    if n - p < q:
        starts = np.concatenate(([0], np.arange(n - p, q, n)))
    else:
        starts = np.zeros(1, dtype=np.int64)
    offs = np.zeros_like(starts)
    offs[0] = p
    lens = np.minimum(n - offs, q - starts)
    rows = (t * q + starts) // n
    return offs.astype(np.int64), starts.astype(np.int64), lens.astype(np.int64), rows


def predict_reuse(plan, batch=1):
    """kernel.py:184-205 — (distinct_runs, total_runs) per input row."""
    if batch < 1:
        raise ArgumentError(f"batch must be >= 1, got {batch}")
    q, r, n = plan.q, plan.r_dim, plan.n
    period = n // math.gcd(n, q)
    distinct = total = 0
    for t in range(min(period, r)):
        p = (t * q) % n
        runs = 1 + (p + q - 1) // n
        cols = (r - t + period - 1) // period
        distinct += runs
        total += runs * cols
    return distinct, total


def op_count(plan, batch):
    """OpCount of the run-memoized algorithm — kernel.py:277-280."""
    period = plan.n // math.gcd(plan.n, plan.q)
    n_ph = min(period, plan.r_dim)
    sum_len = 0
    for t in range(n_ph):
        sum_len += int(runs_of_phase(t, plan)[2].sum())
    distinct, total = predict_reuse(plan)
    return OpCount(
        multiplies=batch * (sum_len + total),
        adds=batch * (sum_len - distinct) + batch * (total - plan.r_dim))


def fused_matmul(x, xf, wf, plan, reuse=None):
    """Y = X @ decompress without materializing W — kernel.py:222-293.

    The reference restricts this to rank 1 (kernel.py:238-240); the same
    sliding-correlation + gather/combine algorithm extends to rank r by
    superposition over rank components, which is what this
    restatement does. float64 accumulation; f32 output iff every input is f32.
    """
    xm = as_matrix(x, name="input")
    xf, wf = check_factors(xf, wf, plan)
    if xm.shape[1] != plan.q:
        raise DimensionError(
            f"cannot multiply {xm.shape[0]}x{xm.shape[1]} by compressed {plan.q}x{plan.r_dim}")
    q, r, n = plan.q, plan.r_dim, plan.n
    batch = xm.shape[0]
    out32 = xm.dtype == FLOAT32 and xf.dtype == FLOAT32 and wf.dtype == FLOAT32
    x64 = xm.astype(FLOAT64)
    g = math.gcd(n, q)
    period = n // g
    step = q // g
    y = np.zeros((batch, r), dtype=FLOAT64)
    for k in range(plan.rank):
        wk = wf[k].astype(FLOAT64)
        # dots[b, (n-1) + start - off] == x[b, start:start+L] . wk[off:off+L]
        dots = np.stack([np.correlate(x64[b], wk, mode="full") for b in range(batch)]) \
            if batch else np.zeros((0, q + n - 1))
        xk = xf[:, k].astype(FLOAT64)
        for t in range(min(period, r)):
            offs, starts, _, rows = runs_of_phase(t, plan)
            lags = (n - 1) + starts - offs
            cols = np.arange(t, r, period)
            xr = rows[None, :] + (np.arange(cols.size) * step)[:, None]   # cols × runs
            y[:, cols] += np.einsum("bk,jk->bj", dots[:, lags], xk[xr])
    if reuse is not None:
        distinct, total = predict_reuse(plan)
        reuse.misses += distinct * batch
        reuse.hits += total * batch - distinct * batch
    ops = op_count(plan, batch)
    return (y.astype(FLOAT32) if out32 else y), ops


def layer_forward(x, xf, wf, plan, bias, activation="identity", act_arg=20.0):
    """kernel.py:296-320 — activation(x @ W + bias), f64 output (bias promotion).

    Rank 1 goes through ``fused_matmul``; rank > 1 through decompress + matmul,
    exactly the routes the reference takes.
    """
    bias = np.asarray(bias, dtype=FLOAT64).ravel()
    if bias.shape[0] != plan.r_dim:
        raise DimensionError(f"bias length {bias.shape[0]} != output width {plan.r_dim}")
    if plan.rank == 1:
        z, _ = fused_matmul(x, xf, wf, plan)
    else:
        xf, wf = check_factors(xf, wf, plan)
        z = matmul(x, decompress(xf, wf, plan))
    return apply_activation(activation, z + bias, act_arg)


# --------------------------------------------------------------------------
# grad.py
# --------------------------------------------------------------------------

@dataclass
class Gradients:
    """grad.py:23-28."""

    d_xf: np.ndarray
    d_wf: np.ndarray
    d_input: np.ndarray
    d_bias: np.ndarray


def layer_backward(x, xf, wf, plan, bias, activation, upstream, act_arg=20.0):
    """grad.py:63-95 — float64 gradients through the inverse re-layout."""
    xm = as_matrix(x, dtype=FLOAT64, name="input")
    up = as_matrix(upstream, dtype=FLOAT64, name="upstream")
    xf, wf = check_factors(xf, wf, plan)
    if xm.shape[1] != plan.q:
        raise DimensionError(f"input width {xm.shape[1]} != layer input width {plan.q}")
    if up.shape != (xm.shape[0], plan.r_dim):
        raise DimensionError(f"upstream shape {up.shape} != layer output shape "
                             f"{(xm.shape[0], plan.r_dim)}")
    w = decompress(xf.astype(FLOAT64), wf.astype(FLOAT64), plan)
    pre = xm @ w + np.asarray(bias, dtype=FLOAT64).ravel()
    g = up * activation_grad(activation, pre, act_arg)
    d_bias = g.sum(axis=0)
    d_w = xm.T @ g
    d_v = np.zeros(plan.m * plan.n, dtype=FLOAT64)
    d_v[: plan.q * plan.r_dim] = d_w.T.ravel()   # gather; discarded tail gets 0
    d_aux = d_v.reshape(plan.m, plan.n)
    return Gradients(
        d_xf=d_aux @ wf.T.astype(FLOAT64),
        d_wf=xf.T.astype(FLOAT64) @ d_aux,
        d_input=g @ w.T,
        d_bias=d_bias)


def loss_and_grad(name, y, target):
    """grad.py:98-116 — mse (2·diff / y.size) and softmax cross-entropy."""
    if name == "mse":
        diff = y - np.asarray(target, dtype=FLOAT64)
        return float(np.mean(diff ** 2)), 2.0 * diff / y.size
    if name == "softmax_cross_entropy":
        labels = np.asarray(target)
        z = y - y.max(axis=1, keepdims=True)
        e = np.exp(z)
        probs = e / e.sum(axis=1, keepdims=True)
        batch = y.shape[0]
        picked = np.maximum(probs[np.arange(batch), labels], 1e-300)
        grad = probs.copy()
        grad[np.arange(batch), labels] -= 1.0
        return float(-np.mean(np.log(picked))), grad / batch
    raise ArgumentError(f"unknown loss {name!r}")


def sgd_step(xf, wf, bias, grads, lr):
    """train.py:107-111 and :221 — plain SGD on factors and bias."""
    return (xf - lr * grads.d_xf, wf - lr * grads.d_wf, bias - lr * grads.d_bias)


# --------------------------------------------------------------------------
# BASELINE.json inputs
# --------------------------------------------------------------------------

def baseline_inputs(plan, batch, seed=0, bias_sd=0.01):
    """spawn_rngs(seed, 5) children in the order [xf, wf, bias, x, target].

    Factors ~ N(0, stddev 1/sqrt(rank)) (BASELINE's "N(0, 1/sqrt(r))"), bias
    ~ N(0, 0.01), x and target ~ N(0, 1); all float64.
    """
    rx, rw, rb, ri, rt = spawn_rngs(seed, 5)
    sd = 1.0 / math.sqrt(plan.rank)
    return dict(
        xf=sample_normal(rx, 0.0, sd, (plan.m, plan.rank)),
        wf=sample_normal(rw, 0.0, sd, (plan.rank, plan.n)),
        bias=sample_normal(rb, 0.0, bias_sd, (plan.r_dim,)),
        x=sample_normal(ri, 0.0, 1.0, (batch, plan.q)),
        target=sample_normal(rt, 0.0, 1.0, (batch, plan.r_dim)))


def round_bf16(a):
    """Round-to-nearest-even to bfloat16, returned as float64 (what the GPU sees)."""
    a32 = np.ascontiguousarray(a, dtype=np.float32)
    u = a32.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(FLOAT64)


# ---- BASELINE config 4: the speech-RNN-shaped network (UNPINNED by the reference) ----------
# The reference has no LSTM. Every contraction below is the pinned
# layer_forward (kernel.py:296-320); the cell is the standard LSTM cell, gate order i, f, g, o.

def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def lstm_cell(gx, gh, c):
    """One cell step: gx/gh are the 4 input/recurrent gate pre-activations (lists), c the state.
    Returns (h', c')."""
    i, f, g, o = (_sigmoid(gx[0] + gh[0]), _sigmoid(gx[1] + gh[1]), np.tanh(gx[2] + gh[2]),
                  _sigmoid(gx[3] + gh[3]))
    cn = f * c + i * g
    return o * np.tanh(cn), cn


def speech_forward(x, layers, clip=20.0, layer=None, store=None):
    """Config-4 forward in f64. x: (T, B, n_in); layers: name -> (xf, wf, Plan, bias) for
    fc1-3, x_{i,f,g,o}, h_{i,f,g,o}, fc4, out. ``layer(name, h, xf, wf, plan, bias)`` overrides
    the contraction (default: layer_forward); ``store(a)`` rounds every activation the device
    stores between layers (default: identity). The recurrence itself stays unrounded."""
    layer = layer or (lambda name, h, xf, wf, plan, b: layer_forward(h, xf, wf, plan, b))
    store = store or (lambda a: a)
    T, B, n_in = x.shape
    h = x.reshape(T * B, n_in).astype(np.float64)

    def run(name, h):
        xf, wf, plan, b = layers[name]
        return layer(name, h, xf, wf, plan, b)

    for name in ("fc1", "fc2", "fc3"):
        h = store(apply_activation("clipped_relu", run(name, h), clip))
    gx = [store(run(f"x_{g}", h)) for g in "ifgo"]
    H = layers["h_i"][2].q
    hp = np.zeros((B, H))
    c = np.zeros((B, H))
    seq = np.zeros((T * B, H))
    for t in range(T):
        gh = [run(f"h_{g}", hp) for g in "ifgo"]
        hp, c = lstm_cell([a[t * B:(t + 1) * B] for a in gx], gh, c)
        seq[t * B:(t + 1) * B] = store(hp)
    h = store(apply_activation("clipped_relu", run("fc4", seq), clip))
    return run("out", h).reshape(T, B, -1)
