"""LayerPlan — the geometry of one compressed matrix (reference planner.py:27-60).

Validation runs through the C ABI (dt_plan_validate) so the Python host and the
kernels agree on one definition. ``plan_layer`` restates the reference's single-matrix
planner (planner.py:92-216: the feasible column-count interval of the ratio constraint, the
smallest n coprime with q, else the largest LCM) and adds the B200 option of SURVEY.md
§8(f)-4: ``prefer="reuse"`` picks a feasible n that divides q, so the layer runs on the
factored reuse path (the row-tile kernel when n % 64 == 0 and s * round_up(rank, 4) <= 32),
trading the LCM-maximising layout for speed. Network planning
(plan_network) stays out of scope.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

from fractions import Fraction

from . import _lib
from .errors import ArgumentError, InfeasiblePlanError


@dataclass(frozen=True)
class LayerPlan:
    """Chosen compression parameters for one q x r_dim matrix (reference notation)."""

    q: int
    r_dim: int
    rank: int
    m: int
    n: int
    achieved_ratio: float = field(init=False)
    lcm_nq: int = field(init=False)

    def __post_init__(self):
        for label in ("q", "r_dim", "rank", "m", "n"):
            v = getattr(self, label)
            if not isinstance(v, int):
                object.__setattr__(self, label, int(v))
        _lib.check(_lib.lib().dt_plan_validate(C.byref(_lib.plan_struct(self))))
        object.__setattr__(self, "achieved_ratio",
                           self.rank * (self.m + self.n) / (self.q * self.r_dim))
        object.__setattr__(self, "lcm_nq", math.lcm(self.n, self.q))

    @property
    def original_elems(self) -> int:
        return self.q * self.r_dim

    @property
    def compressed_elems(self) -> int:
        return self.rank * (self.m + self.n)

    def info(self) -> _lib.PlanInfo:
        """Derived geometry: period, phase_count, reuse flag, segments, tail."""
        out = _lib.PlanInfo()
        _lib.check(_lib.lib().dt_plan_query(C.byref(_lib.plan_struct(self)), C.byref(out)))
        return out

    @property
    def reuse_path(self) -> bool:
        """True iff n | q: the factored-reuse path (a); else the general path (b)."""
        return self.q % self.n == 0


@dataclass(frozen=True)
class NetworkPlan:
    """Per-layer plans of a network (reference planner.py:63-77): ordered (name, LayerPlan)
    pairs, the target and achieved whole-network ratios, the layers that hit their accuracy
    floor, and the dense bias counts the achieved ratio includes."""

    layers: tuple
    target_ratio: float
    achieved_total_ratio: float
    floor_hits: tuple
    bias_counts: tuple = ()

    def plan_for(self, name: str) -> LayerPlan:
        found = [plan for layer_name, plan in self.layers if layer_name == name]
        if not found:
            raise KeyError(name)
        return found[0]


def baseline_plan(in_features: int, out_features: int, rank: int, n_f: int, m_f: int | None = None):
    """Build a plan from BASELINE.json notation (n=in, m=out, n_f, m_f, r)."""
    m = m_f if m_f is not None else -(-(in_features * out_features) // n_f)
    return LayerPlan(q=in_features, r_dim=out_features, rank=rank, m=m, n=n_f)


_COPRIME_SCAN = 100_000  # reference planner.py:24


def _check_args(q, r_dim, rank):
    for label, v in (("q", q), ("r_dim", r_dim), ("rank", rank)):
        if not isinstance(v, int) or isinstance(v, bool) or v < 1:
            raise ArgumentError(f"{label} must be an integer >= 1, got {v!r}")


def _fits(n: int, qr: int, rank: int, a: Fraction) -> bool:
    """rank * (q*r_dim + n^2) <= alpha * q*r_dim * n, exactly (the real-relaxed m = qr/n)."""
    return rank * (qr + n * n) <= a * qr * n


def feasible_n_range(q: int, r_dim: int, rank: int, alpha: float):
    """[n_lo, n_hi] of column counts meeting the ratio, or None (reference planner.py:92-140).
    The constraint is the quadratic rank*n^2 - alpha*qr*n + rank*qr <= 0: its real roots are
    computed in floating point and each end is then moved onto the exact integer boundary."""
    _check_args(q, r_dim, rank)
    if not 0 < alpha <= 1:
        raise ArgumentError(f"alpha must be in (0, 1], got {alpha}")
    a = Fraction(alpha)
    qr = q * r_dim
    b = float(a * qr / rank)
    disc = b * b - 4.0 * qr
    if disc < 0:
        # a tangent or rounding-hidden solution can only sit at the vertex b/2
        mid = max(1, int(round(b / 2)))
        cands = [c for c in range(max(1, mid - 2), mid + 3) if _fits(c, qr, rank, a)]
        return (cands[0], cands[-1]) if cands else None
    root = math.sqrt(disc)
    lo = max(1, int(math.floor((b - root) / 2)) - 2)
    hi = min(qr, int(math.ceil((b + root) / 2)) + 2)
    while lo <= hi and not _fits(lo, qr, rank, a):
        lo += 1
    if lo > hi:
        return None
    while lo > 1 and _fits(lo - 1, qr, rank, a):
        lo -= 1
    while hi >= lo and not _fits(hi, qr, rank, a):
        hi -= 1
    while hi < qr and _fits(hi + 1, qr, rank, a):
        hi += 1
    return lo, hi


def lower_bound_ratio(q: int, r_dim: int, rank: int) -> float:
    """The least achievable ratio rank * min_n(ceil(qr/n) + n) / qr (planner.py:143-176)."""
    _check_args(q, r_dim, rank)
    qr = q * r_dim
    if qr <= 1 << 16:
        ns = range(1, qr + 1)
    else:
        c = math.isqrt(qr)
        w = 3 * math.isqrt(c + 1) + 8
        ns = range(max(1, c - w), min(qr, c + w) + 1)
    return rank * min(-(-qr // n) + n for n in ns) / qr


def _max_lcm(cands, q):
    """Smallest n coprime with q, else the largest LCM(n, q), smallest n on ties
    (planner.py:179-188)."""
    best, best_l = None, -1
    for n in cands:
        if math.gcd(n, q) == 1:
            return n
        l = math.lcm(n, q)
        if l > best_l:
            best, best_l = n, l
    return best


def plan_layer(q: int, r_dim: int, rank: int, alpha: float, prefer: str = "coprime") -> LayerPlan:
    """Plan one q x r_dim matrix at ratio alpha (reference planner.py:191-216).

    prefer="coprime" (the reference): the smallest feasible n coprime with q (maximal LCM(n, q),
    the paper's accuracy argument). prefer="reuse" (B200): the smallest feasible n that divides
    q and takes the row-tile kernel (n % 64 == 0, (q/n) * round_up(rank, 4) <= 32), else the
    smallest feasible divisor of q with n % 8 == 0, else the reference choice — the smallest n
    keeps the most parameters inside the budget (the ratio falls with n below sqrt(q*r_dim)).
    m is the least row count covering the matrix, ceil(q*r_dim / n)."""
    if prefer not in ("coprime", "reuse"):
        raise ArgumentError(f"prefer must be 'coprime' or 'reuse', got {prefer!r}")
    rng = feasible_n_range(q, r_dim, rank, alpha)
    if rng is None:
        bound = lower_bound_ratio(q, r_dim, rank)
        raise InfeasiblePlanError(
            f"ratio {alpha} is below the floor {bound:.6g} for a {q}x{r_dim} matrix", {"": bound})
    n_lo, n_hi = rng
    n = None
    if prefer == "reuse":
        divs = [d for d in range(n_lo, min(n_hi, q) + 1) if q % d == 0]
        rp = -(-rank // 4) * 4
        for ok in (lambda d: d % 64 == 0 and (q // d) * rp <= 32, lambda d: d % 8 == 0):
            hit = [d for d in divs if ok(d)]
            if hit:
                n = hit[0]
                break
    if n is None:
        for cand in range(n_lo, min(n_hi, n_lo + _COPRIME_SCAN) + 1):
            if math.gcd(cand, q) == 1:
                n = cand
                break
    if n is None:
        n = _max_lcm(range(n_lo, n_hi + 1), q)
    return LayerPlan(q=q, r_dim=r_dim, rank=rank, m=-(-(q * r_dim) // n), n=n)
