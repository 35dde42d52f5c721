"""LayerPlan — the geometry of one compressed matrix (reference planner.py:27-60).

Validation runs through the C ABI (dt_plan_validate) so the Python host and the
kernels agree on one definition. Planning algorithms (plan_layer, plan_network)
are out of scope: BASELINE fixes the geometries.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

from . import _lib


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
