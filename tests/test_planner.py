"""plan_layer / feasible_n_range / lower_bound_ratio against the reference planner's own outputs
(tests/golden/planner.npz from tests/golden/make_golden_planner.py, planner.py:92-216), and the
B200 reuse-preferring option."""

import os

import numpy as np
import pytest

import paper_1802_06944_b200 as D

GOLD = os.path.join(os.path.dirname(__file__), "golden", "planner.npz")


@pytest.fixture(scope="module")
def rows():
    return np.load(GOLD)["rows"]


def test_feasible_range_and_plan_match_reference(rows):
    for q, r_dim, rank, alpha, lo, hi, m, n, floor in rows:
        q, r_dim, rank = int(q), int(r_dim), int(rank)
        rng = D.feasible_n_range(q, r_dim, rank, float(alpha))
        assert (rng or (-1, -1)) == (int(lo), int(hi)), (q, r_dim, rank, alpha)
        if n < 0:
            with pytest.raises(D.InfeasiblePlanError):
                D.plan_layer(q, r_dim, rank, float(alpha))
        else:
            p = D.plan_layer(q, r_dim, rank, float(alpha))
            assert (p.m, p.n) == (int(m), int(n)), (q, r_dim, rank, alpha)
        assert D.lower_bound_ratio(q, r_dim, rank) == pytest.approx(floor, rel=0, abs=0)


def test_reuse_preference_picks_row_tile_geometry():
    # config 3's hidden layer at ~1 %: the reference picks a coprime n (general path); the
    # B200 option picks n = 256 | 2048 with (2048/256) * 4 = 32 -> the row-tile kernel
    ref = D.plan_layer(2048, 2048, 3, 0.0125)
    assert ref.q % ref.n != 0
    p = D.plan_layer(2048, 2048, 3, 0.0125, prefer="reuse")
    assert p.q % p.n == 0 and p.n % 64 == 0 and (p.q // p.n) * 4 <= 32
    assert (p.m, p.n) == (16384, 256)          # BASELINE config 3's hidden-layer geometry
    assert p.achieved_ratio <= 0.0125
    # no feasible divisor of q: falls back to the reference choice
    assert D.plan_layer(13, 17, 1, 0.5, prefer="reuse") == D.plan_layer(13, 17, 1, 0.5)
    with pytest.raises(D.ArgumentError):
        D.plan_layer(64, 64, 1, 0.5, prefer="fast")
    with pytest.raises(D.ArgumentError):
        D.feasible_n_range(64, 64, 1, 0.0)
