"""Golden plan_layer / feasible_n_range outputs from the reference planner (planner.py:92-216).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_planner.py

Writes tests/golden/planner.npz: for a sweep of (q, r_dim, rank, alpha) the reference's
feasible interval, chosen (m, n) — or -1 where the reference raises InfeasiblePlanError — and
its lower-bound ratio.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("DEEPTHIN_REF_SRC", "/root/reference/pkg/src"))
from deepthin.errors import InfeasiblePlanError  # noqa: E402
from deepthin.planner import feasible_n_range, lower_bound_ratio, plan_layer  # noqa: E402

SHAPES = [(1024, 1024), (440, 2048), (2048, 2048), (2048, 3000), (494, 2048), (2048, 29),
          (8192, 8192), (96, 130), (13, 17), (4096, 4096), (784, 300)]
RANKS = [1, 3, 16, 32, 64]
ALPHAS = [0.08, 0.04, 0.0195, 0.0129, 0.0099, 0.0057, 0.004, 0.002, 0.5, 1.0]


def main():
    rows = []
    for q, r_dim in SHAPES:
        for rank in RANKS:
            for alpha in ALPHAS:
                rng = feasible_n_range(q, r_dim, rank, alpha)
                try:
                    p = plan_layer(q, r_dim, rank, alpha)
                    m, n = p.m, p.n
                except InfeasiblePlanError:
                    m = n = -1
                lo, hi = rng if rng is not None else (-1, -1)
                rows.append((q, r_dim, rank, alpha, lo, hi, m, n, lower_bound_ratio(q, r_dim, rank)))
    a = np.array(rows, dtype=np.float64)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "planner.npz")
    np.savez_compressed(out, rows=a)
    print(f"wrote {out}: {len(rows)} cases")


if __name__ == "__main__":
    main()
