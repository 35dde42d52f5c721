"""GPU ``bench`` command mirroring the reference CLI's (cli.py:137-189).

    python -m paper_1802_06944_b200 bench [--q 4096] [--r 4096] [--ratio R ...] [--batch 1]
                                          [--rank 1] [--repeat 5] [--seed 0] [--prefer coprime]

Same CSV columns as the reference; the timings are CUDA-event medians on the device:
dense_ms (x @ W with W materialised, bf16 cuBLAS), dense_endtoend_ms (W decompressed on the GPU
then the same GEMM), fused_ms (layer_forward on the bf16 tensor-core path, W never
materialised). ``threads`` reports "gpu". multiplies/reuse_hits are the reference's
OpCount / ReuseTable accounting (kernel.py:184-205, 277-283).
"""

from __future__ import annotations

import argparse
import csv
import statistics
import sys

import numpy as np
import torch

import ctypes as C

from . import _lib
from .core import make_rng, stream_handle
from .errors import InfeasiblePlanError
from .factor import init_factors
from .kernel import ReuseTable, fused_matmul, layer_forward
from .planner import plan_layer

BENCH_RATIOS = (0.08, 0.04, 0.0195, 0.0129, 0.0099, 0.0057, 0.0040, 0.0027, 0.0020, 0.0014)
HEADER = ["q", "r", "ratio", "batch", "threads", "dense_ms", "dense_endtoend_ms", "fused_ms",
          "speedup", "multiplies_dense", "multiplies_fused", "reuse_hits"]


def _timed(fn, repeat):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(repeat):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return statistics.median(out)


def _dense_w(fp):
    """W (q x r_dim) decompressed on the GPU (dt_decompress, factor.py:87-93), bf16."""
    p = fp.plan
    w = torch.empty((p.q, p.r_dim), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().dt_decompress(C.byref(_lib.plan_struct(p)), fp.xf.data_ptr(),
                                        fp.wf.data_ptr(), w.data_ptr(), stream_handle()))
    return w.to(torch.bfloat16)


def bench_one(q, r_dim, ratio, batch, repeat, rank, rng, prefer="coprime"):
    plan = plan_layer(q, r_dim, rank, ratio, prefer=prefer)
    fp = init_factors(plan, 0.05, rng)
    x = torch.tensor(rng.standard_normal((batch, q)), dtype=torch.float32, device="cuda").to(torch.bfloat16)
    zero = np.zeros(r_dim)
    w = _dense_w(fp)
    dense_ms = _timed(lambda: x @ w, repeat)
    e2e_ms = _timed(lambda: x @ _dense_w(fp), repeat)
    fused_ms = _timed(lambda: layer_forward(x, fp, zero, mma="bf16"), repeat)
    table = ReuseTable()
    _, ops = fused_matmul(x, fp, reuse=table, mma="bf16")
    return [q, r_dim, f"{plan.achieved_ratio:.6f}", batch, "gpu", f"{dense_ms:.3f}",
            f"{e2e_ms:.3f}", f"{fused_ms:.3f}", f"{dense_ms / fused_ms:.2f}", q * r_dim * batch,
            ops.multiplies, table.hits]


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_1802_06944_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="median-of-repeat timing: fused kernel vs dense (CSV)")
    b.add_argument("--q", type=int, default=4096)
    b.add_argument("--r", dest="r_dim", type=int, default=4096)
    b.add_argument("--ratio", dest="ratios", type=float, action="append")
    b.add_argument("--batch", type=int, default=1)
    b.add_argument("--repeat", type=int, default=5)
    b.add_argument("--rank", type=int, default=1)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--prefer", choices=["coprime", "reuse"], default="coprime")
    a = ap.parse_args(argv)
    writer = csv.writer(sys.stdout)
    writer.writerow(HEADER)
    rng = make_rng(a.seed)
    for ratio in a.ratios or BENCH_RATIOS:
        try:
            row = bench_one(a.q, a.r_dim, ratio, a.batch, a.repeat, a.rank, rng, a.prefer)
        except InfeasiblePlanError as exc:
            print(f"# ratio {ratio} infeasible: {exc}", file=sys.stderr)
            continue
        writer.writerow(row)
        sys.stdout.flush()
    return 0


if __name__ == "__main__":
    sys.exit(main())
