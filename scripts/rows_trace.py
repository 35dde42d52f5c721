"""One traced launch of the row-tile reuse kernel (timing build, DEEPTHIN_ROWS_TRACE=1): every
CTA's globaltimer stamps, summarised per tile round (median / max over CTAs, µs from the first
CTA's start). Slots (k_tc_rows.cu rtrace): 0 set-up done, 1 after griddepcontrol.wait, per tile
round i: 2+5i phase A start (first x block landed), 3+5i last x block landed, 4+5i phase B start
(every cluster CTA's P landed), 5+5i first D chunk ready for the epilogue, 6+5i epilogue done;
60 the CTA's epilogue finished.

    DEEPTHIN_LIB=paper_1802_06944_b200/_lib/libdeepthin_b200_timing.so python scripts/rows_trace.py
"""
import os
import sys

os.environ["DEEPTHIN_ROWS_TRACE"] = "1"
out = os.environ.setdefault("DEEPTHIN_ROWS_TRACE_FILE", "gpurun_out/rows_trace.bin")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1802_06944_b200 as D  # noqa: E402


def main():
    B = int(os.environ.get("B", 16384))
    q = int(os.environ.get("Q", 2048))
    r_dim = int(os.environ.get("R", 2048))
    plan = D.LayerPlan(q=q, r_dim=r_dim, rank=3, m=q * r_dim // 256, n=256)
    rng = np.random.default_rng(0)
    fp = D.FactorPair(rng.normal(0, .5, (plan.m, 3)).astype(np.float32),
                      rng.normal(0, .5, (3, 256)).astype(np.float32), plan)
    x = torch.randn(B, q, device="cuda").to(torch.bfloat16)
    b = torch.zeros(r_dim, device="cuda")
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    for _ in range(3):
        D.layer_forward(x, fp, b, os.environ.get("ACT", "sigmoid"), mma="bf16",
                        out_dtype=torch.float32 if os.environ.get("OUT") == "f32" else torch.bfloat16)
    torch.cuda.synchronize()
    summarise(out)


def summarise_slab(us, nb, slab, n_chunks, s):
    """Slab kernel (k_tc_slab.cu strace): 0 set-up, 1 after griddepcontrol.wait, 2 first x block
    landed; per group g: 3+8g last phase-A unit issued, 4+8g phase B start (A2 complete), 5+8g
    first D chunk ready, 6+8g the group's stores issued; 62 the CTA's stores complete."""
    print(f"slab kernel: grid {nb} CTAs, {slab} rows per CTA, {n_chunks} chunks, s {s}")

    def col(k):
        v = us[:, k]
        v = v[~np.isnan(v)]
        return f"{np.median(v):7.2f} / {v.min():7.2f} .. {v.max():7.2f} (n={v.size:3d})" if v.size else "      -"
    print(f"  setup done         {col(0)}")
    print(f"  griddep_wait done  {col(1)}")
    print(f"  first x landed     {col(2)}")
    for g in range(7):
        if np.all(np.isnan(us[:, 3 + 8 * g])):
            break
        for k, nm in enumerate(["A issued", "B start", "epi start", "epi issued"]):
            print(f"  group {g} {nm:10s} {col(3 + 8 * g + k)}")
    print(f"  CTA end            {col(62)}")


def summarise(path):
    raw = open(path, "rb").read()
    nb, ktr, cs, n_tiles, n_chunks, s = np.frombuffer(raw[:24], dtype=np.int32)
    h = np.frombuffer(raw[24:], dtype=np.uint64).reshape(nb, ktr).astype(np.float64)
    t0 = h[:, 0][h[:, 0] > 0].min()
    us = np.where(h > 0, (h - t0) * 1e-3, np.nan)
    if cs == 1 and np.any(~np.isnan(us[:, 62])):
        for g in range(2):  # clock64 around the phase-B loop of group g (slots 56+g / 58+g)
            d = h[:, 58 + g] - h[:, 56 + g]
            d = d[h[:, 58 + g] > 0]
            if d.size:
                print(f"  phase-B loop of group {g}: median {np.median(d):.0f} SM clocks")
        return summarise_slab(us, nb, n_tiles, n_chunks, s)
    print(f"grid {nb} CTAs (clusters of {cs}), {n_tiles} tiles, {n_chunks} chunks, s {s}")

    def col(k):
        v = us[:, k]
        v = v[~np.isnan(v)]
        return f"{np.median(v):7.2f} / {v.max():7.2f} (n={v.size:3d})" if v.size else "      -"
    print(f"  setup done         {col(0)}")
    print(f"  griddep_wait done  {col(1)}")
    names = ["A start", "x landed", "B start", "epi start", "epi done"]
    for i in range(10):
        if np.all(np.isnan(us[:, 2 + 5 * i])):
            break
        for k, nm in enumerate(names):
            print(f"  tile {i} {nm:10s} {col(2 + 5 * i + k)}")
    print(f"  CTA end            {col(60)}")
    end = us[:, 60]
    print("  CTA end spread: min %.2f  p10 %.2f  p50 %.2f  p90 %.2f  max %.2f" %
          tuple(np.nanpercentile(end, [0, 10, 50, 90, 100])))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        summarise(sys.argv[1])
    else:
        main()
