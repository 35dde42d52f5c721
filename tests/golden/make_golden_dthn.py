"""Generate ``.dthn`` model-format golden fixtures by importing the reference ``deepthin``.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dthn.py

Writes ``tests/golden/dthn.npz``: the reference's serialized bytes for a small 3-layer network
in float32 and in float64 (with metadata and a floor-hit layer), the factor / bias values they
carry, the reference's expected_file_size, and the reference's parse errors (message + failing
byte offset) on corrupted variants (bad magic, bad version, payload mismatch, truncations,
unknown dtype code, invalid plan, trailing bytes). ``tests/test_model_io.py`` checks the
package's model_io against them.
"""

from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

REF = os.environ.get("DEEPTHIN_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from deepthin.core import make_rng  # noqa: E402
from deepthin.errors import ModelFormatError  # noqa: E402
from deepthin.factor import FactorPair  # noqa: E402
from deepthin.model_io import CompressedModel, deserialize, expected_file_size, serialize  # noqa: E402
from deepthin.factor import init_factors  # noqa: E402
from deepthin.planner import LayerPlan, NetworkPlan, plan_network  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dthn.npz")


def network(dtype):
    specs = [("fc0", 12, 40, 2, 7), ("fc1", 40, 40, 3, 8), ("out", 40, 9, 1, 5)]
    rng = make_rng(42)
    layers, factors, biases = [], [], []
    for name, q, r_dim, rank, n in specs:
        m = -(-(q * r_dim) // n)
        plan = LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
        xf = rng.standard_normal((m, rank)).astype(dtype)
        wf = rng.standard_normal((rank, n)).astype(dtype)
        layers.append((name, plan))
        factors.append(FactorPair(xf=xf, wf=wf, plan=plan))
        biases.append(rng.standard_normal(r_dim).astype(dtype))
    plans = NetworkPlan(layers=tuple(layers), target_ratio=0.25, achieved_total_ratio=0.0,
                        floor_hits=("fc1",), bias_counts=tuple(b.size for b in biases))
    return CompressedModel(plans=plans, factors=factors, biases=biases,
                           metadata={"source": "golden", "units": "frames"})


def planned_model(seed: int, dtype):
    """A network planned by the reference planner (random shapes, ratio, 1-4 layers)."""
    rng = np.random.default_rng(1000 + seed)
    count = 1 + seed % 4
    shapes = [(f"L{seed}_{i}", int(rng.integers(4, 48)), int(rng.integers(4, 48)))
              for i in range(count)]
    net = plan_network(shapes, 1 + seed % 2, float(rng.uniform(0.6, 0.95)),
                       bias_counts=[r for _, _, r in shapes])
    gen = make_rng(seed)
    factors = []
    for _, plan in net.layers:
        fp = init_factors(plan, 0.1, gen)
        if dtype == np.float32:
            fp = fp.with_values(np.asarray(fp.xf, np.float32), np.asarray(fp.wf, np.float32))
        factors.append(fp)
    biases = [gen.standard_normal(plan.r_dim).astype(dtype) for _, plan in net.layers]
    return CompressedModel(plans=net, factors=factors, biases=biases,
                           metadata={"seed": str(seed), "\u00e9t\u00e9": "\u2713"})


def with_payload(data: bytes) -> bytes:
    """Rewrite the declared payload so parsing reaches the damage."""
    return data[:12] + struct.pack("<Q", len(data) - 28) + data[20:]


def corruptions(data: bytes):
    out = {}
    out["bad_magic"] = b"XTHN" + data[4:]
    out["bad_version"] = data[:4] + struct.pack("<I", 7) + data[8:]
    out["payload_mismatch"] = data[:12] + struct.pack("<Q", len(data)) + data[20:]
    out["truncated_header"] = data[:20]
    # a shortened file with a consistent payload count: truncation inside a layer
    cut = data[: len(data) - 50]
    out["truncated_layer"] = cut[:12] + struct.pack("<Q", len(cut) - 28) + cut[20:]
    # trailing bytes with a consistent payload count
    ext = data + b"\x00\x01\x02"
    out["trailing"] = ext[:12] + struct.pack("<Q", len(ext) - 28) + ext[20:]
    # unknown dtype code in the first layer: header 28 + meta (4 + 2 items) + name
    meta_len = 4 + (4 + 6 + 4 + 6) + (4 + 5 + 4 + 6)
    code_at = 28 + meta_len + 4 + 3 + 40
    out["bad_dtype"] = data[:code_at] + b"\x09" + data[code_at + 1:]
    # invalid plan (m*n too small): overwrite fc0's m with 1
    m_at = 28 + meta_len + 4 + 3 + 24
    out["bad_plan"] = data[:m_at] + struct.pack("<Q", 1) + data[m_at + 8:]
    return out


def main():
    g = {}
    errors = {}
    for tag, dtype in (("f32", np.float32), ("f64", np.float64)):
        model = network(dtype)
        data = serialize(model)
        g[f"{tag}_bytes"] = np.frombuffer(data, dtype=np.uint8)
        g[f"{tag}_size"] = np.array([expected_file_size(model)], dtype=np.int64)
        back = deserialize(data)
        for i, (fp, b) in enumerate(zip(back.factors, back.biases)):
            g[f"{tag}_xf{i}"] = fp.xf
            g[f"{tag}_wf{i}"] = fp.wf
            g[f"{tag}_b{i}"] = b
        g[f"{tag}_ratio"] = np.array([back.plans.achieved_total_ratio])
        if tag == "f32":
            for name, bad in corruptions(data).items():
                g[f"bad_{name}"] = np.frombuffer(bad, dtype=np.uint8)
                try:
                    deserialize(bad)
                    errors[name] = None
                except ModelFormatError as exc:
                    errors[name] = {"offset": exc.offset, "message": str(exc)}
            # truncation at every byte of the header / metadata / first layer's fixed fields,
            # then a stride through the payloads
            cuts = list(range(0, 200)) + list(range(200, len(data), 37))
            for cut in cuts:
                bad = with_payload(data[:cut]) if cut >= 28 else data[:cut]
                try:
                    deserialize(bad)
                    errors[f"cut{cut}"] = None
                except ModelFormatError as exc:
                    errors[f"cut{cut}"] = {"offset": exc.offset, "message": str(exc)}
            g["cuts"] = np.array(cuts, dtype=np.int64)
    planned = []
    for seed in range(40):
        model = planned_model(seed, np.float32 if seed % 3 == 0 else np.float64)
        data = serialize(model)
        back = deserialize(data)
        g[f"planned{seed}"] = np.frombuffer(data, dtype=np.uint8)
        planned.append({"size": expected_file_size(model),
                        "layers": [[n, p.q, p.r_dim, p.rank, p.m, p.n] for n, p in back.plans.layers],
                        "floor_hits": list(back.plans.floor_hits),
                        "ratio": back.plans.achieved_total_ratio,
                        "target": back.plans.target_ratio,
                        "metadata": back.metadata})
    g["planned_json"] = np.frombuffer(json.dumps(planned).encode(), dtype=np.uint8)
    g["errors_json"] = np.frombuffer(json.dumps(errors).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays; errors {json.dumps(errors)[:400]}")


if __name__ == "__main__":
    main()
