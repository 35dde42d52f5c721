"""The .dthn model format (reference model_io.py; tests model test_model_io.py and acceptance
criterion 7, test_acceptance.py:322-329). CPU-only: the parser is host code in the native
library (dt_model_parse); no GPU calls.

Pinned against tests/golden/dthn.npz, made by tests/golden/make_golden_dthn.py from the
reference itself: its serialized bytes (float32 / float64, planner-produced networks), the
values it parses out, and its ModelFormatError message + byte offset for corrupted images
(bad magic / version / payload count / dtype code / plan, trailing bytes, and truncation at
every byte of the header, metadata and first layer plus a stride through the payloads).
"""

import json

import numpy as np
import pytest

from paper_1802_06944_b200 import model_io as mi
from paper_1802_06944_b200.errors import ArgumentError, ModelFormatError
from paper_1802_06944_b200.planner import LayerPlan, NetworkPlan


@pytest.fixture(scope="module")
def golden():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "dthn.npz"))


def raw(g, key) -> bytes:
    return g[key].tobytes()


def random_model(seed: int, layers: int | None = None, dtype=np.float64) -> mi.CompressedModel:
    """A random valid network (own geometry sampler; the planner is out of scope)."""
    rng = np.random.default_rng(seed)
    count = layers or int(rng.integers(1, 5))
    entries, factors, biases = [], [], []
    q = int(rng.integers(1, 50))
    for i in range(count):
        r_dim = int(rng.integers(1, 50))
        n = int(rng.integers(1, q * r_dim + 1))
        m = -(-(q * r_dim) // n) + int(rng.integers(0, 2))
        rank = int(rng.integers(1, 4))
        plan = LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
        entries.append((f"layer{i}", plan))
        factors.append(mi.StoredFactors(rng.standard_normal((m, rank)).astype(dtype),
                                        rng.standard_normal((rank, n)).astype(dtype), plan))
        biases.append(rng.standard_normal(r_dim).astype(dtype))
        q = r_dim
    plans = NetworkPlan(layers=tuple(entries), target_ratio=float(rng.uniform(0.1, 0.9)),
                        achieved_total_ratio=0.0,
                        floor_hits=tuple(n for n, _ in entries[:1] if seed % 2),
                        bias_counts=tuple(b.size for b in biases))
    return mi.CompressedModel(plans=plans, factors=factors, biases=biases,
                              metadata={"seed": str(seed), "note": "round trip"})


class TestAgainstReferenceBytes:
    @pytest.mark.parametrize("tag", ["f32", "f64"])
    def test_parse_values_and_reserialize(self, golden, tag):
        data = raw(golden, f"{tag}_bytes")
        model = mi.deserialize(data)
        assert mi.serialize(model) == data
        assert mi.expected_file_size(model) == int(golden[f"{tag}_size"][0]) == len(data)
        assert model.plans.achieved_total_ratio == float(golden[f"{tag}_ratio"][0])
        assert model.metadata == {"source": "golden", "units": "frames"}
        assert model.plans.floor_hits == ("fc1",)
        assert model.layer_names == ["fc0", "fc1", "out"]
        for i, (fp, b) in enumerate(zip(model.factors, model.biases)):
            for got, key in ((fp.xf, "xf"), (fp.wf, "wf"), (b, "b")):
                want = golden[f"{tag}_{key}{i}"]
                assert got.dtype == want.dtype and np.array_equal(got, want)

    def test_planner_networks(self, golden):
        expect = json.loads(raw(golden, "planned_json"))
        for seed, e in enumerate(expect):
            data = raw(golden, f"planned{seed}")
            model = mi.deserialize(data)
            assert mi.serialize(model) == data
            assert mi.expected_file_size(model) == e["size"] == len(data)
            got = [[n, p.q, p.r_dim, p.rank, p.m, p.n] for n, p in model.plans.layers]
            assert got == e["layers"]
            assert list(model.plans.floor_hits) == e["floor_hits"]
            assert model.plans.achieved_total_ratio == e["ratio"]
            assert model.plans.target_ratio == e["target"]
            assert model.metadata == e["metadata"]

    def test_every_reference_error(self, golden):
        errors = json.loads(raw(golden, "errors_json"))
        cuts = set(int(c) for c in golden["cuts"])
        assert len(errors) > 200
        for name, want in errors.items():
            if name.startswith("cut"):
                cut = int(name[3:])
                assert cut in cuts
                data = raw(golden, "f32_bytes")[:cut]
                if cut >= 28:
                    data = data[:12] + (cut - 28).to_bytes(8, "little") + data[20:]
            else:
                data = raw(golden, f"bad_{name}")
            if want is None:
                mi.deserialize(data)
                continue
            with pytest.raises(ModelFormatError) as exc:
                mi.deserialize(data)
            assert (str(exc.value), exc.value.offset) == (want["message"], want["offset"]), name


class TestRoundTrip:
    def test_bytes_bit_identical(self):
        for seed in range(30):
            data = mi.serialize(random_model(seed))
            assert mi.serialize(mi.deserialize(data)) == data

    def test_thousand_models_sizes_exact(self):
        """Acceptance criterion 7: 1000 models, bit-exact, byte-exact size accounting."""
        for seed in range(1000):
            model = random_model(seed, layers=1 + seed % 3,
                                 dtype=np.float32 if seed % 2 else np.float64)
            data = mi.serialize(model)
            assert len(data) == mi.expected_file_size(model)
            assert mi.serialize(mi.deserialize(data)) == data

    def test_float32_payload(self):
        model = random_model(99, dtype=np.float32)
        back = mi.deserialize(mi.serialize(model))
        assert back.factors[0].dtype == np.float32
        for a, b in zip(model.factors, back.factors):
            assert np.array_equal(a.xf, b.xf) and np.array_equal(a.wf, b.wf)

    def test_values_metadata_plans_survive(self):
        model = random_model(7, layers=3)
        back = mi.deserialize(mi.serialize(model))
        assert back.metadata == model.metadata
        assert back.plans.layers == model.plans.layers
        assert back.plans.floor_hits == model.plans.floor_hits
        for a, b in zip(model.biases, back.biases):
            assert np.array_equal(a, b)

    def test_empty_model_is_header_only(self):
        plans = NetworkPlan(layers=(), target_ratio=0.5, achieved_total_ratio=0.0, floor_hits=())
        data = mi.serialize(mi.CompressedModel(plans=plans, factors=[], biases=[]))
        assert len(data) == 28 + 4
        back = mi.deserialize(data)
        assert back.factors == [] and back.metadata == {}

    def test_save_and_load(self, tmp_path):
        model = random_model(8)
        path = tmp_path / "model.dthn"
        written = mi.save_model(model, path)
        assert written == path.stat().st_size == mi.expected_file_size(model)
        assert mi.serialize(mi.load_model(path)) == mi.serialize(model)

    def test_magic(self):
        assert mi.MAGIC == b"DTHN" and mi.serialize(random_model(9))[:4] == b"DTHN"


class TestImageCache:
    def test_deserialized_model_reuses_its_image(self):
        data = mi.serialize(random_model(3, layers=2))
        model = mi.deserialize(data)
        assert model.image()[0] is model._image
        assert model.image()[0] == data

    def test_edits_invalidate_the_image(self):
        model = mi.deserialize(mi.serialize(random_model(4, layers=2)))
        before = model.image()[0]
        model.biases[0][0] += 1.0
        after = model.image()[0]
        assert after != before and mi.deserialize(after).biases[0][0] == model.biases[0][0]
        model.metadata["extra"] = "x"
        assert mi.deserialize(model.image()[0]).metadata["extra"] == "x"

    def test_stored_factors_are_read_only(self):
        model = mi.deserialize(mi.serialize(random_model(5)))
        with pytest.raises(ValueError):
            model.factors[0].xf[0, 0] = 1.0


class TestErrors:
    def test_mismatched_counts(self):
        plans = random_model(1, layers=2).plans
        with pytest.raises(ArgumentError):
            mi.CompressedModel(plans=plans, factors=[], biases=[])

    def test_factor_plan_mismatch(self):
        model = random_model(2, layers=2)
        model.factors[0], model.factors[1] = model.factors[1], model.factors[0]
        with pytest.raises(ArgumentError, match="does not match its plan"):
            mi.serialize(model)

    def test_unsupported_dtype(self):
        model = random_model(2, layers=1)
        fp = model.factors[0]
        model.factors[0] = mi.StoredFactors(fp.xf.astype(np.float16), fp.wf.astype(np.float16),
                                            fp.plan)
        with pytest.raises(ArgumentError, match="unsupported dtype"):
            mi.serialize(model)

    def test_declared_payload_must_match(self):
        data = mi.serialize(random_model(4)) + b"junk"
        with pytest.raises(ModelFormatError) as exc:
            mi.deserialize(data)
        assert exc.value.offset == 12

    def test_trailing_bytes(self):
        data = mi.serialize(random_model(4)) + b"junk"
        data = data[:12] + (len(data) - 28).to_bytes(8, "little") + data[20:]
        with pytest.raises(ModelFormatError, match="4 trailing bytes") as exc:
            mi.deserialize(data)
        assert exc.value.offset == len(data) - 4

    def test_bad_utf8_name_fails_like_the_reference(self):
        """The reference decodes each name as it reads it: invalid utf-8 raises
        UnicodeDecodeError before any later structural error."""
        model = random_model(6, layers=1)
        data = bytearray(mi.serialize(model))
        meta = 4 + sum(8 + len(k) + len(v) for k, v in model.metadata.items())
        data[28 + meta + 4] = 0xFF  # first byte of the first layer name
        data = bytes(data) + b"x"
        data = data[:12] + (len(data) - 28).to_bytes(8, "little") + data[20:]
        with pytest.raises(UnicodeDecodeError):
            mi.deserialize(data)

    def test_huge_declared_lengths_truncate(self):
        """u32/u64 lengths far beyond the file report a truncation, never over-read."""
        model = random_model(6, layers=1)
        data = bytearray(mi.serialize(model))
        meta = 4 + sum(8 + len(k) + len(v) for k, v in model.metadata.items())
        data[28 + meta:28 + meta + 4] = (0xFFFFFFFF).to_bytes(4, "little")
        with pytest.raises(ModelFormatError, match="layer 0 name: need 4294967295 bytes"):
            mi.deserialize(bytes(data))
