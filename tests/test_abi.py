"""CPU tests of the C-ABI library: it loads, exports every declared symbol, and its
host-side geometry (no GPU needed) agrees with the pinned oracle and the
reference's known answers."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import deepthin_oracle as O

import paper_1802_06944_b200 as D
from paper_1802_06944_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"\b(dt_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = declared_functions()
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.dt_version()


def test_library_is_sm100a_only():
    # the fatbin carries sm_100a SASS, no PTX for other arches
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_plan_validation_matches_reference_rules():
    with pytest.raises(D.ArgumentError):
        D.LayerPlan(q=4, r_dim=4, rank=1, m=3, n=5)
    with pytest.raises(D.ArgumentError):
        D.LayerPlan(q=4, r_dim=0, rank=1, m=3, n=5)
    p = D.LayerPlan(q=440, r_dim=2048, rank=24, m=2816, n=320)
    assert p.achieved_ratio == pytest.approx(24 * (2816 + 320) / (440 * 2048))
    assert not p.reuse_path and p.info().period == 8 and p.info().tail == 0


def test_index_laws_match_golden(golden):
    for row in golden["index_laws"]:
        q, r_dim, n, m, pc, d, t = (int(v) for v in row[:7])
        p = D.LayerPlan(q=q, r_dim=r_dim, rank=1, m=m, n=n)
        assert D.phase_count(p) == pc
        assert tuple(D.predict_reuse(p)) == (d, t)
        assert [D.phase(int(c), p) for c in row[11:15]] == row[7:11].tolist()
        info = p.info()
        assert info.reuse == (q % n == 0)
        assert info.tail == m * n - q * r_dim


def test_relayout_and_errors(golden):
    p = D.LayerPlan(q=7, r_dim=5, rank=1, m=7, n=5)
    got = np.array([D.relayout_index(k, p) for k in range(35)])
    assert np.array_equal(got, golden["relayout_7x5"])
    with pytest.raises(D.ArgumentError):
        D.relayout_index(35, p)
    with pytest.raises(D.ArgumentError):
        D.phase(5, p)


def test_op_counts_match_oracle_and_reference(golden):
    for i in range(16):
        q, r_dim, rank, m, n = (int(v) for v in golden[f"fm{i}_plan"])
        p = D.LayerPlan(q=q, r_dim=r_dim, rank=rank, m=m, n=n)
        batch = golden[f"fm{i}_x"].shape[0]
        hits, misses, mul, add = (int(v) for v in golden[f"fm{i}_counts"])
        ops = D.op_count(p, batch)
        assert (ops.multiplies, ops.adds) == (mul, add)
        pred = D.predict_reuse(p, batch)
        assert pred.distinct_runs * batch == misses
        assert pred.total_runs * batch - misses == hits


def test_baseline_config_geometry():
    # c1/c3/c5 single phase (reuse); c2 period 8; c4-fc1 period 160, tail 128
    c1 = D.baseline_plan(1024, 1024, 16, 256, 4096)
    c2 = D.baseline_plan(440, 2048, 24, 320, 2816)
    c4 = D.baseline_plan(494, 2048, 3, 320)
    c5 = D.baseline_plan(8192, 8192, 64, 1024, 65536)
    assert c1.reuse_path and c5.reuse_path and not c2.reuse_path and not c4.reuse_path
    assert c4.m == 3162 and c4.info().period == 160 and c4.info().tail == 128
    assert c2.info().phase_count == 8
    assert tuple(D.predict_reuse(c2)) == (18, 4608)


def test_status_mapping():
    with pytest.raises(D.DimensionError):
        _lib.check(_lib.DT_E_DIM)
    with pytest.raises(D.UnsupportedConfigurationError):
        _lib.check(_lib.DT_E_UNSUPPORTED)
    with pytest.raises(D.CudaError):
        _lib.check(_lib.DT_E_CUDA)


def test_forward_rejects_bad_arguments_before_touching_the_gpu():
    lib = _lib.lib()
    ps = _lib.Plan(440, 2048, 24, 2816, 320)
    rc = lib.dt_forward(C.byref(ps), 4, 7, None, 0, None, None, 0, None, 0, 0.0, None, 0, None, 0,
                        None)
    assert rc == _lib.DT_E_ARG
    rc = lib.dt_forward(C.byref(ps), 4, 0, None, 0, None, None, 0, None, 99, 0.0, None, 0, None, 0,
                        None)
    assert rc == _lib.DT_E_ARG
    bad = _lib.Plan(4, 4, 1, 3, 5)
    assert lib.dt_forward(C.byref(bad), 1, 0, None, 0, None, None, 0, None, 0, 0.0, None, 0, None,
                          0, None) == _lib.DT_E_ARG


def test_new_entry_points_validate_before_touching_the_gpu():
    """Geometry / argument checks of the row-tile, LSTM and training entry points run on the
    host (no device work for a rejected call)."""
    lib = _lib.lib()
    reuse = _lib.Plan(2048, 2048, 3, 16384, 256)      # row-tile geometry (config 3)
    general = _lib.Plan(440, 2048, 24, 2816, 320)     # straddling rows
    assert lib.dt_rows_prepared_bytes(C.byref(reuse), _lib.DT_BF16, _lib.DT_BF16) > 0
    assert lib.dt_rows_prepared_bytes(C.byref(general), _lib.DT_BF16, _lib.DT_BF16) == 0
    assert lib.dt_rows_prepared_bytes(C.byref(reuse), _lib.DT_F32, _lib.DT_BF16) == 0  # bf16 x only
    assert lib.dt_rows_prepare(C.byref(general), 0, _lib.DT_BF16, None, None, None, None, None) \
        == _lib.DT_E_UNSUPPORTED
    assert lib.dt_rows_prepare(C.byref(reuse), 0, _lib.DT_BF16, None, None, None, None, None) \
        == _lib.DT_E_ARG
    assert lib.dt_rows_posts_per_tile(C.byref(reuse)) == 4 * 16  # cluster of 4 x 16 epilogue warps
    lstm = _lib.Plan(2048, 2048, 32, 16384, 256)
    assert lib.dt_lstm_sequence_workspace_bytes(C.byref(lstm), 64) > 0
    assert lib.dt_lstm_sequence_workspace_bytes(C.byref(lstm), 65) == 0   # batch <= 64
    assert lib.dt_lstm_gates_workspace_bytes(C.byref(general), 8) == 0    # square reuse only
    P4 = C.c_void_p * 4
    assert lib.dt_lstm_sequence(C.byref(lstm), 10, 65, P4(), P4(), P4(), P4(), None, None, 0,
                                None) == _lib.DT_E_UNSUPPORTED
    assert lib.dt_lstm_cell(4, 8, None, 4, None, None, None, None, None) == _lib.DT_E_DIM  # ld < hidden
    # P is kept for the tensor-core backward (k_train.cu): reuse geometries with rank % 4 == 0
    # (TMA pitches of P and of H's bf16 hi | lo rows); rank 3 trains on the FFMA backward
    assert lib.dt_forward_p_bytes(C.byref(reuse), 128) == 0
    c5 = _lib.Plan(8192, 8192, 64, 65536, 1024)
    assert lib.dt_forward_p_bytes(C.byref(c5), 128) == 128 * 8 * 64 * 4
    assert lib.dt_forward_p_bytes(C.byref(general), 128) == 0
    assert lib.dt_profile_kernel_kind(7) == _lib.DT_E_ARG


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = D.LayerPlan(q=8, r_dim=8, rank=1, m=8, n=8)
    with pytest.raises(D.CudaError):
        D.FactorPair(np.ones((8, 1)), np.ones((1, 8)), p)


def test_forward_path_selection():
    """dt_forward_path (host-only): the kernel family per geometry and dtypes."""
    import torch
    cases = {(440, 2048, 3, 320): ("runs", "hilo"), (2048, 2048, 3, 256): ("rows", "rows"),
             (8192, 8192, 64, 1024): ("factored", "factored"), (440, 512, 4, 320): ("pair", "hilo")}
    for (q, r, k, n), want in cases.items():
        p = D.LayerPlan(q=q, r_dim=r, rank=k, m=-(-(q * r) // n), n=n)
        got = tuple(D.forward_path(p, "bf16", torch.bfloat16, y) for y in (torch.bfloat16, torch.float32))
        assert got == want, (q, r, k, n, got)
        assert D.forward_path(p, "ffma", torch.float32, torch.float32) == "ffma"
        # a fp32 x disqualifies the bf16-only kernels (rows / runs); the staged forms remain
        assert D.forward_path(p, "bf16", torch.float32, torch.bfloat16) in ("factored", "pair")
    with pytest.raises(D.ArgumentError):
        D.forward_path(p, "ffma", torch.float32, torch.float32, factors="bf16")
