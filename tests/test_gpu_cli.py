"""The GPU bench command prints the reference CLI's CSV (cli.py:137-189)."""

import csv
import io
import subprocess
import sys

import pytest

from paper_1802_06944_b200.cli import HEADER

pytestmark = pytest.mark.gpu


def test_bench_csv_columns_and_counts():
    out = subprocess.run([sys.executable, "-m", "paper_1802_06944_b200", "bench", "--q", "1024",
                          "--r", "1024", "--ratio", "0.04", "--ratio", "0.0001", "--batch", "64",
                          "--rank", "2", "--repeat", "3", "--prefer", "reuse"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    rows = list(csv.reader(io.StringIO(out.stdout)))
    assert rows[0] == HEADER and len(rows) == 2          # the infeasible ratio is skipped
    assert "infeasible" in out.stderr
    r = dict(zip(HEADER, rows[1]))
    assert int(r["multiplies_dense"]) == 1024 * 1024 * 64 and float(r["fused_ms"]) > 0
    assert float(r["ratio"]) <= 0.04
