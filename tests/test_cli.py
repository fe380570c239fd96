"""`python -m paper_2603_00035_b200 solve|bench` mirrors rfeik's cmd_solve and
cmd_bench (tools/main.cpp:56-85, :304-347): files, stdout, CSV, exit codes."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, assert_bitwise

pytestmark = pytest.mark.gpu


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2603_00035_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_cli_solve_bitwise_vs_reference(reflib, tmp_path):
    from paper_2603_00035_b200 import field_io as fio

    n = 48
    F = reflib.random_feasible_fields(n, 21, 0.2)
    src = np.zeros((n, n), np.uint8)
    src[20, 30] = 1
    fio.write_metric(tmp_path / "g.rfek", *F[:3])
    fio.write_drift(tmp_path / "b.rfek", *F[3:])
    fio.write_mask(tmp_path / "s.rfek", src)
    out = _run("solve", "--metric", str(tmp_path / "g.rfek"), "--drift", str(tmp_path / "b.rfek"),
               "--sources", str(tmp_path / "s.rfek"), "--h", str(1.0 / n), "--out", str(tmp_path / "t.rfek"))
    assert out.returncode == 0, out.stderr
    want = reflib.solve(*F, src, 1.0 / n)
    assert_bitwise(fio.read_arrival(tmp_path / "t.rfek"), want.t)
    assert out.stdout.strip() == f"iters={want.iterations} max_delta={fio._to_chars(float(want.history[-1]))}"
    # iteration cap hit -> numerical exit code
    out = _run("solve", "--metric", str(tmp_path / "g.rfek"), "--drift", str(tmp_path / "b.rfek"),
               "--sources", str(tmp_path / "s.rfek"), "--h", str(1.0 / n), "--out", str(tmp_path / "t2.rfek"),
               "--max-iters", "1")
    assert out.returncode == 3
    assert _run("solve", "--metric", "x").returncode == 2


def test_cli_bench_csv(tmp_path):
    out = _run("bench", "--sizes", "16,32", "--repeat", "2", "--out", str(tmp_path / "b.csv"))
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[0].startswith("size=16 iters=2 median_ms=") and lines[1].startswith("size=32 iters=")
    rows = (tmp_path / "b.csv").read_text().strip().splitlines()
    assert [r.split(",")[0] for r in rows] == ["16", "32"]
