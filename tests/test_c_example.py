"""The boundary from plain C (examples/solve.c, the shape of a cgo/JNI/FFI
binding): it compiles and links against include/rfk.h + librfk.so on any host,
refuses to run without a device, and on a B200 gives the oracle's bits."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, assert_bitwise

SRC = os.path.join(ROOT, "examples", "solve.c")
LIBDIR = os.path.join(ROOT, "paper_2603_00035_b200")


def _build(tmp_path):
    exe = str(tmp_path / "solve_c")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR, "-lrfk", "-lm",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_example_matches_oracle(tmp_path, oracle):
    exe = _build(tmp_path)
    out = tmp_path / "t.bin"
    rows, cols = 64, 48
    p = subprocess.run([exe, str(rows), str(cols), str(out)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    planes = np.fromfile(out, dtype=np.float64).reshape(6, rows, cols)
    F, t = planes[:5], planes[5]
    src = np.zeros((rows, cols), np.uint8)
    src[rows // 2, cols // 2] = 1
    ref = oracle.solve(*F, src, 1.0 / rows)
    assert f"iterations {ref.iterations} converged 1" in p.stdout
    assert_bitwise(t, ref.t)
