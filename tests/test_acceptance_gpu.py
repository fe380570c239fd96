"""The reference's own acceptance gate (proj/tests/acceptance_main.cpp),
linked against the B200 drop-in (oracle/Makefile `acceptance`: the
reference's stencil/sweeper/adjoint translation units replaced by
paper_2603_00035_b200/csrc/shim/randers_shim.cpp over librfk.so), must print
the reference's published criterion values textually
(tests/golden/acceptance_transcript.txt = proj/test_output.txt:13-29 with the
wall-clock timings stripped)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def test_reference_acceptance_gate_textually_identical():
    if not os.path.exists(BIN):
        pytest.skip("acceptance_b200 not built (needs the reference sources at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    # the timing suffix is wall clock; everything before it must match the
    # published transcript (trailing blanks are layout, not values)
    lines = [re.sub(r"\s*\[(total )?\s*[0-9.]+s\]\s*$", "", l).rstrip() for l in out.stdout.strip().splitlines()]
    want = [l.rstrip() for l in
            open(os.path.join(ROOT, "tests", "golden", "acceptance_transcript.txt")).read().strip().splitlines()]
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert lines == want
