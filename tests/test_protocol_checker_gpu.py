"""The sweep's cross-warp / cross-CTA shared-memory protocols under the
protocol checker (compute-sanitizer is refused on this pool): the diagnostic
build librfk_chk.so tags every ring slot with the position / step it holds
and checks every read (rfk_sweep.cu, RFK_SWEEP_CHECKED).  Golden solves in
three sweep orders, random skinny / tiny / non-square grids, concurrent
batched grids and one 4096^2 solve must run with no violation and give the
oracle's bits (scripts/check_protocols.py).  The fault-injected build (one
chunk staged past the ring) is caught: profiles/r02_protocols_fault.log."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_protocol_checker_clean():
    lib = os.path.join(ROOT, "paper_2603_00035_b200", "librfk_chk.so")
    if not os.path.exists(lib):
        pytest.skip("librfk_chk.so not built")
    env = dict(os.environ, RFK_LIBRARY=lib, REPS="3")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "check_protocols.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "0 violations" in p.stdout
