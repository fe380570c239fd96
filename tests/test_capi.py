"""CPU tests of the boundary: librfk.so builds for sm_100a, loads, exports
every entry point include/rfk.h declares, and refuses to compute without a
device (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rfk.h")
LIB = os.path.join(ROOT, "paper_2603_00035_b200", "librfk.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"RFK_API\s+[\w\s\*]+?\b(rfk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "librfk.so not built"
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = C.CDLL(LIB)
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (rfk_\w+)", out))
    assert set(syms) == exported, (set(syms) ^ exported)


def test_python_binding_lists_the_header():
    from paper_2603_00035_b200 import _lib
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_version():
    from paper_2603_00035_b200 import _lib
    lib = _lib.load()
    assert lib.rfk_version() >= 1
    assert lib.rfk_status_string(4) == b"inconsistent fixed point"


def test_no_device_means_no_compute():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2603_00035_b200 import _lib
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.rfk_create(C.byref(h), 0) == _lib.RFK_ERR_NO_DEVICE
    import paper_2603_00035_b200 as rfk
    with pytest.raises(rfk.NoDevice):
        rfk.Context()
