"""RFEK1 field files and CSV export (field_io.cpp:39-158): byte-identical to
the reference's writer, readable by the reference's reader, same errors."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2603_00035_b200 import field_io as fio


def _ref(reflib):
    L = reflib.lib
    L.ref_write_field.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
    L.ref_read_field_dims.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.ref_read_field.argtypes = [C.c_char_p, C.c_void_p]
    L.ref_export_csv.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_void_p]
    return L


def _planes(rows=7, cols=5, ch=3, seed=0):
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(ch, rows, cols)) * 10.0 ** rng.integers(-12, 12, size=(ch, rows, cols))
    p.flat[0], p.flat[1], p.flat[2] = 1.0, -0.0, 1e10
    return p


def test_write_matches_reference_bytes(reflib, tmp_path):
    L = _ref(reflib)
    p = _planes()
    mine, theirs = tmp_path / "a.rfek", tmp_path / "b.rfek"
    fio.write_field(mine, list(p))
    assert L.ref_write_field(str(theirs).encode(), 7, 5, 3, np.ascontiguousarray(p).ctypes.data) == 0
    assert mine.read_bytes() == theirs.read_bytes()
    back = fio.read_field(theirs)
    for a, b in zip(back, p):
        np.testing.assert_array_equal(a.view(np.uint64), b.view(np.uint64))
    r, c, k = C.c_int(), C.c_int(), C.c_int()
    assert L.ref_read_field_dims(str(mine).encode(), C.byref(r), C.byref(c), C.byref(k)) == 0
    assert (r.value, c.value, k.value) == (7, 5, 3)


def test_typed_files_and_errors(tmp_path):
    g = _planes(4, 6, 3, 1)
    fio.write_metric(tmp_path / "g.rfek", *g)
    assert all(np.array_equal(a, b) for a, b in zip(fio.read_metric(tmp_path / "g.rfek"), g))
    m = (np.arange(24).reshape(4, 6) % 5 == 0).astype(np.uint8)
    fio.write_mask(tmp_path / "m.rfek", m)
    np.testing.assert_array_equal(fio.read_mask(tmp_path / "m.rfek"), m)
    with pytest.raises(fio.DimensionMismatch):
        fio.read_drift(tmp_path / "g.rfek")
    (tmp_path / "bad").write_bytes(b"RFEK2\n" + bytes(20))
    with pytest.raises(fio.BadMagic):
        fio.read_field(tmp_path / "bad")
    (tmp_path / "short").write_bytes(fio.MAGIC + bytes(5))
    with pytest.raises(fio.TruncatedFile):
        fio.read_field(tmp_path / "short")
    (tmp_path / "zero").write_bytes(fio.MAGIC + np.array([0, 3, 1], "<u4").tobytes())
    with pytest.raises(fio.ZeroDimension):
        fio.read_field(tmp_path / "zero")
    full = fio.MAGIC + np.array([2, 2, 1], "<u4").tobytes() + bytes(8 * 3)
    (tmp_path / "trunc").write_bytes(full)
    with pytest.raises(fio.TruncatedFile):
        fio.read_field(tmp_path / "trunc")
    with pytest.raises(fio.IoFailure):
        fio.read_field(tmp_path / "missing")


def test_export_csv_matches_reference(reflib, tmp_path):
    L = _ref(reflib)
    p = _planes(9, 8, 1, 2)[0]
    p[0, :6] = [1.0, 0.5, 1e-5, 123456.0, 1e16, 0.1 + 0.2]
    mine, theirs = tmp_path / "a.csv", tmp_path / "b.csv"
    fio.export_csv(p, mine)
    assert L.ref_export_csv(str(theirs).encode(), 9, 8, np.ascontiguousarray(p).ctypes.data) == 0
    assert mine.read_text() == theirs.read_text()
