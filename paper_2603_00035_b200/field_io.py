"""RFEK1 field files and CSV export (the reference's field_io.hpp:10-39,
src/field_io.cpp:39-158), for interop with the reference's tooling.

Layout: magic ``b"RFEK1\\n"``, three little-endian u32 (rows, cols,
channels), then rows*cols*channels little-endian f64, row-major with the
channel index fastest.  Host-side numpy (file I/O is not a device path);
the error types mirror randers::BadMagic / TruncatedFile / ZeroDimension /
DimensionMismatch / IoFailure.
"""
from __future__ import annotations

import numpy as np

from .api import DimensionMismatch, Error, ZeroDimension

MAGIC = b"RFEK1\n"


class BadMagic(Error):
    pass


class TruncatedFile(Error):
    pass


class IoFailure(Error):
    pass


def _host(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)


def write_field(path, channels) -> None:
    """write_field (field_io.cpp:84-103): channels of one shape."""
    chans = [np.asarray(_host(c), dtype=np.float64) for c in channels]
    if not chans:
        raise DimensionMismatch("write_field: no channels")
    shape = chans[0].shape
    if len(shape) != 2 or any(c.shape != shape for c in chans):
        raise DimensionMismatch("write_field: channel dimensions differ")
    rows, cols = shape
    head = MAGIC + np.array([rows, cols, len(chans)], dtype="<u4").tobytes()
    body = np.stack(chans, axis=-1).astype("<f8", copy=False).tobytes()
    try:
        with open(path, "wb") as f:
            f.write(head)
            f.write(body)
    except OSError as e:
        raise IoFailure(f"cannot open {path} for writing") from e


def read_field(path) -> list:
    """read_field (field_io.cpp:54-82): the list of channel planes."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoFailure(f"cannot open {path}") from e
    if len(data) < 6 or data[:6] != MAGIC:
        raise BadMagic(f"bad magic in {path}")
    if len(data) < 18:
        raise TruncatedFile(f"truncated header in {path}")
    rows, cols, chans = (int(v) for v in np.frombuffer(data, dtype="<u4", count=3, offset=6))
    if rows == 0 or cols == 0 or chans == 0:
        raise ZeroDimension(f"zero dimension in {path}")
    if len(data) < 18 + 8 * rows * cols * chans:
        raise TruncatedFile(f"truncated payload in {path}")
    v = np.frombuffer(data, dtype="<f8", count=rows * cols * chans, offset=18).reshape(rows, cols, chans)
    return [np.ascontiguousarray(v[:, :, k]).astype(np.float64) for k in range(chans)]


def _expect(path, k, what):
    ch = read_field(path)
    if len(ch) != k:
        raise DimensionMismatch(f"{what} file needs {k} channel{'s' if k > 1 else ''}")
    return ch


def write_metric(path, g11, g12, g22):
    write_field(path, [g11, g12, g22])


def read_metric(path):
    return tuple(_expect(path, 3, "metric"))


def write_drift(path, b1, b2):
    write_field(path, [b1, b2])


def read_drift(path):
    return tuple(_expect(path, 2, "drift"))


def write_mask(path, mask):
    write_field(path, [(np.asarray(_host(mask)) != 0).astype(np.float64)])


def read_mask(path):
    return (_expect(path, 1, "mask")[0] != 0.0).astype(np.uint8)


def write_arrival(path, t):
    write_field(path, [t])


def read_arrival(path):
    return _expect(path, 1, "arrival")[0]


def _to_chars(x: float) -> str:
    """std::to_chars(double) with no format: the shortest round-trip digits in
    fixed or scientific notation, whichever is shorter (fixed on a tie)."""
    if x != x:
        return "nan" if not np.signbit(x) else "-nan"
    if np.isinf(x):
        return "inf" if x > 0 else "-inf"
    fixed = np.format_float_positional(x, unique=True, trim="-")
    sci = np.format_float_scientific(x, unique=True, trim="-", exp_digits=2)
    return fixed if len(fixed) <= len(sci) else sci


def export_csv(field, path) -> None:
    """export_csv (field_io.cpp:105-118)."""
    a = np.asarray(_host(field), dtype=np.float64)
    try:
        with open(path, "w", newline="") as f:
            for row in a:
                f.write(",".join(_to_chars(float(v)) for v in row))
                f.write("\n")
    except OSError as e:
        raise IoFailure(f"cannot open {path} for writing") from e
