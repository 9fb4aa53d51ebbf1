"""VQH1 point files, loaded straight into pinned host memory and HBM.

Follows the reference's binary format and its checks
(``proj/src/io.cpp:67-88``, magic ``proj/include/vqhull/io.hpp:19``):
4-byte magic ``VQH1``, little-endian u64 ``n``, then ``xs[n]`` and ``ys[n]``
as f64 — exactly the SoA layout the device path keeps in HBM, so a file is
two reads into pinned buffers and two H2D copies, no reshuffle.  Errors
raise :class:`LoadError` with the reference's messages (bad magic, truncated
header, truncated payload, non-finite coordinate at point i).  The text
format (``pbbs_sequencePoint2d``) is out of scope.
"""
from __future__ import annotations

import os
import struct
from typing import Tuple

import numpy as np

MAGIC = b"VQH1"
HEADER_BYTES = 12

__all__ = ["LoadError", "MAGIC", "save_vqh1", "load_vqh1", "load_vqh1_device"]


class LoadError(ValueError):
    """The reference's ``vqhull::LoadError`` (io.hpp)."""


def save_vqh1(path: str, xs, ys) -> None:
    """Write ``xs``/``ys`` as one VQH1 file (the reference's ``save_points``)."""
    xs = np.ascontiguousarray(xs, dtype="<f8")
    ys = np.ascontiguousarray(ys, dtype="<f8")
    if xs.shape != ys.shape or xs.ndim != 1:
        raise ValueError("xs and ys must be 1-D arrays of the same length")
    with _open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<Q", xs.size))
        f.write(xs.tobytes())
        f.write(ys.tobytes())


def _open(path: str, mode: str):
    try:
        return open(path, mode)
    except OSError:
        raise LoadError(f"{path}: cannot open" + (" for writing" if "w" in mode else "")) from None


def _header(path: str, f) -> int:
    size = os.fstat(f.fileno()).st_size
    magic = f.read(4)
    if len(magic) != 4 or magic != MAGIC:
        raise LoadError(f"{path}: bad magic")
    raw = f.read(8)
    if len(raw) != 8:
        raise LoadError(f"{path}: truncated header")
    (n,) = struct.unpack("<Q", raw)
    if size != HEADER_BYTES + 16 * n:
        raise LoadError(f"{path}: truncated payload (header claims {n} points)")
    return n


def _check_finite(path: str, xs: np.ndarray, ys: np.ndarray) -> None:
    bad = ~(np.isfinite(xs) & np.isfinite(ys))
    if bad.any():
        raise LoadError(f"{path}: non-finite coordinate at point {int(np.argmax(bad))}")


def _read_into(path: str, f, buf: np.ndarray, n: int) -> None:
    view = memoryview(buf).cast("B")
    got = 0
    while got < 8 * n:
        k = f.readinto(view[got:])
        if not k:
            raise LoadError(f"{path}: truncated payload (expected {n} points)")
        got += k


def load_vqh1(path: str) -> Tuple[np.ndarray, np.ndarray]:
    """Host arrays (the reference's ``load_points`` for a binary path)."""
    with _open(path, "rb") as f:
        n = _header(path, f)
        xs = np.empty(n, dtype="<f8")
        ys = np.empty(n, dtype="<f8")
        _read_into(path, f, xs, n)
        _read_into(path, f, ys, n)
    _check_finite(path, xs, ys)
    return xs, ys


def load_vqh1_device(path: str, device="cuda", stream=None):
    """Device-resident ``(X, Y)`` float64 tensors for :func:`hull_device`.

    Each coordinate array is read into a pinned buffer and copied to HBM
    asynchronously on ``stream``, so the ``xs`` copy overlaps the ``ys`` read.
    The finiteness check runs on the host buffers before the copies are
    awaited; the pinned buffers are kept alive until the copies finish.
    """
    import torch

    with _open(path, "rb") as f:
        n = _header(path, f)
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        hy = torch.empty(n, dtype=torch.float64, pin_memory=True)
        X = torch.empty(n, dtype=torch.float64, device=device)
        Y = torch.empty(n, dtype=torch.float64, device=device)
        s = stream if stream is not None else torch.cuda.current_stream(X.device)
        with torch.cuda.stream(s):
            _read_into(path, f, hx.numpy(), n)
            X.copy_(hx, non_blocking=True)
            _read_into(path, f, hy.numpy(), n)
            Y.copy_(hy, non_blocking=True)
    try:
        _check_finite(path, hx.numpy(), hy.numpy())
    finally:
        s.synchronize()
    return X, Y
