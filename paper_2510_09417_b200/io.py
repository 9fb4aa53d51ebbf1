"""VQH1 point files, loaded straight into pinned host memory and HBM.

Follows the reference's binary format and its checks
(``proj/src/io.cpp:67-88``, magic ``proj/include/vqhull/io.hpp:19``):
4-byte magic ``VQH1``, little-endian u64 ``n``, then ``xs[n]`` and ``ys[n]``
as f64 — exactly the SoA layout the device path keeps in HBM, so a file is
two reads into pinned buffers and two H2D copies, no reshuffle.  Errors
raise :class:`LoadError` with the reference's messages (bad magic, truncated
header, truncated payload, non-finite coordinate at point i).  The reference's
text format (``pbbs_sequencePoint2d``, ``io.cpp:100-160``) is read and written
too (:func:`read_points`, :func:`write_points`); it is kept as written in
round 1 and not developed further.
"""
from __future__ import annotations

import os
import re
import struct
from typing import Tuple

import numpy as np

MAGIC = b"VQH1"
TEXT_HEADER = "pbbs_sequencePoint2d"
HEADER_BYTES = 12

__all__ = ["LoadError", "MAGIC", "TEXT_HEADER", "save_vqh1", "load_vqh1", "load_vqh1_device",
           "format_for_path", "read_points", "write_points", "to_chars"]


# what std::from_chars(double) accepts (general format): no leading '+', no
# hex; inf / nan spellings parse and are then rejected by the finiteness check
_NUM = re.compile(r"-?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")


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


# ---- text format and format dispatch ------------------------------------

def to_chars(v: float) -> str:
    """``std::to_chars(double)`` without a format: the shortest round-trip
    digits (Python's ``repr`` finds the same ones), printed fixed or
    scientific (``e±dd``) whichever is shorter, fixed on a tie; an integral
    value in fixed form prints exactly.  Pinned by tests/golden/to_chars.txt
    (libstdc++'s own output, tests/golden/make_to_chars.cpp)."""
    from decimal import Decimal

    v = float(v)
    if v != v:  # libstdc++ prints the sign of a NaN
        return "-nan" if str(v).startswith("-") or np.signbit(v) else "nan"
    if v in (float("inf"), float("-inf")):
        return "-inf" if v < 0 else "inf"
    neg = v < 0 or (v == 0 and str(v).startswith("-"))
    if v == 0:
        return "-0" if neg else "0"
    _, dig, exp = Decimal(repr(abs(v))).as_tuple()
    ds = "".join(map(str, dig)).lstrip("0")
    t = len(ds) - len(ds.rstrip("0"))
    ds, exp = ds[:len(ds) - t], exp + t
    k = len(ds)
    x = exp + k - 1  # value = d.ddd x 10^x
    sci = ds[0] + ("." + ds[1:] if k > 1 else "") + ("e-" if x < 0 else "e+") + f"{abs(x):02d}"
    if x >= k - 1:  # an integer: fixed form prints its exact digits, as printf("%.0f")
        fix = str(int(abs(v)))
    elif x >= 0:
        fix = ds[:x + 1] + "." + ds[x + 1:]
    else:
        fix = "0." + "0" * (-x - 1) + ds
    out = fix if len(fix) <= len(sci) else sci
    return "-" + out if neg else out


def format_for_path(path: str) -> str:
    """``"text"`` for ``.txt`` / ``.pbbs``, else ``"binary"`` (``io.cpp:91-98``)."""
    dot = path.rfind(".")
    return "text" if dot >= 0 and path[dot:] in (".txt", ".pbbs") else "binary"


def _read_text(path: str) -> Tuple[np.ndarray, np.ndarray]:
    with _open(path, "rb") as f:
        lines = f.read().decode("latin-1").split("\n")
    if not lines or (len(lines) == 1 and lines[0] == ""):
        raise LoadError(f"{path}: empty file")
    head = lines[0][:-1] if lines[0].endswith("\r") else lines[0]
    if head != TEXT_HEADER:
        raise LoadError(f'{path}: unrecognized header "{head}"')
    xs, ys = [], []
    if lines[-1] == "":
        lines.pop()
    for lineno, line in enumerate(lines[1:], start=2):
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        vals, cur = [], 0
        for _ in range(2):  # from_chars after skipping spaces/tabs; the rest of the line is ignored
            while cur < len(line) and line[cur] in " \t":
                cur += 1
            m = _NUM.match(line, cur)
            if not m:
                raise LoadError(f"{path}: malformed coordinate on line {lineno}")
            lit = m.group(0)
            try:
                v = float(lit)
            except ValueError:  # e.g. nan(...) payloads float() does not take
                raise LoadError(f"{path}: malformed coordinate on line {lineno}") from None
            # std::from_chars reports result_out_of_range (the reference:
            # malformed) for a finite literal that overflows, or a nonzero one
            # that underflows to zero
            mant = lit.lower().split("e")[0]
            if (v == 0.0 and any(c in mant for c in "123456789")) or \
                    (v in (float("inf"), float("-inf")) and "inf" not in lit.lower()):
                raise LoadError(f"{path}: malformed coordinate on line {lineno}")
            vals.append(v)
            cur = m.end()
        xs.append(vals[0])
        ys.append(vals[1])
    xs = np.array(xs, dtype=np.float64)
    ys = np.array(ys, dtype=np.float64)
    _check_finite(path, xs, ys)
    return xs, ys


def read_points(path: str) -> Tuple[np.ndarray, np.ndarray]:
    """The reference's ``read_points``: VQH1 if the file starts with the
    magic, else the text format (``io.cpp:134-144``)."""
    with _open(path, "rb") as f:
        binary = f.read(4) == MAGIC
    return load_vqh1(path) if binary else _read_text(path)


def write_points(path: str, xs, ys, fmt: str = "") -> None:
    """The reference's ``write_points``; ``fmt`` defaults to
    :func:`format_for_path`."""
    fmt = fmt or format_for_path(path)
    if fmt != "text":
        save_vqh1(path, xs, ys)
        return
    xs = np.asarray(xs, dtype=np.float64)
    ys = np.asarray(ys, dtype=np.float64)
    body = "".join(f"{to_chars(a)} {to_chars(b)}\n" for a, b in zip(xs.tolist(), ys.tolist()))
    with _open(path, "wb") as f:
        f.write((TEXT_HEADER + "\n" + body).encode("ascii"))
