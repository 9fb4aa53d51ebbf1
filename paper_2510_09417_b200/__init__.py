"""B200-native VQhull hot path — Python front-end over the C ABI.

Mirrors the reference's public surface for this path (VQhull,
``/root/reference/proj/include/vqhull``):

==========================  ===============================================
this module                 reference
==========================  ===============================================
``vqhull_compute``          ``vqhull_compute``   (vqhull_c.h:23-24)
``convex_hull``             ``convex_hull``      (hull.hpp:58) -> HullPolygon
``find_extremes``           ``find_extremes``    (geometry.hpp:135-138)
``extract_subsets``         ``extract_subsets``  (extract.hpp:79-82)
``generate``                ``generate``         (dataset.hpp:50) + square
==========================  ===============================================

Every computation runs in ``lib/libvqhull_b200.so`` (hand-written sm_100a
kernels).  There is no CPU fallback: if the library or a GPU is missing the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "LIB_PATH", "VQhullError", "lib", "available", "vqhull_compute", "convex_hull",
    "hull_indices", "hull_device", "find_extremes", "extract_subsets", "generate", "stats",
    "set_timing", "set_stable", "HullPolygon", "ExtractOutcome", "KINDS", "Stats",
    "shard_candidates", "shard_repack", "merge_candidates", "hull_multi", "RetryWithFloor",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# VQHULL_LIB selects another build of the same library (e.g. the debug build
# lib/libvqhull_b200_dbg.so with device bounds checks)
LIB_PATH = os.environ.get("VQHULL_LIB", os.path.join(HERE, "lib", "libvqhull_b200.so"))

VQHULL_OK, VQHULL_EINVAL, VQHULL_ESIZE, VQHULL_ECUDA, VQHULL_ERETRY = 0, 1, 2, 3, 4
KINDS = {"kuzmin": 0, "circle": 1, "disk": 2, "square": 3}

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_szp = C.POINTER(C.c_size_t)
_ip = C.POINTER(C.c_int)


class VQhullError(RuntimeError):
    def __init__(self, rc: int, what: str):
        super().__init__(f"{what} failed with code {rc}")
        self.rc = rc


class Stats(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("hull_size", C.c_uint64), ("levels", C.c_uint32),
        ("launches", C.c_uint32), ("survivors_root", C.c_uint64), ("level_points", C.c_uint64),
        ("finisher_points", C.c_uint64), ("finisher_segments", C.c_uint64),
        ("segments", C.c_uint64), ("bytes_moved", C.c_uint64),
        ("ms_extremes", C.c_float), ("ms_bootstrap", C.c_float),
        ("ms_root_partition", C.c_float), ("ms_levels", C.c_float), ("ms_finisher", C.c_float),
        ("ms_other", C.c_float), ("ms_total", C.c_float), ("timing_valid", C.c_uint32),
        ("bytes_extremes", C.c_uint64), ("bytes_bootstrap", C.c_uint64),
        ("bytes_root_partition", C.c_uint64), ("bytes_levels", C.c_uint64),
        ("bytes_finisher", C.c_uint64),
        ("root_filtered", C.c_uint32),
        ("root_filter_on", C.c_uint32),
        ("root_reruns", C.c_uint32),
        ("tail_launches", C.c_uint32),
        ("tail_levels", C.c_uint32),
        ("shard_tested", C.c_uint64),
        ("shard_candidates", C.c_uint64),
        ("shard_cert_vertices", C.c_uint32),
        ("pad0", C.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_LIB = None


def lib() -> C.CDLL:
    """Load the native library (built by ``__graft_entry__.build()``)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.vqhull_compute.argtypes = [_dp, _dp, C.c_size_t, C.c_int, _szp, _szp]
        L.vqhull_cuda_hull.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, _u64p,
                                       C.c_void_p]
        L.vqhull_cuda_hull_u32.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                                           _u64p, C.c_void_p]
        L.vqhull_cuda_find_extremes.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, _u64p, _u64p,
                                                C.c_void_p]
        L.vqhull_cuda_extract_subsets.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, _dp, _dp,
                                                  _u64p, _u64p, _dp, _ip, _dp, _ip, C.c_void_p]
        L.vqhull_cuda_get_stats.argtypes = [C.POINTER(Stats)]
        L.vqhull_cuda_set_timing.argtypes = [C.c_int]
        L.vqhull_cuda_set_stable.argtypes = [C.c_int]
        L.vqhull_cuda_set_root_reference.argtypes = [C.c_int]
        L.vqhull_cuda_set_root_mode.argtypes = [C.c_int]
        L.vqhull_cuda_set_filter_inner.argtypes = [C.c_int]
        L.vqhull_cuda_trim.argtypes = []
        L.vqhull_cuda_last_error.restype = C.c_char_p
        L.vqhull_b200_version.restype = C.c_char_p
        L.vqhull_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                      C.c_void_p, C.c_int]
        L.vqhull_cuda_shard_candidates.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                                                   C.c_double, C.c_void_p, C.c_uint64, _u64p,
                                                   C.c_void_p]
        L.vqhull_cuda_shard_repack.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.vqhull_cuda_merge_candidates.argtypes = [C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p,
                                                   _u64p, _dp, C.c_void_p]
        L.vqhull_cuda_hull_multi.argtypes = [_dp, _dp, C.c_uint64, C.c_int, _u64p, _u64p]
        _LIB = L
    return _LIB


def available() -> bool:
    """True when the library loads and sees a CUDA device."""
    try:
        return bool(lib().vqhull_cuda_available())
    except OSError:
        return False


def _check(rc: int, what: str) -> None:
    if rc == VQHULL_ECUDA:
        raise VQhullError(rc, f"{what}: {lib().vqhull_cuda_last_error().decode()}")
    if rc:
        raise VQhullError(rc, what)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# host-array API (the reference's C entry point)
# ---------------------------------------------------------------------------
def vqhull_compute(xs, ys, workers: int = 1) -> Tuple[int, np.ndarray]:
    """vqhull_compute semantics: returns (rc, clockwise first-occurrence indices)."""
    xs, ys = _f64(xs), _f64(ys)
    if xs.shape != ys.shape:
        raise ValueError("xs and ys differ in length")
    n = xs.size
    out = np.zeros(max(n, 1), dtype=np.uint64)
    cnt = C.c_size_t(0)
    rc = lib().vqhull_compute(xs.ctypes.data_as(_dp), ys.ctypes.data_as(_dp), n, workers,
                              out.ctypes.data_as(_szp), C.byref(cnt))
    return rc, out[: cnt.value].copy()


def hull_indices(xs, ys) -> np.ndarray:
    rc, idx = vqhull_compute(xs, ys)
    _check(rc, "vqhull_compute")
    return idx


@dataclass
class HullPolygon:
    """hull.hpp:17-22 — vertices clockwise from the leftmost(-lowest) point."""
    xs: np.ndarray
    ys: np.ndarray
    indices: np.ndarray

    def size(self) -> int:
        return int(self.indices.size)

    def empty(self) -> bool:
        return self.indices.size == 0


def convex_hull(xs, ys) -> HullPolygon:
    """convex_hull(PointSet) — coordinates of the hull, computed on the GPU."""
    xs, ys = _f64(xs), _f64(ys)
    idx = hull_indices(xs, ys)
    return HullPolygon(xs[idx.astype(np.int64)], ys[idx.astype(np.int64)], idx)


# ---------------------------------------------------------------------------
# device-array API (torch tensors as HBM handles)
# ---------------------------------------------------------------------------
def _stream_ptr(stream, device=None) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _check_pair(x, y, what: str, writable: bool = False) -> None:
    """Both coordinate arrays: float64 CUDA tensors of one length on one
    device (the kernels index y by x's positions and launch on x's device)."""
    import torch
    for t in (x, y):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
            raise TypeError(f"{what}: coordinates must be float64 CUDA tensors")
        if writable and not t.is_contiguous():
            raise ValueError(f"{what}: in-place call needs contiguous tensors")
    if x.numel() != y.numel():
        raise ValueError(f"{what}: x has {x.numel()} points, y has {y.numel()}")
    if x.device != y.device:
        raise ValueError(f"{what}: x is on {x.device}, y on {y.device}")


def hull_device(x, y, stream=None, out=None, u32: bool = False):
    """Hull of device-resident points (torch float64 CUDA tensors).

    Returns a CUDA tensor of indices (int64 view of the uint64 list, or int32
    when ``u32``) — clockwise, first occurrence.  Runs on x's device (its
    current stream unless ``stream`` is given).
    """
    import torch
    _check_pair(x, y, "hull_device")
    x, y = x.contiguous(), y.contiguous()
    n = x.numel()
    want = torch.int32 if u32 else torch.int64
    if out is None:
        out = torch.empty(max(n, 1), dtype=want, device=x.device)
    elif out.dtype != want or out.device != x.device or out.numel() < n or not out.is_contiguous():
        raise ValueError(f"hull_device: out must be a contiguous {want} tensor on {x.device} "
                         f"with room for {n} indices")
    cnt = C.c_uint64(0)
    fn = lib().vqhull_cuda_hull_u32 if u32 else lib().vqhull_cuda_hull
    if x.device.index == torch.cuda.current_device():  # (the common case: no device switch)
        rc = fn(x.data_ptr(), y.data_ptr(), n, out.data_ptr(), C.byref(cnt), _stream_ptr(stream, x.device))
    else:
        with torch.cuda.device(x.device):
            rc = fn(x.data_ptr(), y.data_ptr(), n, out.data_ptr(), C.byref(cnt), _stream_ptr(stream, x.device))
    _check(rc, "vqhull_cuda_hull")
    return out[: cnt.value]


# ---------------------------------------------------------------------------
# sharded hull building blocks (distributed.py drives them)
# ---------------------------------------------------------------------------
class RetryWithFloor(Exception):
    """The merge found a shard whose margin scale is too small for the largest
    coordinate in play: recompute every shard with ``floor``."""

    def __init__(self, floor: float):
        super().__init__(f"recompute the shards with margin floor {floor!r}")
        self.floor = floor


def shard_candidates(x, y, offset: int, cap: int, floor: float = 0.0, stream=None):
    """Local stage of the sharded hull on x's device: returns (pack, count),
    pack a float64 tensor of cap + 1 rows x 3 (header {count, M_eff, A}, then
    the first min(count, cap) candidates {x, y, global index bits}).  A
    count above cap: call :func:`shard_repack` with a larger buffer."""
    import torch
    _check_pair(x, y, "shard_candidates")
    x, y = x.contiguous(), y.contiguous()
    pack = torch.empty((cap + 1, 3), dtype=torch.float64, device=x.device)
    cnt = C.c_uint64(0)
    with torch.cuda.device(x.device):
        rc = lib().vqhull_cuda_shard_candidates(x.data_ptr(), y.data_ptr(), x.numel(), int(offset),
                                                float(floor), pack.data_ptr(), cap, C.byref(cnt),
                                                _stream_ptr(stream, x.device))
    _check(rc, "vqhull_cuda_shard_candidates")
    return pack, int(cnt.value)


def shard_repack(pack, stream=None) -> None:
    """The last shard_candidates' rows again into ``pack`` (rows - 1 of room)."""
    import torch
    with torch.cuda.device(pack.device):
        rc = lib().vqhull_cuda_shard_repack(pack.data_ptr(), pack.shape[0] - 1,
                                           _stream_ptr(stream, pack.device))
    _check(rc, "vqhull_cuda_shard_repack")


def merge_candidates(packs, stream=None):
    """Merge on packs' device: ``packs`` (nranks, rows, 3) float64 in offset
    order.  Returns the global clockwise index list (int64 CUDA tensor);
    raises :class:`RetryWithFloor` when the shards must be recomputed."""
    import torch
    packs = packs.contiguous()
    nranks, rows = packs.shape[0], packs.shape[1]
    out = torch.empty(max(nranks * (rows - 1), 1), dtype=torch.int64, device=packs.device)
    cnt = C.c_uint64(0)
    fl = C.c_double(0.0)
    with torch.cuda.device(packs.device):
        rc = lib().vqhull_cuda_merge_candidates(packs.data_ptr(), nranks, rows, out.data_ptr(),
                                                C.byref(cnt), C.byref(fl),
                                                _stream_ptr(stream, packs.device))
    if rc == VQHULL_ERETRY:
        raise RetryWithFloor(fl.value)
    _check(rc, "vqhull_cuda_merge_candidates")
    return out[: cnt.value]


def hull_multi(xs, ys, shards: int) -> np.ndarray:
    """Single-process multi-GPU hull of host arrays (vqhull_cuda_hull_multi):
    ``shards`` contiguous shards over the visible devices, merged on device 0."""
    xs, ys = _f64(xs), _f64(ys)
    if xs.shape != ys.shape:
        raise ValueError("xs and ys differ in length")
    n = xs.size
    out = np.zeros(max(n, 1), dtype=np.uint64)
    cnt = C.c_uint64(0)
    rc = lib().vqhull_cuda_hull_multi(xs.ctypes.data_as(_dp), ys.ctypes.data_as(_dp), n, shards,
                                      out.ctypes.data_as(_u64p), C.byref(cnt))
    _check(rc, "vqhull_cuda_hull_multi")
    return out[: cnt.value].copy()


def find_extremes(x, y, stream=None) -> Tuple[int, int]:
    """find_extremes on device tensors -> (lo, hi).  Raises on empty input."""
    import torch
    _check_pair(x, y, "find_extremes")
    x, y = x.contiguous(), y.contiguous()
    lo, hi = C.c_uint64(), C.c_uint64()
    with torch.cuda.device(x.device):
        rc = lib().vqhull_cuda_find_extremes(x.data_ptr(), y.data_ptr(), x.numel(), C.byref(lo),
                                             C.byref(hi), _stream_ptr(stream, x.device))
    if rc == VQHULL_EINVAL and x.numel() == 0:
        raise ValueError("find_extremes: empty input")
    _check(rc, "vqhull_cuda_find_extremes")
    return lo.value, hi.value


@dataclass
class ExtractOutcome:
    """extract.hpp:19-24"""
    w_l: int
    w_r: int
    r1: Optional[Tuple[float, float]]
    r2: Optional[Tuple[float, float]]


def extract_subsets(x, y, edge_a, edge_b, stream=None) -> ExtractOutcome:
    """In-place fused partition + arg-max on device tensors (extract_subsets)."""
    import torch
    _check_pair(x, y, "extract_subsets", writable=True)
    ea = (C.c_double * 4)(*[float(v) for v in edge_a])
    eb = (C.c_double * 4)(*[float(v) for v in edge_b])
    wl, wr = C.c_uint64(), C.c_uint64()
    r1, r2 = (C.c_double * 2)(), (C.c_double * 2)()
    h1, h2 = C.c_int(), C.c_int()
    with torch.cuda.device(x.device):
        rc = lib().vqhull_cuda_extract_subsets(x.data_ptr(), y.data_ptr(), x.numel(), ea, eb,
                                               C.byref(wl), C.byref(wr), r1, C.byref(h1), r2,
                                               C.byref(h2), _stream_ptr(stream, x.device))
    _check(rc, "vqhull_cuda_extract_subsets")
    return ExtractOutcome(wl.value, wr.value, (r1[0], r1[1]) if h1.value else None,
                          (r2[0], r2[1]) if h2.value else None)


def stats() -> dict:
    s = Stats()
    _check(lib().vqhull_cuda_get_stats(C.byref(s)), "vqhull_cuda_get_stats")
    return s.as_dict()


def set_stable(on: bool) -> None:
    """Order-preserving (look-back) partition offsets instead of atomic claims."""
    _check(lib().vqhull_cuda_set_stable(int(bool(on))), "vqhull_cuda_set_stable")


def set_root_reference(on: bool) -> None:
    """Root stage without the octagon filter: find_extremes, bootstrap arg-max
    and the fused levels-1+2 pass.  Same hull either way."""
    _check(lib().vqhull_cuda_set_root_reference(int(bool(on))), "vqhull_cuda_set_root_reference")


def trim() -> None:
    """Release the engine's device buffers (they are re-allocated on demand)."""
    _check(lib().vqhull_cuda_trim(), "vqhull_cuda_trim")


ROOT_MODES = {"split": 0, "octagon": 1, "reference": 2}


def set_root_mode(mode: str) -> None:
    """Root stage: "split" (default: sampled octagon, filter pass, level 1 over
    the survivors), "octagon" (exact extremes pass + filtered level 1 in one
    pass) or "reference" (find_extremes, bootstrap, fused levels 1+2).  Same
    hull in every mode."""
    _check(lib().vqhull_cuda_set_root_mode(ROOT_MODES[mode]), "vqhull_cuda_set_root_mode")


FILTER_INNER = {"auto": -1, "box": 0, "octagon": 1, "disk": 2, "disk_only": 3}


def set_filter_inner(mode: str) -> None:
    """The filter pass's fast inner test: "auto" (default: the sample pass
    picks the largest region), or force "box", "octagon" or "disk".  Same
    hull (and, on ordinary inputs, the same survivors) in every mode."""
    _check(lib().vqhull_cuda_set_filter_inner(FILTER_INNER[mode]), "vqhull_cuda_set_filter_inner")


def set_timing(on: bool) -> None:
    _check(lib().vqhull_cuda_set_timing(int(bool(on))), "vqhull_cuda_set_timing")


# ---------------------------------------------------------------------------
# datasets (dataset.hpp:39-50 + the harness-defined square)
# ---------------------------------------------------------------------------
def generate(kind: str, n: int, seed: int, first: int = 0, threads: Optional[int] = None,
             out: Optional[Tuple] = None):
    """Points [first, first+n) of the (kind, seed) stream.

    ``out`` may be a pair of preallocated float64 buffers (numpy arrays or
    pinned CPU torch tensors); otherwise numpy arrays are returned.
    """
    if threads is None:
        threads = max(1, os.cpu_count() or 1)
    if out is None:
        xs = np.empty(n, dtype=np.float64)
        ys = np.empty(n, dtype=np.float64)
        px, py = xs.ctypes.data, ys.ctypes.data
    else:
        xs, ys = out
        px = xs.ctypes.data if isinstance(xs, np.ndarray) else xs.data_ptr()
        py = ys.ctypes.data if isinstance(ys, np.ndarray) else ys.data_ptr()
    rc = lib().vqhull_generate(KINDS[kind], seed, first, n, px, py, threads)
    _check(rc, "vqhull_generate")
    return xs, ys
