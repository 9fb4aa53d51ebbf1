"""TEST INFRASTRUCTURE — ctypes front-ends for the CPU checkers.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference /
cpu_baseline legs may import this package.  The product package
(``paper_2510_09417_b200``) never does.

* ``Oracle``    — our plain-C restatement (``oracle/vqhull_oracle.c``).
* ``Reference`` — the unmodified reference library compiled from
  ``/root/reference/proj/src`` (``oracle/_ref/libvqhull_ref.so``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle_vqhull.so")
REF_SO = os.path.join(HERE, "_ref", "libvqhull_ref.so")

_dp = C.POINTER(C.c_double)
_sz = C.POINTER(C.c_size_t)
_u64p = C.POINTER(C.c_uint64)
_ip = C.POINTER(C.c_int)

# DatasetKind order of the reference (dataset.hpp:12)
KIND = {"kuzmin": 0, "circle": 1, "disk": 2}


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def build(reference: bool = True) -> None:
    """Compile the oracle (and the reference when its sources are present)."""
    import subprocess

    targets = ["oracle"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(reference=False)
        L = self.lib = C.CDLL(path)
        L.oracle_find_extremes.argtypes = [_dp, _dp, C.c_size_t, _sz, _sz]
        L.oracle_extract_subsets.argtypes = [_dp, _dp, C.c_size_t, _dp, _dp, _sz, _sz,
                                             _dp, _ip, _dp, _ip]
        L.oracle_convex_hull.argtypes = [_dp, _dp, C.c_size_t, _dp, _dp, _sz]
        L.oracle_trace_hull.argtypes = [_dp, _dp, C.c_size_t, _u64p, C.c_size_t, _sz,
                                        _u64p, _sz]
        L.oracle_compute.argtypes = [_dp, _dp, C.c_size_t, C.c_int, _u64p, _sz]
        L.oracle_fnv1a64_u64.argtypes = [_u64p, C.c_size_t]
        L.oracle_fnv1a64_u64.restype = C.c_uint64

    def find_extremes(self, xs, ys):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        lo, hi = C.c_size_t(), C.c_size_t()
        if self.lib.oracle_find_extremes(px, py, len(xs), C.byref(lo), C.byref(hi)):
            raise ValueError("find_extremes: empty input")
        return lo.value, hi.value

    def extract_subsets(self, xs, ys, edge_a, edge_b):
        """In place on copies; returns (xs, ys, w_l, w_r, r1|None, r2|None)."""
        xs = np.array(xs, dtype=np.float64, copy=True)
        ys = np.array(ys, dtype=np.float64, copy=True)
        ea, pa = _f64(edge_a)
        eb, pb = _f64(edge_b)
        wl, wr = C.c_size_t(), C.c_size_t()
        r1, r2 = (C.c_double * 2)(), (C.c_double * 2)()
        h1, h2 = C.c_int(), C.c_int()
        rc = self.lib.oracle_extract_subsets(xs.ctypes.data_as(_dp), ys.ctypes.data_as(_dp),
                                             len(xs), pa, pb, C.byref(wl), C.byref(wr),
                                             r1, C.byref(h1), r2, C.byref(h2))
        assert rc == 0
        return (xs, ys, wl.value, wr.value, (r1[0], r1[1]) if h1.value else None,
                (r2[0], r2[1]) if h2.value else None)

    def convex_hull(self, xs, ys):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        ox = np.empty(max(n, 1))
        oy = np.empty(max(n, 1))
        cnt = C.c_size_t()
        assert self.lib.oracle_convex_hull(px, py, n, ox.ctypes.data_as(_dp),
                                           oy.ctypes.data_as(_dp), C.byref(cnt)) == 0
        return ox[: cnt.value].copy(), oy[: cnt.value].copy()

    def trace_hull(self, xs, ys):
        """(model_bytes, n_calls, hull_size, calls[k,4])"""
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        cap = n + 2
        calls = np.zeros((cap, 4), dtype=np.uint64)
        ncalls, hs = C.c_size_t(), C.c_size_t()
        mb = C.c_uint64()
        assert self.lib.oracle_trace_hull(px, py, n, calls.ctypes.data_as(_u64p), cap,
                                          C.byref(ncalls), C.byref(mb), C.byref(hs)) == 0
        return mb.value, ncalls.value, hs.value, calls[: ncalls.value]

    def compute(self, xs, ys, workers: int = 1):
        """vqhull_compute semantics: (rc, indices as uint64 array)."""
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        out = np.zeros(max(n, 1), dtype=np.uint64)
        cnt = C.c_size_t()
        rc = self.lib.oracle_compute(px, py, n, workers, out.ctypes.data_as(_u64p),
                                     C.byref(cnt))
        return rc, out[: cnt.value].copy()

    def hull_indices(self, xs, ys):
        rc, idx = self.compute(xs, ys)
        if rc:
            raise ValueError("invalid input")
        return idx

    def fnv1a64(self, idx) -> int:
        a = np.ascontiguousarray(idx, dtype=np.uint64)
        return int(self.lib.oracle_fnv1a64_u64(a.ctypes.data_as(_u64p), len(a)))


class Reference:
    """The reference library itself (present only where oracle/_ref was built)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_convex_hull.argtypes = [_dp, _dp, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                      C.c_int, _dp, _dp, C.c_size_t, _sz]
        L.ref_bench_hull.argtypes = [_dp, _dp, C.c_size_t, C.c_int, C.c_int, _dp, _sz]
        L.ref_find_extremes.argtypes = [_dp, _dp, C.c_size_t, _sz, _sz]
        L.ref_extract_subsets.argtypes = [_dp, _dp, C.c_size_t, _dp, _dp, C.c_int, C.c_int,
                                          _sz, _sz, _dp, _ip, _dp, _ip]
        L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int, _dp, _dp]
        L.ref_generate_square.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _dp, _dp]
        L.ref_scale_baseline.argtypes = [C.c_uint64, C.c_int, C.c_int]
        L.ref_scale_baseline.restype = C.c_double
        L.ref_rng_at.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_rng_at.restype = C.c_uint64
        L.ref_uniform01.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_uniform01.restype = C.c_double
        L.ref_trace_hull.argtypes = [_dp, _dp, C.c_size_t, _u64p, _sz, _sz, _u64p, C.c_size_t]
        L.ref_monotone_chain.argtypes = [_dp, _dp, C.c_size_t, _dp, _dp, _sz]
        L.vqhull_compute.argtypes = [_dp, _dp, C.c_size_t, C.c_int, _sz, _sz]
        L.ref_hw_threads.restype = C.c_uint

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def hw_threads(self) -> int:
        return int(self.lib.ref_hw_threads())

    def convex_hull(self, xs, ys, workers=1, lanes=8, portable=False, max_depth=512,
                    cap=None):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        cap = max(n, 1) if cap is None else cap
        ox = np.empty(cap)
        oy = np.empty(cap)
        cnt = C.c_size_t()
        rc = self.lib.ref_convex_hull(px, py, n, workers, lanes, int(portable), max_depth,
                                      ox.ctypes.data_as(_dp), oy.ctypes.data_as(_dp), cap,
                                      C.byref(cnt))
        assert rc == 0, f"ref_convex_hull rc={rc} (h={cnt.value}, cap={cap})"
        return ox[: cnt.value].copy(), oy[: cnt.value].copy()

    def bench_hull(self, xs, ys, workers, reps):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        secs = np.zeros(reps)
        hs = C.c_size_t()
        assert self.lib.ref_bench_hull(px, py, len(xs), workers, reps,
                                       secs.ctypes.data_as(_dp), C.byref(hs)) == 0
        return secs, hs.value

    def find_extremes(self, xs, ys):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        lo, hi = C.c_size_t(), C.c_size_t()
        if self.lib.ref_find_extremes(px, py, len(xs), C.byref(lo), C.byref(hi)):
            raise ValueError("find_extremes: empty input")
        return lo.value, hi.value

    def extract_subsets(self, xs, ys, edge_a, edge_b, lanes=8, portable=False):
        xs = np.array(xs, dtype=np.float64, copy=True)
        ys = np.array(ys, dtype=np.float64, copy=True)
        ea, pa = _f64(edge_a)
        eb, pb = _f64(edge_b)
        wl, wr = C.c_size_t(), C.c_size_t()
        r1, r2 = (C.c_double * 2)(), (C.c_double * 2)()
        h1, h2 = C.c_int(), C.c_int()
        rc = self.lib.ref_extract_subsets(xs.ctypes.data_as(_dp), ys.ctypes.data_as(_dp),
                                          len(xs), pa, pb, lanes, int(portable),
                                          C.byref(wl), C.byref(wr), r1, C.byref(h1), r2,
                                          C.byref(h2))
        assert rc == 0
        return (xs, ys, wl.value, wr.value, (r1[0], r1[1]) if h1.value else None,
                (r2[0], r2[1]) if h2.value else None)

    def generate(self, kind: str, n: int, seed: int, workers: int = 8):
        xs = np.empty(n)
        ys = np.empty(n)
        assert self.lib.ref_generate(KIND[kind], n, seed, workers, xs.ctypes.data_as(_dp),
                                     ys.ctypes.data_as(_dp)) == 0
        return xs, ys

    def generate_square(self, n: int, seed: int, first: int = 0, workers: int = 8):
        """BASELINE config 2's square from the reference's own RNG
        (rng::uniform01, dataset.cpp:32-50): x = 2U(2k)-1, y = 2U(2k+1)-1."""
        xs = np.empty(n)
        ys = np.empty(n)
        assert self.lib.ref_generate_square(seed, first, n, workers, xs.ctypes.data_as(_dp),
                                            ys.ctypes.data_as(_dp)) == 0
        return xs, ys

    def generate_any(self, kind: str, n: int, seed: int, workers: int = 8):
        """Points [0, n) of any BASELINE kind, generated by the reference."""
        if kind == "square":
            return self.generate_square(n, seed, 0, workers)
        return self.generate(kind, n, seed, workers)

    def scale_baseline(self, workers: int, reps: int = 5, buffer_bytes: int = 0) -> float:
        """stream_scale_baseline (bench.cpp:33-74): in-place a[i] = s*a[i],
        best-of-reps GB/s at 16 B per element; default buffer 4x the LLC."""
        return float(self.lib.ref_scale_baseline(buffer_bytes, reps, workers))

    def rng_at(self, seed, index) -> int:
        return int(self.lib.ref_rng_at(seed, index))

    def uniform01(self, seed, index) -> float:
        return float(self.lib.ref_uniform01(seed, index))

    def trace_hull(self, xs, ys):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        mb = C.c_uint64()
        nc, hs = C.c_size_t(), C.c_size_t()
        assert self.lib.ref_trace_hull(px, py, len(xs), C.byref(mb), C.byref(nc),
                                       C.byref(hs), None, 0) == 0
        return mb.value, nc.value, hs.value

    def monotone_chain(self, xs, ys):
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        ox = np.empty(max(n, 1))
        oy = np.empty(max(n, 1))
        cnt = C.c_size_t()
        assert self.lib.ref_monotone_chain(px, py, n, ox.ctypes.data_as(_dp),
                                           oy.ctypes.data_as(_dp), C.byref(cnt)) == 0
        return ox[: cnt.value].copy(), oy[: cnt.value].copy()

    def compute(self, xs, ys, workers=1, cap=None):
        """The reference's own vqhull_compute.  It writes only the h hull
        indices (vqhull_c.cpp:51-61), so for huge inputs with a known small
        hull `cap` bounds the output buffer instead of n entries."""
        xs, px = _f64(xs)
        ys, py = _f64(ys)
        n = len(xs)
        out = np.zeros(max(min(n, cap) if cap else n, 1), dtype=np.uint64)
        cnt = C.c_size_t()
        rc = self.lib.vqhull_compute(px, py, n, workers,
                                     out.ctypes.data_as(_sz), C.byref(cnt))
        assert cnt.value <= out.size, "hull larger than the output cap"
        return rc, out[: cnt.value].copy()
