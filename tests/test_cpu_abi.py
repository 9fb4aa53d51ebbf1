"""CPU: the product library loads, exports every symbol include/vqhull_b200.h
declares, and its host-side logic (argument checks, generators) matches the
reference — no compute call needs a GPU here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import golden_io as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "vqhull_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vqhull_\w+)\s*\(", txt)))


def test_library_exports_header(vq):
    syms = header_symbols()
    assert "vqhull_compute" in syms and "vqhull_cuda_hull" in syms
    L = vq.lib()
    for s in syms:
        assert hasattr(L, s), f"{s} not exported"


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2510_09417_b200", "lib", "libvqhull_b200.so")
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_vqhull_compute_argument_checks(vq):
    """vqhull_c.cpp:29-34, checked before any device work."""
    L = vq.lib()
    dp = C.POINTER(C.c_double)
    szp = C.POINTER(C.c_size_t)
    xs = np.array([0.0, 1.0])
    idx = np.zeros(2, dtype=np.uint64)
    cnt = C.c_size_t(7)
    px, py = xs.ctypes.data_as(dp), xs.ctypes.data_as(dp)
    pi = idx.ctypes.data_as(szp)
    assert L.vqhull_compute(px, py, 2, 1, pi, None) == 1          # out_count NULL
    assert L.vqhull_compute(px, py, 2, 0, pi, C.byref(cnt)) == 1  # workers < 1
    assert cnt.value == 7                                          # untouched, as in the reference
    cnt.value = 7
    assert L.vqhull_compute(None, None, 0, 1, None, C.byref(cnt)) == 0  # empty input
    assert cnt.value == 0
    assert L.vqhull_compute(None, py, 2, 1, pi, C.byref(cnt)) == 1  # NULL array with n > 0
    assert L.vqhull_compute(px, py, 2, 1, None, C.byref(cnt)) == 1


def test_generators_match_reference_golden(vq):
    g = G.generators()
    for kind, pts in g["first_points"].items():
        xs, ys = vq.generate(kind, 4, 42, threads=1)
        assert [[float(x).hex(), float(y).hex()] for x, y in zip(xs, ys)] == pts
    # the constants written in the reference's own test, test_dataset_io.cpp:40-43
    consts = g["reference_test_constants"]
    got = {f"rng_at_{s}_{i}": v for s, i, v in g["rng_at"]}
    for k, v in consts.items():
        assert got[k] == v


def test_generator_sharding_is_counter_based(vq):
    xs, ys = vq.generate("disk", 100_000, 5, threads=4)
    a, b = vq.generate("disk", 1000, 5, first=50_000, threads=1)
    assert np.array_equal(a, xs[50_000:51_000]) and np.array_equal(b, ys[50_000:51_000])


def test_generator_matches_reference_live(vq, reference):
    for kind in ("disk", "circle", "kuzmin"):
        a = vq.generate(kind, 70_000, 3)
        b = reference.generate(kind, 70_000, 3)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_square_is_exact_affine_of_reference_rng(vq, reference):
    xs, ys = vq.generate("square", 1000, 2)
    for i in (0, 1, 999):
        assert xs[i] == 2.0 * reference.uniform01(2, 2 * i) - 1.0
        assert ys[i] == 2.0 * reference.uniform01(2, 2 * i + 1) - 1.0


def test_no_cpu_fallback_without_gpu(vq):
    """The product path fails loudly when no device is present."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    rc, _ = vq.vqhull_compute([0.0, 1.0, 0.5], [0.0, 0.0, 1.0])
    assert rc == vq.VQHULL_ECUDA
