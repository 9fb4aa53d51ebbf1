"""CPU: pin the oracle (our C restatement) to the reference.

Against (a) the committed golden vectors produced by the reference library
itself and (b) the reference library run live (oracle/_ref) when present.
Mirrors proj/tests/test_geometry.cpp, test_extract.cpp, test_hull.cpp,
test_dataset_io.cpp and test_bench.cpp.
"""
import os

import numpy as np
import pytest

import golden_io as G


# --- test_geometry.cpp:32-51 find_extremes tie-breaks --------------------------
def test_find_extremes_examples(oracle):
    assert oracle.find_extremes([0.0], [0.0]) == (0, 0)
    assert oracle.find_extremes([1, -2, 3], [5, 0, 1]) == (1, 2)
    assert oracle.find_extremes([0, 0, 0], [1, -1, 0]) == (1, 0)
    with pytest.raises(ValueError):
        oracle.find_extremes([], [])


def test_find_extremes_vs_reference(oracle, reference):
    rng = np.random.default_rng(11)
    for _ in range(300):
        n = int(rng.integers(1, 500))
        xs = rng.integers(-3, 4, n).astype(float)
        ys = rng.integers(-3, 4, n).astype(float)
        assert oracle.find_extremes(xs, ys) == reference.find_extremes(xs, ys)


# --- test_extract.cpp:183-242 --------------------------------------------------
@pytest.mark.parametrize("case", G.extract_cases(), ids=lambda c: c["name"])
def test_extract_golden(oracle, case):
    ox, oy, wl, wr, r1, r2 = oracle.extract_subsets(case["xs"], case["ys"], case["ea"], case["eb"])
    assert (wl, wr) == (case["w_l"], case["w_r"])
    assert r1 == case["r1"] and r2 == case["r2"]
    assert np.array_equal(G.sorted_pairs(ox[:wl], oy[:wl]), G.sorted_pairs(*case["s1"].T))
    assert np.array_equal(G.sorted_pairs(ox[wr:], oy[wr:]), G.sorted_pairs(*case["s2"].T))


def test_eight_point_example(oracle):
    xs = [1, 2, 3, 1, 0.5, 2, 3, 2.5]
    ys = [1, -1, 2, 0, -3, 4, 0, -0.5]
    _, _, wl, wr, r1, r2 = oracle.extract_subsets(xs, ys, [0, 0, 4, 0], [4, 0, 0, 0])
    assert (wl, wr, r1, r2) == (3, 5, (2.0, 4.0), (0.5, -3.0))


# --- test_hull.cpp -------------------------------------------------------------
@pytest.mark.parametrize("case", G.hull_cases(), ids=lambda c: c[0])
def test_hull_golden(oracle, case):
    name, xs, ys, idx, hx, hy = case
    rc, got = oracle.compute(xs, ys)
    assert rc == 0
    assert np.array_equal(got, idx)
    cx, cy = oracle.convex_hull(xs, ys)
    assert np.array_equal(cx, hx) and np.array_equal(cy, hy)


def test_compute_argument_errors(oracle):
    assert oracle.compute([], [])[0] == 0
    assert oracle.compute([0.0, np.nan], [0.0, 1.0])[0] == 1
    assert oracle.compute([0.0, np.inf], [0.0, 1.0])[0] == 1
    assert oracle.compute([0.0, 1.0], [0.0, 1.0], workers=0)[0] == 1


def test_oracle_vs_reference_random(oracle, reference):
    rng = np.random.default_rng(4242)
    for it in range(400):
        n = int(rng.integers(0, 400))
        k = it % 4
        if k == 0:
            xs = rng.integers(-4, 5, n).astype(float); ys = rng.integers(-4, 5, n).astype(float)
        elif k == 1:
            xs = rng.uniform(-1, 1, n); ys = rng.uniform(-1, 1, n)
        elif k == 2:
            t = rng.uniform(0, 2 * np.pi, n); xs = np.cos(t); ys = np.sin(t)
        else:
            xs = rng.integers(-10**6, 10**6, n).astype(float); ys = rng.integers(-10**6, 10**6, n).astype(float)
        a, b = oracle.compute(xs, ys), reference.compute(xs, ys)
        assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_monotone_chain_agrees_on_integers(oracle, reference):
    # bench.cpp:288-318: on the exactness envelope the hull equals monotone chain
    rng = np.random.default_rng(99)
    for _ in range(100):
        n = int(rng.integers(1, 300))
        xs = rng.integers(-50, 51, n).astype(float)
        ys = rng.integers(-50, 51, n).astype(float)
        hx, hy = oracle.convex_hull(xs, ys)
        mx, my = reference.monotone_chain(xs, ys)
        assert np.array_equal(hx, mx) and np.array_equal(hy, my)


# --- test_bench.cpp:36-54 byte model ------------------------------------------
def test_byte_model_identical_points(oracle):
    n = 100
    mb, ncalls, h, calls = oracle.trace_hull(np.full(n, 2.0), np.full(n, 3.0))
    assert (h, ncalls) == (1, 1)
    assert mb == 24 * n


def test_byte_model_matches_reference(oracle, reference):
    rng = np.random.default_rng(5)
    for _ in range(10):
        n = int(rng.integers(1, 20000))
        xs, ys = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        mb, ncalls, h, _ = oracle.trace_hull(xs, ys)
        assert (mb, ncalls, h) == reference.trace_hull(xs, ys)


# --- configs (BASELINE.json), golden index lists ------------------------------
@pytest.mark.parametrize("name", ["config1_disk_1e6_s1", "config5_proxy_disk_4e7_s5"])
def test_oracle_config_golden(oracle, vq, name):
    cfg = G.configs()[name]
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    assert [float(xs[0]).hex(), float(ys[0]).hex()] == cfg["first_point"]
    idx = oracle.hull_indices(xs, ys)
    assert idx.size == cfg["h"]
    assert f"{oracle.fnv1a64(idx):016x}" == cfg["fnv1a64_u64le"]
    if "indices" in cfg:
        assert idx.tolist() == cfg["indices"]


def test_config5_global_golden_index_mapping(oracle, reference):
    """tests/golden/make_config5_global.py maps the reference's hull
    coordinates to first input indices by a scan; on a small input with
    duplicates it equals the reference mapping (vqhull_c.cpp:46-61)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_config5_global import first_occurrence

    xs, ys = reference.generate("disk", 50_000, 5, 4)
    xs[-50:], ys[-50:] = xs[:50], ys[:50]
    xs[7], ys[7] = -0.0 * xs[7], ys[7]  # (a signed zero never matters here; the scan uses ==)
    hx, hy = reference.convex_hull(xs, ys, workers=2)
    got = first_occurrence(xs, ys, hx, hy, chunk=1 << 12)
    rc, ref = reference.compute(xs, ys)
    assert rc == 0 and np.array_equal(got, ref)
