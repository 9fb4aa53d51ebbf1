"""Generates the golden vectors under tests/golden/ FROM THE REFERENCE ITSELF.

Runs only where /root/reference exists (this container): it drives
oracle/_ref/libvqhull_ref.so — the unmodified reference library compiled from
/root/reference/proj/src — and records its outputs.  The committed files are
then the fixtures every parity test (CPU oracle and GPU path) is held to.

    python tests/golden/make_golden.py            # small fixtures + configs 1-3
    python tests/golden/make_golden.py --config4  # + Kuzmin 1e9 (16 GB RAM)

Files:
  hull_cases.npz     named small instances with the reference's clockwise
                     first-occurrence index list (vqhull_compute) and vertex
                     coordinates (convex_hull)
  extract_cases.npz  extract_subsets instances: w_l, w_r, r1, r2 and the S1/S2
                     multisets (reference AVX-512/auto backend)
  generators.json    rng::at / uniform01 values and first generated points
  configs.json       BASELINE configs: h, FNV-1a-64 of the index list (u64 LE),
                     head/tail indices, reference byte model
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Oracle, Reference  # noqa: E402


def fnv1a64(idx: np.ndarray) -> str:
    return f"{Oracle().fnv1a64(idx):016x}"


def ref_indices(R: Reference, xs, ys) -> np.ndarray:
    rc, idx = R.compute(xs, ys)
    assert rc == 0
    return idx


def small_cases(R: Reference):
    rng = np.random.default_rng(20251020)
    cases = []

    def add(name, xs, ys):
        xs = np.asarray(xs, dtype=np.float64)
        ys = np.asarray(ys, dtype=np.float64)
        cases.append((name, xs, ys))

    # test_hull.cpp:71-115 degenerate hulls
    add("single", [0.0], [0.0])
    add("identical100", [3.0] * 100, [-4.0] * 100)
    add("two_points", [5.0, -2.0], [1.0, 7.0])
    add("collinear10", np.arange(10.0), np.arange(10.0))
    add("vertical7", [2.0] * 7, np.arange(7.0) - 3)
    # test_hull.cpp:117-130 unit square with center
    add("square_center", [1, 0, 0.5, 0, 1], [1, 0, 0.5, 1, 0])
    # test_hull.cpp:320-330 C ABI: index 5 duplicates index 0
    add("cabi_dup", [0, 4, 4, 0, 2, 0], [0, 0, 4, 4, 2, 0])
    # test_hull.cpp:220-240 deep recursion on a convex power-of-two curve
    i = np.arange(600)
    add("pow2_curve600", np.ldexp(1.0, i), np.ldexp(1.0, -i))
    # signed zeros and duplicates of extremes / apexes
    add("signed_zero", [0.0, -0.0, 1.0, -1.0, 0.0, -0.0, 0.0], [1.0, 1.0, 0.0, 0.0, -1.0, -1.0, 0.0])
    add("dup_extremes", [-1, -1, 1, 1, 0, 0, -1, 1], [0, 0, 0, 0, 1, 1, 0, 0])
    add("x_ties_lo_hi", [0, 0, 0, 5, 5, 5, 2], [1, -1, 0, 3, -3, 0, 9])
    # clustered integer instances (test_hull.cpp:162-179 style, own seeds)
    for k in range(60):
        n = int(rng.integers(1, 201))
        add(f"int4_{k}", rng.integers(-4, 5, n), rng.integers(-4, 5, n))
    for k in range(30):
        n = int(rng.integers(1, 2001))
        add(f"int500_{k}", rng.integers(-500, 501, n), rng.integers(-500, 501, n))
    for k in range(30):
        n = int(rng.integers(50, 850))
        add(f"dbl_{k}", rng.uniform(-1, 1, n), rng.uniform(-1, 1, n))
    for k in range(10):
        n = int(rng.integers(100, 3000))
        t = rng.uniform(0, 2 * np.pi, n)
        add(f"circle_{k}", np.cos(t), np.sin(t))
    # exact-on-circle integer lattice points + interior points
    pts = [(x, y) for x in range(-25, 26) for y in range(-25, 26) if x * x + y * y == 625]
    add("lattice_circle", [p[0] for p in pts] * 2 + [0, 1, 2], [p[1] for p in pts] * 2 + [0, 1, 2])
    # larger segments (exercise the tiled level kernel, > 256 points per side)
    for k in range(6):
        n = int(rng.integers(5000, 40000))
        if k % 2:
            t = rng.uniform(0, 2 * np.pi, n)
            add(f"big_circle_{k}", np.cos(t), np.sin(t))
        else:
            add(f"big_int_{k}", rng.integers(-2000, 2001, n), rng.integers(-2000, 2001, n))

    names, off, xs_all, ys_all, ioff, idx_all, hx_all, hy_all = [], [0], [], [], [0], [], [], []
    for name, xs, ys in cases:
        idx = ref_indices(R, xs, ys)
        hx, hy = R.convex_hull(xs, ys)
        # the index list must point at the coordinates convex_hull returned
        assert np.array_equal(xs[idx.astype(np.int64)], hx) and np.array_equal(ys[idx.astype(np.int64)], hy)
        names.append(name)
        xs_all.append(xs)
        ys_all.append(ys)
        off.append(off[-1] + xs.size)
        idx_all.append(idx)
        hx_all.append(hx)
        hy_all.append(hy)
        ioff.append(ioff[-1] + idx.size)
    np.savez_compressed(
        os.path.join(HERE, "hull_cases.npz"),
        names=np.array(names), off=np.array(off, dtype=np.int64),
        xs=np.concatenate(xs_all), ys=np.concatenate(ys_all),
        ioff=np.array(ioff, dtype=np.int64), idx=np.concatenate(idx_all).astype(np.uint64),
        hx=np.concatenate(hx_all), hy=np.concatenate(hy_all))
    print(f"hull_cases: {len(names)} cases")


def extract_cases(R: Reference):
    rng = np.random.default_rng(808)
    recs = []
    # test_extract.cpp:183-210 golden eight points
    recs.append(("eight_points", [1, 2, 3, 1, 0.5, 2, 3, 2.5], [1, -1, 2, 0, -3, 4, 0, -0.5],
                 [0, 0, 4, 0], [4, 0, 0, 0]))
    for k in range(40):  # test_extract.cpp:212-225 style
        n = int(rng.integers(0, 4097))
        recs.append((f"int1000_{k}", rng.integers(-1000, 1001, n), rng.integers(-1000, 1001, n),
                     [-900, -11, 850, 17], [850, 17, -900, -11]))
    for k in range(60):  # test_extract.cpp:227-242: tiny, duplicate-heavy, skew edges
        n = int(rng.integers(0, 40))
        p = rng.integers(-6, 7, 2)
        q = rng.integers(-6, 7, 2)
        recs.append((f"tiny_{k}", rng.integers(-6, 7, n), rng.integers(-6, 7, n),
                     [p[0], p[1], q[0], q[1]], [q[0], q[1], p[0], p[1]]))
    for k in range(20):  # two edges sharing an apex (the recursion's own shape)
        n = int(rng.integers(100, 6000))
        xs, ys = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        a = rng.uniform(-1, 1, 2)
        r = rng.uniform(-1, 1, 2) * 1.5
        b = rng.uniform(-1, 1, 2)
        recs.append((f"apex_{k}", xs, ys, [a[0], a[1], r[0], r[1]], [r[0], r[1], b[0], b[1]]))
    names, off, X, Y, E, WL, WR, R1, R2, HAS = [], [0], [], [], [], [], [], [], [], []
    s1o, s2o, S1, S2 = [0], [0], [], []
    for name, xs, ys, ea, eb in recs:
        xs = np.asarray(xs, dtype=np.float64)
        ys = np.asarray(ys, dtype=np.float64)
        ox, oy, wl, wr, r1, r2 = R.extract_subsets(xs, ys, np.asarray(ea, float), np.asarray(eb, float))
        s1 = sorted(zip(ox[:wl], oy[:wl]))
        s2 = sorted(zip(ox[wr:], oy[wr:]))
        names.append(name)
        X.append(xs)
        Y.append(ys)
        off.append(off[-1] + xs.size)
        E.append(list(map(float, ea)) + list(map(float, eb)))
        WL.append(wl)
        WR.append(wr)
        HAS.append([r1 is not None, r2 is not None])
        R1.append(r1 if r1 else (0.0, 0.0))
        R2.append(r2 if r2 else (0.0, 0.0))
        S1.append(np.array(s1, dtype=np.float64).reshape(-1, 2))
        S2.append(np.array(s2, dtype=np.float64).reshape(-1, 2))
        s1o.append(s1o[-1] + len(s1))
        s2o.append(s2o[-1] + len(s2))
    np.savez_compressed(
        os.path.join(HERE, "extract_cases.npz"), names=np.array(names),
        off=np.array(off, dtype=np.int64), xs=np.concatenate(X), ys=np.concatenate(Y),
        edges=np.array(E), w_l=np.array(WL, dtype=np.int64), w_r=np.array(WR, dtype=np.int64),
        has=np.array(HAS, dtype=bool), r1=np.array(R1), r2=np.array(R2),
        s1off=np.array(s1o, dtype=np.int64), s2off=np.array(s2o, dtype=np.int64),
        s1=np.concatenate(S1), s2=np.concatenate(S2))
    print(f"extract_cases: {len(names)} cases")


def generators(R: Reference):
    out = {"rng_at": [], "uniform01": [], "first_points": {}}
    for seed, idx in [(42, 0), (42, 1), (7, 123456789), (1, 0), (5, 7999999999)]:
        out["rng_at"].append([seed, idx, str(R.rng_at(seed, idx))])
        out["uniform01"].append([seed, idx, R.uniform01(seed, idx).hex()])
    for kind in ("disk", "circle", "kuzmin"):
        xs, ys = R.generate(kind, 4, 42, workers=1)
        out["first_points"][kind] = [[float(x).hex(), float(y).hex()] for x, y in zip(xs, ys)]
    # the constants of the reference's own test (test_dataset_io.cpp:40-47)
    out["reference_test_constants"] = {
        "rng_at_42_0": "13679457532755275413",
        "rng_at_42_1": "2949826092126892291",
        "rng_at_7_123456789": "12208133997311326809",
    }
    with open(os.path.join(HERE, "generators.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("generators.json written")


CONFIGS = [
    # name, kind, n, seed  (BASELINE.json configs; "square" is harness-defined)
    ("config1_disk_1e6_s1", "disk", 10**6, 1),
    ("config2_square_1e8_s2", "square", 10**8, 2),
    ("config3_circle_1e7_s3", "circle", 10**7, 3),
    ("config4_kuzmin_1e9_s4", "kuzmin", 10**9, 4),
    ("config5_proxy_disk_4e7_s5", "disk", 4 * 10**7, 5),
]


def gen_points(R: Reference, kind, n, seed):
    if kind == "square":
        # harness-defined: x = 2u(2i)-1, y = 2u(2i+1)-1 with the reference RNG;
        # built with numpy from the reference's own uniform01 of a few points
        # is too slow, so the product generator is used and cross-checked here
        import paper_2510_09417_b200 as vq
        xs, ys = vq.generate("square", n, seed)
        for i in (0, 1, n // 2, n - 1):
            assert xs[i] == 2.0 * R.uniform01(seed, 2 * i) - 1.0
            assert ys[i] == 2.0 * R.uniform01(seed, 2 * i + 1) - 1.0
        return xs, ys
    return R.generate(kind, n, seed, workers=8)


def first_occurrence(xs, ys, hx, hy) -> np.ndarray:
    """vqhull_c.cpp:46-61 semantics for small h, independent of the oracle."""
    out = np.empty(hx.size, dtype=np.uint64)
    for v in range(hx.size):
        out[v] = np.flatnonzero((xs == hx[v]) & (ys == hy[v]))[0]
    return out


def configs(R: Reference, with4: bool):
    path = os.path.join(HERE, "configs.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for name, kind, n, seed in CONFIGS:
        if name.startswith("config4") and not with4:
            continue
        xs, ys = gen_points(R, kind, n, seed)
        if n <= 10**7:
            idx = ref_indices(R, xs, ys)           # the reference C ABI itself
            mb, ncalls, h = R.trace_hull(xs, ys)
        else:
            hx, hy = R.convex_hull(xs, ys, workers=8, cap=1 << 20)
            idx = first_occurrence(xs, ys, hx, hy)
            mb, ncalls, h = (R.trace_hull(xs, ys) if n <= 10**8 else (None, None, hx.size))
        data[name] = {
            "kind": kind, "n": n, "seed": seed, "h": int(idx.size), "fnv1a64_u64le": fnv1a64(idx),
            "head": [int(v) for v in idx[:8]], "tail": [int(v) for v in idx[-8:]],
            "model_bytes": None if mb is None else int(mb),
            "ref_calls": None if ncalls is None else int(ncalls),
            "first_point": [float(xs[0]).hex(), float(ys[0]).hex()],
        }
        if idx.size <= 100000:
            data[name]["indices"] = [int(v) for v in idx]
        print(name, data[name]["h"], data[name]["fnv1a64_u64le"], flush=True)
        with open(path, "w") as f:
            json.dump(data, f, indent=1)
        del xs, ys


if __name__ == "__main__":
    R = Reference()
    if "--configs-only" not in sys.argv:
        small_cases(R)
        extract_cases(R)
        generators(R)
    configs(R, "--config4" in sys.argv)
