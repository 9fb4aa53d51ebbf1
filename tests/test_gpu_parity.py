"""GPU parity: the sm_100a path, called through the C ABI, against the golden
vectors (produced by the reference) and the oracle run live on the same
seeded inputs.  Bit-exact index lists; integer/index work has no tolerance.

Mirrors proj/tests/test_hull.cpp, test_extract.cpp, test_geometry.cpp and the
acceptance criteria C1/C4/C8 (acceptance.cpp:63-82, 182-208, 337-371).
"""
import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


def dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def gpu_indices(vq, xs, ys):
    return vq.hull_device(dev(xs), dev(ys)).cpu().numpy().astype(np.uint64)


# --- C ABI (host arrays) on every golden hull case -----------------------------
@pytest.mark.parametrize("case", G.hull_cases(), ids=lambda c: c[0])
def test_vqhull_compute_golden(vq, cuda, case):
    name, xs, ys, idx, hx, hy = case
    rc, got = vq.vqhull_compute(xs, ys)
    assert rc == 0
    assert np.array_equal(got, idx), f"{name}: {got[:10]} vs {idx[:10]}"


@pytest.mark.parametrize("case", G.hull_cases()[::3], ids=lambda c: c[0])
def test_device_hull_golden(vq, cuda, case):
    name, xs, ys, idx, hx, hy = case
    got = gpu_indices(vq, xs, ys)
    assert np.array_equal(got, idx)
    poly = vq.convex_hull(xs, ys)
    assert np.array_equal(poly.xs, hx) and np.array_equal(poly.ys, hy)


def test_u32_device_output(vq, cuda):
    xs, ys = vq.generate("disk", 200_000, 9)
    ref = gpu_indices(vq, xs, ys)
    got = vq.hull_device(dev(xs), dev(ys), u32=True).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, ref)


# --- test_hull.cpp:320-345: C ABI semantics and errors ------------------------
def test_cabi_duplicates_and_errors(vq, cuda):
    rc, idx = vq.vqhull_compute([0, 4, 4, 0, 2, 0], [0, 0, 4, 4, 2, 0])
    assert rc == 0 and idx.tolist() == [0, 3, 2, 1]
    assert vq.vqhull_compute([], [])[0] == 0
    assert vq.vqhull_compute([0.0, np.nan], [0.0, 1.0])[0] == 1
    assert vq.vqhull_compute([0.0, 1.0, 2.0], [0.0, -np.inf, 1.0])[0] == 1
    assert vq.vqhull_compute([0.0, 1.0], [0.0, 1.0], workers=0)[0] == 1
    # the engine is still healthy after a rejected call
    rc, idx = vq.vqhull_compute([1, 0, 0.5, 0, 1], [1, 0, 0.5, 1, 0])
    assert rc == 0 and idx.tolist() == [1, 3, 0, 4]


# --- find_extremes (test_geometry.cpp:32-51) -----------------------------------
def test_find_extremes(vq, cuda, oracle):
    assert vq.find_extremes(dev([0.0]), dev([0.0])) == (0, 0)
    assert vq.find_extremes(dev([1, -2, 3]), dev([5, 0, 1])) == (1, 2)
    assert vq.find_extremes(dev([0, 0, 0]), dev([1, -1, 0])) == (1, 0)
    with pytest.raises(ValueError):
        vq.find_extremes(dev([]), dev([]))
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 300000))
        xs = rng.integers(-30, 31, n).astype(float)
        ys = rng.integers(-30, 31, n).astype(float)
        assert vq.find_extremes(dev(xs), dev(ys)) == oracle.find_extremes(xs, ys)
    # misaligned (odd offset) device pointer takes the scalar-load path
    xs, ys = rng.uniform(-1, 1, 100001), rng.uniform(-1, 1, 100001)
    X, Y = dev(xs), dev(ys)
    assert vq.find_extremes(X[1:], Y[1:]) == oracle.find_extremes(xs[1:], ys[1:])


# --- extract_subsets (test_extract.cpp:183-299) --------------------------------
@pytest.mark.parametrize("case", G.extract_cases(), ids=lambda c: c["name"])
def test_extract_golden(vq, cuda, case):
    X, Y = dev(case["xs"]), dev(case["ys"])
    out = vq.extract_subsets(X, Y, case["ea"], case["eb"])
    assert (out.w_l, out.w_r) == (case["w_l"], case["w_r"])
    assert out.r1 == case["r1"] and out.r2 == case["r2"]
    x, y = X.cpu().numpy(), Y.cpu().numpy()
    assert np.array_equal(G.sorted_pairs(x[:out.w_l], y[:out.w_l]), G.sorted_pairs(*case["s1"].T))
    assert np.array_equal(G.sorted_pairs(x[out.w_r:], y[out.w_r:]), G.sorted_pairs(*case["s2"].T))


def test_extract_large_vs_oracle(vq, cuda, oracle):
    """Multi-tile segments: the decoupled look-back must give the same sets/r."""
    rng = np.random.default_rng(17)
    for n in (4095, 4096, 4097, 100_000, 1_000_003):
        xs, ys = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        ea, eb = [-1.0, -0.2, 0.3, 1.4], [0.3, 1.4, 1.0, 0.1]
        ox, oy, wl, wr, r1, r2 = oracle.extract_subsets(xs, ys, ea, eb)
        X, Y = dev(xs), dev(ys)
        out = vq.extract_subsets(X, Y, ea, eb)
        assert (out.w_l, out.w_r, out.r1, out.r2) == (wl, wr, r1, r2)
        x, y = X.cpu().numpy(), Y.cpu().numpy()
        assert np.array_equal(G.sorted_pairs(x[:wl], y[:wl]), G.sorted_pairs(ox[:wl], oy[:wl]))
        assert np.array_equal(G.sorted_pairs(x[wr:], y[wr:]), G.sorted_pairs(ox[wr:], oy[wr:]))


# --- random instances vs the oracle (test_hull.cpp:162-209, acceptance C1) -----
def random_instance(rng, it):
    n = int(rng.integers(0, 5000)) if it % 4 else int(rng.integers(0, 60))
    k = it % 5
    if k == 0:
        return rng.integers(-4, 5, n).astype(float), rng.integers(-4, 5, n).astype(float)
    if k == 1:
        return rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    if k == 2:
        t = rng.uniform(0, 2 * np.pi, n)
        return np.cos(t), np.sin(t)
    if k == 3:
        return (rng.integers(-(1 << 24), 1 << 24, n).astype(float),
                rng.integers(-(1 << 24), 1 << 24, n).astype(float))
    # duplicates + signed zeros
    base = rng.integers(-3, 4, (max(n, 1) // 4 + 1, 2)).astype(float)
    pts = base[rng.integers(0, base.shape[0], n)]
    xs, ys = pts[:, 0].copy(), pts[:, 1].copy()
    z = rng.random(n) < 0.3
    xs[z & (xs == 0)] = -0.0
    return xs, ys


def test_random_vs_oracle(vq, cuda, oracle):
    rng = np.random.default_rng(2024)
    for it in range(600):
        xs, ys = random_instance(rng, it)
        ref = oracle.hull_indices(xs, ys) if len(xs) else np.zeros(0, np.uint64)
        got = gpu_indices(vq, xs, ys) if len(xs) else np.zeros(0, np.uint64)
        assert np.array_equal(got, ref), f"iteration {it}: n={len(xs)}"


def test_acceptance_c1_integer_instances(vq, cuda, reference):
    """acceptance.cpp:63-82: integer instances equal the exact monotone chain."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        n = int(rng.integers(1, 2000))
        xs = rng.integers(-1000, 1001, n).astype(float)
        ys = rng.integers(-1000, 1001, n).astype(float)
        poly = vq.convex_hull(xs, ys)
        mx, my = reference.monotone_chain(xs, ys)
        assert np.array_equal(poly.xs, mx) and np.array_equal(poly.ys, my)


def test_deep_recursion_pow2_curve(vq, cuda):
    """test_hull.cpp:220-240: every point on the hull, one peeled per level."""
    m = 600
    i = np.arange(m)
    xs, ys = np.ldexp(1.0, i), np.ldexp(1.0, -i)
    idx = vq.hull_indices(xs, ys)
    assert idx.size == m
    assert idx[0] == 0 and idx[1] == m - 1
    assert idx[2:].tolist() == list(range(m - 2, 0, -1))


# --- BASELINE configs ----------------------------------------------------------
@pytest.mark.parametrize("name", ["config1_disk_1e6_s1", "config3_circle_1e7_s3",
                                  "config5_proxy_disk_4e7_s5", "config2_square_1e8_s2"])
def test_config_golden(vq, cuda, oracle, name):
    cfg = G.configs()[name]
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    got = gpu_indices(vq, xs, ys)
    assert got.size == cfg["h"]
    assert f"{oracle.fnv1a64(got):016x}" == cfg["fnv1a64_u64le"]
    assert got[:8].tolist() == cfg["head"] and got[-8:].tolist() == cfg["tail"]
    if cfg["n"] <= 10**7:  # the oracle, live on this host, on the same bytes
        assert np.array_equal(got, oracle.hull_indices(xs, ys))
    # C ABI with host buffers gives the same list
    rc, got2 = vq.vqhull_compute(xs, ys)
    assert rc == 0 and np.array_equal(got2, got)


@pytest.mark.slow
def test_config4_kuzmin_1e9(vq, cuda, oracle):
    cfg = G.configs().get("config4_kuzmin_1e9_s4")
    if cfg is None:
        pytest.skip("config4 golden not generated")
    import torch

    n = cfg["n"]
    X = torch.empty(n, dtype=torch.float64, pin_memory=True)
    Y = torch.empty(n, dtype=torch.float64, pin_memory=True)
    vq.generate(cfg["kind"], n, cfg["seed"], out=(X, Y))
    got = vq.hull_device(X.cuda(), Y.cuda()).cpu().numpy().astype(np.uint64)
    assert got.tolist() == cfg["indices"]


@pytest.mark.slow
def test_config5_disk_4e9_one_gpu(vq, cuda, oracle):
    """BASELINE config 5 (disk, 4e9 points) on ONE device: > 2^31 positions,
    lean per-level sizing; golden from the reference library
    (tests/golden/make_config5.py)."""
    cfg = G.configs().get("config5_disk_4e9_s5")
    if cfg is None:
        pytest.skip("config5 golden not generated")
    import torch

    n = cfg["n"]
    vq.trim()  # earlier tests' engine buffers back to the device
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 150 * 2**30:
        pytest.skip("needs ~150 GB of device memory")
    X = torch.empty(n, dtype=torch.float64, pin_memory=True)
    Y = torch.empty(n, dtype=torch.float64, pin_memory=True)
    vq.generate(cfg["kind"], n, cfg["seed"], out=(X, Y))
    Xd, Yd = X.cuda(), Y.cuda()
    del X, Y
    # u32 output (indices < 2^32, torch int32 storage): reinterpret unsigned
    got = vq.hull_device(Xd, Yd, u32=True).cpu().numpy().view(np.uint32).astype(np.uint64)
    del Xd, Yd
    torch.cuda.empty_cache()
    assert got.size == cfg["h"]
    assert f"{oracle.fnv1a64(got):016x}" == cfg["fnv1a64_u64le"]
    assert got.tolist() == cfg["indices"]


# --- size-independent properties at full size ----------------------------------
def test_permutation_invariance(vq, cuda):
    """Shuffled input -> the same vertex sequence."""
    for kind, n in (("disk", 2_000_000), ("circle", 1_000_000), ("square", 3_000_000)):
        xs, ys = vq.generate(kind, n, 77)
        idx = gpu_indices(vq, xs, ys).astype(np.int64)
        perm = np.random.default_rng(5).permutation(n)
        idx2 = gpu_indices(vq, xs[perm], ys[perm]).astype(np.int64)
        assert np.array_equal(xs[idx], xs[perm][idx2]) and np.array_equal(ys[idx], ys[perm][idx2])


def test_hull_contains_all_points(vq, cuda):
    """No input point strictly left of any directed hull edge (test_hull.cpp:25-52).
    Integer coordinates below 2^25 keep the reference predicate exact
    (SPEC.md:75), so the check is exact; it is evaluated on the GPU in f64."""
    import torch

    for kind, n in (("disk", 5_000_000), ("kuzmin", 5_000_000), ("circle", 300_000)):
        xs, ys = vq.generate(kind, n, 3)
        scale = 2.0**22 / max(np.abs(xs).max(), np.abs(ys).max())
        xs, ys = np.round(xs * scale), np.round(ys * scale)
        X, Y = dev(xs), dev(ys)
        idx = vq.hull_device(X, Y)
        hx, hy = X[idx], Y[idx]
        qx, qy = torch.roll(hx, -1), torch.roll(hy, -1)
        for e in range(0, hx.numel(), 64):  # 64 edges per batch
            px_, py_ = hx[e:e + 64, None], hy[e:e + 64, None]
            qx_, qy_ = qx[e:e + 64, None], qy[e:e + 64, None]
            left = (px_ - X) * (qy_ - Y) > (py_ - Y) * (qx_ - X)
            assert not bool(left.any())


def test_stats_and_timing(vq, cuda):
    xs, ys = vq.generate("disk", 1_000_000, 1)
    vq.set_timing(True)
    try:
        vq.hull_indices(xs, ys)
        s = vq.stats()
    finally:
        vq.set_timing(False)
    assert s["n"] == 1_000_000 and s["hull_size"] == 333
    assert s["timing_valid"] == 1 and s["ms_total"] > 0
    # at least: the root pass's x and y of every point, and the survivors
    assert s["launches"] >= 3 and s["bytes_moved"] >= 16 * 1_000_000


# --- both output-offset modes give the same hulls ------------------------------
def test_stable_lookback_mode(vq, cuda, oracle):
    """VQHULL stable mode (decoupled look-back, order-preserving compaction)
    must produce exactly the same index lists as the default atomic mode."""
    vq.set_stable(True)
    try:
        for name, xs, ys, idx, hx, hy in G.hull_cases()[::2]:
            rc, got = vq.vqhull_compute(xs, ys)
            assert rc == 0 and np.array_equal(got, idx), name
        rng = np.random.default_rng(99)
        for it in range(120):
            xs, ys = random_instance(rng, it)
            if len(xs):
                assert np.array_equal(gpu_indices(vq, xs, ys), oracle.hull_indices(xs, ys))
        for name in ("config1_disk_1e6_s1", "config3_circle_1e7_s3"):
            cfg = G.configs()[name]
            xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
            got = gpu_indices(vq, xs, ys)
            assert f"{oracle.fnv1a64(got):016x}" == cfg["fnv1a64_u64le"]
        # the stable mode's extract keeps S1 in input order (order-preserving)
        rng = np.random.default_rng(5)
        xs, ys = rng.uniform(-1, 1, 300_000), rng.uniform(-1, 1, 300_000)
        X, Y = dev(xs), dev(ys)
        out = vq.extract_subsets(X, Y, [-1.0, 0.0, 1.0, 0.5], [1.0, 0.5, -1.0, 0.0])
        x = X.cpu().numpy()[:out.w_l]
        a = (-1.0 - xs) * (0.5 - ys) > (0.0 - ys) * (1.0 - xs)
        assert np.array_equal(x, xs[a])
    finally:
        vq.set_stable(False)


# --- root stage: octagon filter vs the unfiltered reference-order root ---------
def test_root_modes_agree(vq, cuda, oracle):
    """The split root (default), the one-pass octagon root and the unfiltered
    one (find_extremes + bootstrap + fused levels 1+2) give identical lists."""
    rng = np.random.default_rng(77)
    cases = [(xs, ys) for _, xs, ys, *_ in G.hull_cases()]
    cases += [random_instance(rng, it) for it in range(200)]
    for kind, n, seed in (("disk", 1_000_000, 1), ("circle", 300_000, 3), ("kuzmin", 2_000_000, 4),
                          ("square", 2_000_000, 2)):
        cases.append(vq.generate(kind, n, seed))
    for i, (xs, ys) in enumerate(cases):
        if not len(xs):
            continue
        a = gpu_indices(vq, xs, ys)
        for mode in ("octagon", "reference"):
            vq.set_root_mode(mode)
            try:
                b = gpu_indices(vq, xs, ys)
            finally:
                vq.set_root_mode("split")
            assert np.array_equal(a, b), f"case {i}: n={len(xs)} mode={mode}"


def test_filter_inner_modes_agree(vq, cuda):
    """The filter pass's fast inner region (box, octagon or disk — normally
    the sample pass picks the largest) only decides which points reach the
    chord test: every forced choice gives the same survivors and the same
    hull.  The disk is the one derived in closed form."""
    for kind, n, seed in (("disk", 2_000_000, 5), ("square", 2_000_000, 2), ("kuzmin", 2_000_000, 4),
                          ("disk", 10_000_000, 1), ("circle", 2_000_000, 3)):
        xs, ys = vq.generate(kind, n, seed)
        a = gpu_indices(vq, xs, ys)
        s0 = vq.stats()
        assert s0["root_filtered"] == 2
        for mode in ("box", "octagon", "disk", "disk_only"):
            vq.set_filter_inner(mode)
            try:
                b = gpu_indices(vq, xs, ys)
                s1 = vq.stats()
            finally:
                vq.set_filter_inner("auto")
            assert np.array_equal(a, b), f"{kind} n={n}: inner={mode}"
            assert s1["survivors_root"] == s0["survivors_root"], f"{kind} n={n}: inner={mode}"


def test_root_mode_selection(vq, cuda):
    xs, ys = vq.generate("square", 1_000_000, 2)
    vq.hull_indices(xs, ys)
    s = vq.stats()
    assert s["root_filtered"] == 2 and s["root_filter_on"] == 1 and s["root_reruns"] == 0
    # the octagon of a uniform square hugs its border: almost nothing survives
    assert s["survivors_root"] < 20_000
    vq.set_root_mode("octagon")
    try:
        vq.hull_indices(xs, ys)
        assert vq.stats()["root_filtered"] == 1
    finally:
        vq.set_root_mode("split")
    # inputs that are 8- but not 16-byte aligned still take the split root
    # (the filter pass streams them from the 16-byte boundary below)
    X, Y = dev(np.concatenate([[0.0], xs])), dev(np.concatenate([[0.0], ys]))
    got = vq.hull_device(X[1:], Y[1:]).cpu().numpy().astype(np.uint64)
    assert vq.stats()["root_filtered"] == 2
    assert np.array_equal(got, vq.hull_indices(xs, ys))
    vq.set_stable(True)
    try:
        vq.hull_indices(xs, ys)
        assert vq.stats()["root_filtered"] == 0
    finally:
        vq.set_stable(False)


def test_tail_kernel_paths(vq, cuda, oracle, monkeypatch):
    """The persistent recursion kernel: the whole recursion in one launch
    (small survivor sets); a level wider than its tile bound handed to the
    host-driven kernels, which finish the recursion (forced here with small
    bounds), including circle-like inputs."""
    xs, ys = vq.generate("square", 2_000_000, 2)
    got = gpu_indices(vq, xs, ys)
    s = vq.stats()
    assert s["tail_launches"] == 1 and s["tail_levels"] == s["levels"] - 1
    assert np.array_equal(got, oracle.hull_indices(xs, ys))
    handed_over = 0
    for bound in ("2", "8", "40"):
        monkeypatch.setenv("VQHULL_TAIL_MAXTILES", bound)
        for kind, n, seed in (("square", 8_000_000, 2), ("disk", 4_000_000, 5), ("circle", 400_000, 3)):
            xs, ys = vq.generate(kind, n, seed)
            got = gpu_indices(vq, xs, ys)
            s = vq.stats()
            handed_over += s["tail_levels"] < s["levels"] - 1
            assert np.array_equal(got, oracle.hull_indices(xs, ys)), (bound, kind)
    monkeypatch.delenv("VQHULL_TAIL_MAXTILES")
    assert handed_over >= 3


def test_graph_cache_alternating_inputs(vq, cuda, oracle):
    """Replayed hull graphs are keyed by the caller's buffers: alternating
    between two inputs (as a sharded hull alternates shard and candidates)
    replays the right graph every time, also after the data changed."""
    import torch

    bufs = []
    for kind, n, seed in (("square", 3_000_000, 2), ("disk", 2_000_000, 1)):
        xs, ys = vq.generate(kind, n, seed)
        bufs.append((torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda(), oracle.hull_indices(xs, ys)))
    for rep in range(6):
        X, Y, ref = bufs[rep % 2]
        got = vq.hull_device(X, Y).cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, ref), rep
    # same buffers, new contents: the replay reads the new points
    X, Y, _ = bufs[0]
    xs, ys = vq.generate("disk", X.numel(), 9)
    X.copy_(torch.from_numpy(xs))
    Y.copy_(torch.from_numpy(ys))
    got = vq.hull_device(X, Y).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, oracle.hull_indices(xs, ys))


def test_split_root_far_outlier_rerun(vq, cuda, oracle):
    """A survivor far beyond the sampled octagon's scale voids the margin
    argument: the call is rerun unfiltered, with the same (reference) result."""
    for far in (1e10, -3e9, 5e12):
        xs, ys = vq.generate("disk", 7_000_000, 11)
        # runs 5 and 19 of 1024 points are never sampled (at n = 7e6 the
        # sample takes every 2nd run; never an odd one), so the polygon
        # cannot see these two points
        xs[5 * 1024 + 17], ys[5 * 1024 + 17] = far, 0.25
        xs[19 * 1024 + 100], ys[19 * 1024 + 100] = 0.5, far / 3
        got = gpu_indices(vq, xs, ys)
        assert vq.stats()["root_reruns"] == 1
        assert np.array_equal(got, oracle.hull_indices(xs, ys))
    xs, ys = vq.generate("disk", 7_000_000, 11)
    gpu_indices(vq, xs, ys)
    assert vq.stats()["root_reruns"] == 0


def test_filter_near_boundary_points(vq, cuda, oracle):
    """Points a few ulps inside / on / outside the octagon's chords and near its
    x breakpoints must never be dropped wrongly."""
    rng = np.random.default_rng(8)
    for it in range(40):
        t = rng.uniform(0, 2 * np.pi, 2000)
        xs, ys = np.cos(t), np.sin(t)
        # points on and next to the chords between the 8 extremes
        i8 = np.array([np.argmin(xs), np.argmax(ys - xs), np.argmax(ys), np.argmax(xs + ys),
                       np.argmax(xs), np.argmax(xs - ys), np.argmin(ys), np.argmin(xs + ys)])
        vx, vy = xs[i8], ys[i8]
        f = rng.uniform(0, 1, (8, 50))
        cx = vx[:, None] + f * (np.roll(vx, -1)[:, None] - vx[:, None])
        cy = vy[:, None] + f * (np.roll(vy, -1)[:, None] - vy[:, None])
        k = rng.integers(-3, 4, cx.shape)
        cx = cx + k * np.spacing(cx)
        xs = np.concatenate([xs, cx.ravel(), vx + np.spacing(vx)])
        ys = np.concatenate([ys, cy.ravel(), vy])
        assert np.array_equal(gpu_indices(vq, xs, ys), oracle.hull_indices(xs, ys)), f"it {it}"


def test_octagon_diagonal_ties(vq, cuda, oracle):
    """Exact ties in x+y / x-y at the extremes: diamonds and rotated squares on
    integer lattices, with duplicates; end points must be chosen."""
    rng = np.random.default_rng(21)
    for it in range(80):
        c = int(rng.integers(1, 40))
        n = int(rng.integers(5, 3000))
        x = rng.integers(-c, c + 1, n)
        y = rng.integers(-c, c + 1, n)
        keep = np.abs(x) + np.abs(y) <= c if it % 2 else np.abs(x - y) + np.abs(x + y) <= 2 * c
        xs, ys = x[keep].astype(float), y[keep].astype(float)
        k = int(rng.integers(1, 6))
        d = rng.integers(0, c + 1, k)
        xs = np.concatenate([xs, d, -d, c - d, d - c]).astype(float)
        ys = np.concatenate([ys, c - d, d - c, -d, d]).astype(float)
        perm = rng.permutation(xs.size)
        xs, ys = xs[perm], ys[perm]
        assert np.array_equal(gpu_indices(vq, xs, ys), oracle.hull_indices(xs, ys)), f"it {it}"


def test_filter_off_for_extreme_magnitudes(vq, cuda, oracle):
    """Coordinates near the double range: margins would overflow, the filter
    stays off and the result is the plain reference recursion."""
    # (beyond ~1e154 the reference's own products overflow and its choices
    # depend on the scan order; that range is out of scope)
    for scale in (1e152, 1e-310):
        xs = np.array([1.0, -1.0, 0.0, 0.7, 0.3, -0.2]) * scale
        ys = np.array([1.0, 0.9, -1.0, -0.7, 0.4, 0.1]) * scale
        got = gpu_indices(vq, xs, ys)
        assert vq.stats()["root_filter_on"] == 0
        assert np.array_equal(got, oracle.hull_indices(xs, ys))


def test_sharded_hull_nccl_world1(vq, cuda, oracle):
    """The multi-GPU path end to end on the device with NCCL (world size 1
    here: one GPU in this pool): local hull, the header-row candidate
    all-gather over NCCL, the candidates' one-CTA hull, global indices."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2510_09417_b200.distributed import sharded_hull

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for kind, n, seed in (("square", 2_000_000, 2), ("disk", 1_000_000, 1)):
            xs, ys = vq.generate(kind, n, seed)
            X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
            got = sharded_hull(X, Y, 0).cpu().numpy().astype(np.uint64)
            assert np.array_equal(got, oracle.hull_indices(xs, ys)), kind
    finally:
        dist.destroy_process_group()


def test_vqhull_compute_pageable_staged_copy(vq, cuda, oracle):
    """vqhull_compute on pageable host arrays large enough for the staged
    copy (worker threads -> pinned ring -> async H2D, driver.cu h2d()): the
    same list as from page-locked arrays and as the oracle's; odd sizes so
    the last chunk of each array is partial."""
    import torch

    n = 9_000_001
    xs, ys = vq.generate("disk", n, 9)
    ref = oracle.hull_indices(xs, ys)
    rc, got = vq.vqhull_compute(xs, ys)  # pageable numpy arrays
    assert rc == 0 and np.array_equal(got, ref)
    X = torch.from_numpy(xs).pin_memory()
    Y = torch.from_numpy(ys).pin_memory()
    rc, got2 = vq.vqhull_compute(X.numpy(), Y.numpy())
    assert rc == 0 and np.array_equal(got2, ref)
    # one pageable, one page-locked
    rc, got3 = vq.vqhull_compute(xs, Y.numpy())
    assert rc == 0 and np.array_equal(got3, ref)


def test_filter_pass_unaligned_arrays(vq, cuda, oracle):
    """Caller arrays at odd element offsets (8- but not 16-byte aligned), x
    and y independently, at sizes around the tile size: the filter pass reads
    them through shifted bulk copies; same list as the oracle's."""
    import torch

    rng = np.random.default_rng(5)
    for n in (1023, 1024, 1025, 1026, 2047, 2048, 2049, 5 * 1024 + 1, 300_001, 2_000_000):
        t = rng.uniform(0, 2 * np.pi, n)
        r = np.sqrt(rng.uniform(0, 1, n))
        xs, ys = r * np.cos(t), r * np.sin(t)
        ref = oracle.hull_indices(xs, ys)
        for ox, oy in ((1, 1), (1, 0), (0, 1), (3, 2)):
            X = torch.zeros(n + 4, dtype=torch.float64, device="cuda")
            Y = torch.zeros(n + 4, dtype=torch.float64, device="cuda")
            X[ox:ox + n] = torch.from_numpy(xs).cuda()
            Y[oy:oy + n] = torch.from_numpy(ys).cuda()
            got = vq.hull_device(X[ox:ox + n], Y[oy:oy + n]).cpu().numpy().astype(np.uint64)
            assert np.array_equal(got, ref), (n, ox, oy)
            if n > 1024:
                assert vq.stats()["root_filtered"] == 2


def test_large_trees_hybrid_emission(vq, cuda, oracle):
    """Recursion trees too large for the one-CTA emission kernel: their top
    levels are emitted by that kernel, the levels below by one launch each
    (driver.cu, the emission section).  Circle-like inputs of several sizes
    and shapes (every point a vertex; an ellipse; a circle with interior
    points and duplicated vertices), against the oracle."""
    rng = np.random.default_rng(11)
    cases = []
    for n in (1_200_000, 2_500_000):
        t = rng.uniform(0, 2 * np.pi, n)
        cases.append((np.cos(t), np.sin(t)))
    t = rng.uniform(0, 2 * np.pi, 1_500_000)
    cases.append((3.0 * np.cos(t), 0.25 * np.sin(t)))
    t = rng.uniform(0, 2 * np.pi, 2_000_000)
    r = np.where(rng.random(t.size) < 0.7, 1.0, np.sqrt(rng.uniform(0, 1, t.size)))
    xs, ys = r * np.cos(t), r * np.sin(t)
    xs[-50_000:], ys[-50_000:] = xs[:50_000], ys[:50_000]  # duplicated vertices: first occurrence wins
    cases.append((xs, ys))
    for i, (xs, ys) in enumerate(cases):
        got = gpu_indices(vq, xs, ys)
        s = vq.stats()
        assert np.array_equal(got, oracle.hull_indices(xs, ys)), f"case {i}"
        assert s["finisher_segments"] > 1000 and s["launches"] > 20, s  # host-driven levels + finisher + emission
