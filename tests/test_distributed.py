"""CPU, world_size 2 over gloo: the sharded hull's host protocol
(paper_2510_09417_b200.distributed: packing, the all-gather rounds, the
margin retry, first occurrence across shards, global indices) with the CPU
stand-ins of tests/sharded_cpu.py in place of the device stages.  The
certificate makes the merge exact by construction, so every case — circle
included, where the hull of local hulls differs from the global recursion —
must equal the oracle's global hull."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def make_points(kind, n, seed, dup=0, scale_split=False, nan_at=None):
    from paper_2510_09417_b200 import generate

    xs, ys = generate(kind, n, seed, threads=2)
    if dup:  # copies of points of shard 0 placed in the last shard
        xs[-dup:], ys[-dup:] = xs[:dup], ys[:dup]
    if scale_split:  # shard 0 tiny, shard 1 huge: the margin retry
        xs[: n // 2] *= 1e-7
        ys[: n // 2] *= 1e-7
        xs[n // 2:] *= 1e3
        ys[n // 2:] *= 1e3
    if nan_at is not None:
        xs[nan_at] = np.nan
    return xs, ys


def _worker(rank, world, port, spec, cap, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from sharded_cpu import CPUStages

        from paper_2510_09417_b200 import distributed as D
        from paper_2510_09417_b200.distributed import shard_range, sharded_hull

        xs, ys = make_points(*spec)
        off, cnt = shard_range(xs.size, rank, world)
        x = torch.from_numpy(xs[off:off + cnt].copy())
        y = torch.from_numpy(ys[off:off + cnt].copy())
        try:
            g = sharded_hull(x, y, off, stages=CPUStages(), cap=cap)
            q.put((rank, g.numpy(), D.last_info()))
        except Exception as e:  # noqa: BLE001 — reported to the parent
            q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def run_world(world, spec, cap=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, cap, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, g, info = q.get(timeout=300)
        res[r] = (g, info)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("spec", [("disk", 200_000, 5), ("square", 100_000, 2),
                                  ("kuzmin", 100_000, 4), ("disk", 50_000, 7, 4000),
                                  ("circle", 100_000, 3)])
def test_sharded_hull_world2_equals_global(oracle, spec):
    res = run_world(2, spec)
    xs, ys = make_points(*spec)
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in (0, 1):
        g, info = res[r]
        assert isinstance(g, np.ndarray), g
        assert np.array_equal(g, ref)
        assert info["margin_retries"] == 0
        # (circle: every point is a candidate, more than the fast path's room)
        assert info["gather_rounds"] == (2 if spec[0] == "circle" else 1)


def test_sharded_hull_world3_circle(oracle):
    """Points on a circle, three shards: the local hulls each lose
    near-collinear points the global recursion keeps; the certified
    candidates do not."""
    spec = ("circle", 60_000, 9)
    res = run_world(3, spec)
    xs, ys = make_points(*spec)
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in range(3):
        assert np.array_equal(res[r][0], ref)


def test_sharded_hull_two_round_gather(oracle):
    """More candidates than the one-collective capacity (forced to 8): the
    second, count-padded all-gather."""
    spec = ("disk", 100_000, 3)
    res = run_world(2, spec, cap=8)
    xs, ys = make_points(*spec)
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in (0, 1):
        assert np.array_equal(res[r][0], ref)
        assert res[r][1]["gather_rounds"] == 2


def test_sharded_hull_margin_retry(oracle):
    """Shards of wildly different scale: the merge's scale check fails once,
    every rank recomputes its candidates with the margin floor."""
    spec = ("disk", 40_000, 11, 0, True)
    res = run_world(2, spec)
    xs, ys = make_points(*spec)
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in (0, 1):
        assert np.array_equal(res[r][0], ref)
        assert res[r][1]["margin_retries"] == 1


def test_sharded_hull_nonfinite_fails_on_every_rank():
    spec = ("disk", 20_000, 1, 0, False, 15_000)
    res = run_world(2, spec)
    for r in (0, 1):
        assert isinstance(res[r][0], str) and "non-finite" in res[r][0]


def test_certificate_never_drops_a_hull_vertex(oracle):
    """The CPU certificate on its own: the global hull's vertices of a shard
    are always kept (they are on the boundary of every polygon of input
    points that contains them)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from sharded_cpu import certify

    for kind, n, seed in (("disk", 50_000, 2), ("circle", 20_000, 4), ("square", 50_000, 6)):
        xs, ys = make_points(kind, n, seed)
        h = oracle.hull_indices(xs, ys).astype(np.int64)
        keep, _ = certify(xs, ys, h)
        assert keep[h].all()
        if kind != "circle":
            assert keep.sum() < 0.05 * n


def test_shard_range_partitions():
    from paper_2510_09417_b200.distributed import shard_range

    for n in (0, 1, 7, 1000, 10**9 + 3):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == n
            for (o1, c1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + c1 == o2


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus 2 without two visible GPUs exits non-zero instead of
    printing an n_gpus: 1 line."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode != 0
    assert "n_gpus" not in p.stdout
    assert "refusing" in p.stderr


def test_bench_workload_strings_match_between_arms():
    import importlib.util

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    a1 = b.parse(["--gpus", "1"])
    w1 = b.Workload(a1, 1)
    assert w1.cfg == 2 and w1.total == 10**8 and "BASELINE configs[1]" in w1.name
    a8 = b.parse(["--gpus", "8"])
    w8 = b.Workload(a8, 8)
    assert w8.cfg == 5 and w8.strong and w8.total == 4 * 10**9
    offs = [w8.shard(r) for r in range(8)]
    assert sum(c for _, c in offs) == 4 * 10**9 and offs[1][0] == 5 * 10**8
    # the reference arm prints the same config object for the same flags
    assert b.Workload(a8, 8).config() == w8.config()


def test_reference_arm_never_loads_the_product_library(reference):
    """`bench.py --impl reference` times the reference library only: it runs
    with the product library made unloadable (VQHULL_LIB pointing nowhere) and
    no GPU visible, and prints the driver's line for the reference arm."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VQHULL_LIB="/nonexistent/libvqhull_b200.so", CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "1",
                        "--points", "200000", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=root)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["unit"] == "points/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config1: disk seed=1, n=200000")
