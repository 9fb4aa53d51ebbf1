"""GPU: the sharded hull with the sm_100a local stage and merge.

* the single-process multi-device C ABI (vqhull_cuda_hull_multi, and
  vqhull_compute with VQHULL_GPUS) with several shards — on this one-GPU pool
  the shards of a device run one after another, the merge is the same;
* the torch.distributed path (paper_2510_09417_b200.distributed) at world
  size 2: two processes on cuda:0, candidates exchanged over gloo through
  host memory (no rank's kernels wait on another's);
* against the reference's golden lists and the oracle, circle included:
  there the hull of the local hulls is NOT the reference's answer, the
  certified candidates are.
"""
import os
import socket

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu


def _golden(name):
    return G.configs()[name]


def _check_golden(oracle, got, cfg):
    assert got.size == cfg["h"]
    assert f"{oracle.fnv1a64(got):016x}" == cfg["fnv1a64_u64le"]


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_hull_multi_config5_proxy(vq, cuda, oracle, shards):
    cfg = _golden("config5_proxy_disk_4e7_s5")
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    got = vq.hull_multi(xs, ys, shards)
    _check_golden(oracle, got, cfg)
    s = vq.stats()
    assert s["hull_size"] == cfg["h"]


@pytest.mark.parametrize("kind,n,seed,shards", [("disk", 1_000_000, 1, 4), ("square", 3_000_000, 2, 2),
                                                ("kuzmin", 2_000_000, 4, 5), ("circle", 1_000_000, 3, 2),
                                                ("circle", 2_000_000, 7, 8), ("disk", 10_000, 2, 16)])
def test_hull_multi_vs_oracle(vq, cuda, oracle, kind, n, seed, shards):
    xs, ys = vq.generate(kind, n, seed)
    got = vq.hull_multi(xs, ys, shards)
    assert np.array_equal(got, oracle.hull_indices(xs, ys))


def test_hull_multi_config3_circle_and_naive_merge_differs(vq, cuda, oracle):
    """Config 3 (every point on the circle) in 4 shards equals the reference
    golden; the hull of the 4 local hulls does not."""
    import torch

    cfg = _golden("config3_circle_1e7_s3")
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    got = vq.hull_multi(xs, ys, 4)
    _check_golden(oracle, got, cfg)
    # the naive scheme: hull of the union of local hulls
    cand = []
    n = xs.size
    for r in range(4):
        a, b = r * n // 4, (r + 1) * n // 4
        X, Y = torch.from_numpy(xs[a:b]).cuda(), torch.from_numpy(ys[a:b]).cuda()
        cand.append(vq.hull_device(X, Y).cpu().numpy() + a)
    cand = np.sort(np.concatenate(cand))
    naive = cand[vq.hull_indices(xs[cand], ys[cand]).astype(np.int64)]
    assert not np.array_equal(naive.astype(np.uint64), got)


def test_hull_multi_duplicates_across_shards(vq, cuda, oracle):
    xs, ys = vq.generate("disk", 400_000, 8)
    xs[-5000:], ys[-5000:] = xs[:5000], ys[:5000]  # copies in the last shard
    got = vq.hull_multi(xs, ys, 4)
    ref = oracle.hull_indices(xs, ys)
    assert np.array_equal(got, ref)
    assert got.max() < 400_000 - 5000  # first occurrences win


def test_hull_multi_margin_retry(vq, cuda, oracle):
    """Shards of wildly different scale: the merge's scale check asks for the
    candidates again with a margin floor."""
    xs, ys = vq.generate("disk", 200_000, 11)
    xs[:100_000] *= 1e-7
    ys[:100_000] *= 1e-7
    xs[100_000:] *= 1e3
    ys[100_000:] *= 1e3
    got = vq.hull_multi(xs, ys, 2)
    assert np.array_equal(got, oracle.hull_indices(xs, ys))


def test_hull_multi_errors(vq, cuda):
    xs, ys = vq.generate("disk", 50_000, 1)
    xs[40_000] = np.nan
    with pytest.raises(vq.VQhullError) as e:
        vq.hull_multi(xs, ys, 3)
    assert e.value.rc == 1
    assert vq.hull_multi(np.zeros(0), np.zeros(0), 2).size == 0
    # the engines are healthy after the rejected call
    xs, ys = vq.generate("square", 20_000, 2)
    assert vq.hull_multi(xs, ys, 2).size > 0


def test_vqhull_compute_through_shards(vq, cuda, oracle, monkeypatch):
    """The drop-in entry point with VQHULL_GPUS set takes the sharded path."""
    cfg = _golden("config1_disk_1e6_s1")
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    for g in ("1", "3"):
        monkeypatch.setenv("VQHULL_GPUS", g)
        rc, got = vq.vqhull_compute(xs, ys)
        assert rc == 0
        _check_golden(oracle, got, cfg)
    monkeypatch.delenv("VQHULL_GPUS")


def test_shard_candidates_pack_layout(vq, cuda, oracle):
    """The local stage's pack: header {count, M_eff, A}, candidates sorted by
    global index, every local hull vertex among them."""
    import torch

    xs, ys = vq.generate("disk", 2_000_000, 3)
    X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    off = 123_456_789_012
    pack, k = vq.shard_candidates(X, Y, off, cap=1 << 16)
    P = pack.cpu().numpy()
    assert P[0, 0] == k and 0 < k < 20_000
    assert 0.9 < P[0, 1] <= 1.0 and P[0, 2] <= 1.0
    # A = the largest |coordinate| in play: at least the candidates', at most the shard's
    assert np.abs(P[1:1 + k, :2]).max() <= P[0, 2] <= max(np.abs(xs).max(), np.abs(ys).max())
    g = P[1:1 + k, 2].copy().view(np.int64)
    assert np.all(np.diff(g) > 0) and g.min() >= off
    loc = g - off
    assert np.array_equal(P[1:1 + k, 0], xs[loc]) and np.array_equal(P[1:1 + k, 1], ys[loc])
    h = oracle.hull_indices(xs, ys).astype(np.int64)
    assert np.isin(h, loc).all()
    s = vq.stats()
    assert s["shard_candidates"] == k and s["shard_cert_vertices"] == h.size
    assert s["shard_tested"] < 0.05 * xs.size  # the filter pass's survivors only
    # a second, smaller pack then the repack
    small, k2 = vq.shard_candidates(X, Y, off, cap=4)
    assert k2 == k and small[0, 0].item() == k
    big = torch.empty((k + 1, 3), dtype=torch.float64, device="cuda")
    vq.shard_repack(big)
    assert np.array_equal(big.cpu().numpy()[: k + 1], P[: k + 1])


@pytest.mark.parametrize("n,seed", [(2_000_000, 5), (700_000, 1), (5_000_000, 2)])
def test_shard_header_scale(vq, cuda, n, seed):
    """A in the header is a real magnitude on every shard (a stale counter
    word once made it garbage and forced a needless margin retry)."""
    import torch

    xs, ys = vq.generate("disk", n, seed)
    for lo, hi in ((0, n // 2), (n // 2, n)):
        X, Y = torch.from_numpy(xs[lo:hi]).cuda(), torch.from_numpy(ys[lo:hi]).cuda()
        for _ in range(2):
            pack, k = vq.shard_candidates(X, Y, lo, cap=1 << 16)
            P = pack.cpu().numpy()
            cand = np.abs(P[1:1 + k, :2]).max()
            assert cand <= P[0, 2] <= max(np.abs(xs[lo:hi]).max(), np.abs(ys[lo:hi]).max()), P[0]
            assert 0.9 < P[0, 1] <= 1.0


# --- torch.distributed at world size 2 on one GPU (gloo, host staging) -------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_09417_b200 as vq
        from paper_2510_09417_b200 import distributed as D

        xs, ys = vq.generate(kind, n, seed)
        off, cnt = D.shard_range(n, rank, world)
        X = torch.from_numpy(xs[off:off + cnt].copy()).cuda()
        Y = torch.from_numpy(ys[off:off + cnt].copy()).cuda()
        g = D.sharded_hull(X, Y, off)
        q.put((rank, g.cpu().numpy(), D.last_info()))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def _run_world(kind, n, seed, world=2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, g, info = q.get(timeout=600)
        res[r] = (g, info)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_world2_config5_proxy(vq, cuda, oracle):
    cfg = _golden("config5_proxy_disk_4e7_s5")
    res = _run_world(cfg["kind"], cfg["n"], cfg["seed"])
    for r in (0, 1):
        g, info = res[r]
        assert isinstance(g, np.ndarray), g
        _check_golden(oracle, g.astype(np.uint64), cfg)
        assert info["gather_rounds"] == 1


@pytest.mark.parametrize("kind,n,seed", [("square", 4_000_000, 2), ("kuzmin", 4_000_000, 4),
                                         ("circle", 1_000_000, 3)])
def test_world2_vs_oracle(vq, cuda, oracle, kind, n, seed):
    res = _run_world(kind, n, seed)
    xs, ys = vq.generate(kind, n, seed)
    ref = oracle.hull_indices(xs, ys)
    for r in (0, 1):
        g, _ = res[r]
        assert isinstance(g, np.ndarray), g
        assert np.array_equal(g.astype(np.uint64), ref)


@pytest.mark.slow
def test_world2_config3_circle(vq, cuda, oracle):
    cfg = _golden("config3_circle_1e7_s3")
    res = _run_world(cfg["kind"], cfg["n"], cfg["seed"])
    for r in (0, 1):
        _check_golden(oracle, res[r][0].astype(np.uint64), cfg)


@pytest.mark.slow
def test_hull_multi_beyond_u32(vq, cuda, oracle):
    """n = 2^32 + 4096 points (above one device's 32-bit range): the sharded
    drop-in takes them in shards below 2^32 (run one after another on this
    GPU), with 64-bit global indices.  No reference run fits this host, so the
    check is consistency: 2 and 3 shards give the same list, which reaches
    indices above 2^32, and its first 4e9-point part agrees with config 5's
    golden hull where the two overlap."""
    import torch

    n = (1 << 32) + 4096
    torch.cuda.empty_cache()
    vq.trim()
    free, _ = torch.cuda.mem_get_info()
    if free < 150 * 2**30:
        pytest.skip("needs ~150 GB of device memory")
    import psutil
    if psutil.virtual_memory().available < 90 * 2**30:
        pytest.skip("needs ~90 GB of host memory")
    xs = np.empty(n)
    ys = np.empty(n)
    vq.generate("disk", n, 5, out=(xs, ys))
    # a far vertex above 2^32, and an exact copy of it further up (the first
    # occurrence must win with 64-bit indices)
    far = (1 << 32) + 100
    xs[far], ys[far] = 3.0, 3.0
    xs[far + 50], ys[far + 50] = 3.0, 3.0
    g2 = vq.hull_multi(xs, ys, 2)
    vq.trim()
    g3 = vq.hull_multi(xs, ys, 3)
    vq.trim()
    assert np.array_equal(g2, g3)
    assert far in g2.tolist() and far + 50 not in g2.tolist()
    # its vertices below 4e9 are vertices of config 5's (4e9-point) hull
    # (a point that is a vertex of a superset's hull is one of the subset's)
    cfg = G.configs()["config5_disk_4e9_s5"]
    low = g2[g2 < 4 * 10**9]
    assert np.isin(low, np.array(cfg["indices"], dtype=np.uint64)).all()
    # with the drop-in entry point (it picks the shard count itself)
    rc, g = vq.vqhull_compute(xs, ys)
    assert rc == 0 and np.array_equal(g, g2)
    del xs, ys


def test_bench_multi_gpu_path_on_one_gpu(cuda, tmp_path):
    """bench.py's N > 1 flow (torchrun, sharded config 5 with a reduced n,
    timing, max over ranks, e2e) end to end, both ranks on this one GPU over
    gloo (VQHULL_BENCH_SHARE_GPU, a test hook): the JSON line it prints."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VQHULL_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--points", "4000000", "--steps", "2", "--warmup", "1",
           "--no-cpu"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("config5: disk seed=5, n=4000000 total, sharded evenly over 2 GPU(s)")
    assert d["details"]["merge"]["margin_retries"] == 0 and d["details"]["merge"]["hull"] > 100
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
