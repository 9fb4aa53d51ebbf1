"""CPU, world_size 2 over gloo: the sharded-hull host logic (candidate
all-gather, first-occurrence resolution across shards, global index mapping)
with the oracle standing in for the per-rank local hull."""
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


def _oracle_local_hull(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    from oracle import Oracle

    idx = Oracle().hull_indices(x.numpy(), y.numpy())
    return torch.from_numpy(idx.astype(np.int64))


def _worker(rank, world, port, kind, n, seed, dup, q, cap=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_09417_b200 import distributed as D
        from paper_2510_09417_b200 import generate
        from paper_2510_09417_b200.distributed import shard_range, sharded_hull

        if cap is not None:  # force the two-round gather
            D.GATHER_CAP = cap

        xs, ys = generate(kind, n, seed, threads=2)
        if dup:  # copies of points of shard 0 placed in the last shard
            xs[-dup:], ys[-dup:] = xs[:dup], ys[:dup]
        off, cnt = shard_range(n, rank, world)
        x = torch.from_numpy(xs[off:off + cnt].copy())
        y = torch.from_numpy(ys[off:off + cnt].copy())
        g = sharded_hull(x, y, off, local_hull=_oracle_local_hull)
        q.put((rank, g.numpy()))
    finally:
        dist.destroy_process_group()


def run_world(world, kind, n, seed, dup=0, cap=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, seed, dup, q, cap)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("kind,n,seed,dup", [("disk", 200_000, 5, 0), ("square", 100_000, 2, 0),
                                             ("kuzmin", 100_000, 4, 0), ("disk", 50_000, 7, 4000)])
def test_sharded_hull_world2_equals_global(oracle, kind, n, seed, dup):
    from paper_2510_09417_b200 import generate

    res = run_world(2, kind, n, seed, dup)
    xs, ys = generate(kind, n, seed, threads=2)
    if dup:
        xs[-dup:], ys[-dup:] = xs[:dup], ys[:dup]
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in (0, 1):
        assert np.array_equal(res[r], ref)


def test_sharded_hull_two_round_gather(oracle):
    """A local hull larger than the one-collective capacity (forced to 8
    candidates) takes the second, count-padded all-gather."""
    from paper_2510_09417_b200 import generate

    res = run_world(2, "disk", 100_000, 3, cap=8)
    xs, ys = generate("disk", 100_000, 3, threads=2)
    ref = oracle.hull_indices(xs, ys).astype(np.int64)
    for r in (0, 1):
        assert np.array_equal(res[r], ref)


def test_shard_range_partitions():
    from paper_2510_09417_b200.distributed import shard_range

    for n in (0, 1, 7, 1000, 10**9 + 3):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == n
            for (o1, c1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + c1 == o2
