"""Multi-GPU sharded hull: one process per GPU, torch.distributed for plumbing.

Scheme (BASELINE north star): rank r owns a contiguous shard
[offset_r, offset_r + n_r) of the global point sequence and computes its local
hull with the sm_100a path.  The local hull vertices — a few thousand
(x, y, global index) candidates — are exchanged with ONE all-gather (NCCL over
NVLink on GPUs; gloo in the CPU tests), and every rank computes the hull of
the candidates (the same sm_100a path) and maps it back to global indices.

Exactness: conv(∪ local hulls) = conv(all points), and each local hull carries
first-occurrence indices within its shard; candidates are ordered by global
index before the final hull, so a vertex present in several shards resolves
to its smallest global index — the reference's first-occurrence rule
(vqhull_c.cpp:51-61).  Under the reference's non-robust f64 predicates the
merged result can differ from a single global pass on near-degenerate inputs
(probe P3: circle); tests gate each distribution on the oracle.

There is no data-path collective other than this candidate all-gather: the
partition work itself is embarrassingly parallel across shards.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

LocalHull = Callable[[torch.Tensor, torch.Tensor], torch.Tensor]


def _default_local_hull(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    from . import hull_device

    return hull_device(x, y)


def gather_candidates(cx: torch.Tensor, cy: torch.Tensor, cg: torch.Tensor,
                      group: Optional[dist.ProcessGroup] = None):
    """All-gather variable-length (x, y, global index) candidate lists.

    Packs each candidate as three 64-bit words (the index bit-cast into f64
    storage) so one collective moves everything; counts go first so the
    payload can be padded to the largest shard.
    """
    dev = cx.device
    k = torch.tensor([cx.numel()], dtype=torch.int64, device=dev)
    world = dist.get_world_size(group)
    counts = [torch.zeros_like(k) for _ in range(world)]
    dist.all_gather(counts, k, group=group)
    counts = [int(c.item()) for c in counts]
    kmax = max(max(counts), 1)
    pack = torch.zeros((kmax, 3), dtype=torch.float64, device=dev)
    pack[: cx.numel(), 0] = cx
    pack[: cx.numel(), 1] = cy
    pack[: cx.numel(), 2] = cg.to(torch.int64).view(torch.float64)
    bufs = [torch.empty_like(pack) for _ in range(world)]
    dist.all_gather(bufs, pack, group=group)
    parts = [b[:c] for b, c in zip(bufs, counts)]
    allp = torch.cat(parts, dim=0)
    gidx = allp[:, 2].contiguous().view(torch.int64)
    return allp[:, 0].contiguous(), allp[:, 1].contiguous(), gidx


def sharded_hull(x: torch.Tensor, y: torch.Tensor, offset: int,
                 group: Optional[dist.ProcessGroup] = None,
                 local_hull: Optional[LocalHull] = None) -> torch.Tensor:
    """Global clockwise hull indices (int64, on x's device) of the union of
    every rank's shard.  Called by every rank of `group` with its own shard."""
    hull = local_hull or _default_local_hull
    li = hull(x, y).to(torch.int64)
    cx, cy = x[li], y[li]
    cg = li + int(offset)
    ax, ay, ag = gather_candidates(cx, cy, cg, group)
    # first occurrence == smallest global index: order candidates by it
    order = torch.argsort(ag)
    ax, ay, ag = ax[order].contiguous(), ay[order].contiguous(), ag[order]
    fi = hull(ax, ay).to(torch.int64)
    return ag[fi]


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous, even split of [0, n_total): (offset, count)."""
    base, rem = divmod(n_total, world)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)
