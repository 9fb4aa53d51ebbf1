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


# candidates a rank sends in the one-collective fast path (local hulls are a
# few dozen to a few thousand vertices; larger ones take a second round)
GATHER_CAP = 8192


def gather_candidates(cx: torch.Tensor, cy: torch.Tensor, cg: torch.Tensor,
                      group: Optional[dist.ProcessGroup] = None, cap: Optional[int] = None):
    """All-gather variable-length (x, y, global index) candidate lists.

    Packs each candidate as three 64-bit words (the index bit-cast into f64
    storage) behind a header row holding the count, padded to `cap` rows, so
    ONE collective moves counts and payload.  If any rank has more than `cap`
    candidates (every rank sees that in the headers), a second all-gather
    padded to the largest count follows.
    """
    dev = cx.device
    k = cx.numel()
    world = dist.get_world_size(group)
    cap = GATHER_CAP if cap is None else cap

    def packed(rows: int, with_header: bool) -> torch.Tensor:
        h = 1 if with_header else 0
        pack = torch.zeros((rows + h, 3), dtype=torch.float64, device=dev)
        if with_header:
            pack[0, 0] = float(k)
        m = min(k, rows)
        pack[h:h + m, 0] = cx[:m]
        pack[h:h + m, 1] = cy[:m]
        pack[h:h + m, 2] = cg[:m].to(torch.int64).view(torch.float64)
        return pack

    first = packed(cap, True)
    bufs = [torch.empty_like(first) for _ in range(world)]
    dist.all_gather(bufs, first, group=group)
    counts = [int(c) for c in torch.stack([b[0, 0] for b in bufs]).cpu().tolist()]
    if max(counts) <= cap:
        parts = [b[1:1 + c] for b, c in zip(bufs, counts)]
    else:  # rare: a local hull larger than the fast path's capacity
        kmax = max(counts)
        full = packed(kmax, False)
        bufs = [torch.empty_like(full) for _ in range(world)]
        dist.all_gather(bufs, full, group=group)
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
