"""Multi-GPU sharded hull: one process per GPU, torch.distributed for plumbing.

Scheme (BASELINE north star), exact by construction:

1. rank r owns a contiguous shard [offset_r, offset_r + n_r) of the global
   point sequence and runs the local stage on its GPU
   (``vqhull_cuda_shard_candidates``): its local hull with the sm_100a path,
   then a certificate that keeps every point it cannot PROVE to lie deep
   inside that local hull (the split root's margin argument),
   sorted by global index and packed behind a header row {count, M_eff, A};
2. ONE all-gather of the packs (NCCL over NVLink on GPUs; gloo in the CPU
   tests); a second, count-padded round only when a rank has more than
   ``GATHER_CAP`` candidates;
3. every rank merges (``vqhull_cuda_merge_candidates``): the ordinary hull
   over the union of the candidates, in global-index order so that equal
   coordinates resolve to their first occurrence (vqhull_c.cpp:51-61), mapped
   back to global indices.

Why not just the hull of the local hulls: the reference's f64 predicates are
not robust, so a global recursion can keep near-collinear points a shard's
recursion dropped (circle 1e7, 9,994,016 vs 9,994,044 vertices).
Only points that provably cannot affect any decision of the global recursion
are left behind, so the merge IS the reference's global recursion.  The
margin's rounding bound needs the largest coordinate in play within 2^12 of
every shard's scale; the merge checks it and, if a shard's scale is too
small (wildly different shards), every rank recomputes its candidates with a
margin floor (``RetryWithFloor``) — one more round, then it always holds.

There is no data-path collective other than this candidate all-gather.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist

# candidates a rank sends in the one-collective fast path (disk 4e9 over 8
# GPUs: ~3k per rank); larger candidate sets take a second round
GATHER_CAP = 8192

LocalStage = Callable[..., Tuple[torch.Tensor, int]]

_LAST = {"launches": 0, "info": {}}


def last_launches() -> int:
    """Kernels the last sharded_hull launched on this rank (local + merge)."""
    return int(_LAST["launches"])


def last_info() -> dict:
    """Candidate counts, rounds and retries of the last sharded_hull."""
    return dict(_LAST["info"])


class DeviceStages:
    """The sm_100a local stage and merge (the product path)."""

    def __init__(self):
        from . import lib

        lib()  # fail loudly without the native library

    def local(self, x, y, offset: int, cap: int, floor: float):
        from . import shard_candidates, stats

        pack, k = shard_candidates(x, y, offset, cap, floor)
        return pack, k, int(stats()["launches"])

    def repack(self, pack):
        from . import shard_repack

        shard_repack(pack)

    def merge(self, packs):
        from . import merge_candidates, stats

        out = merge_candidates(packs)
        return out, int(stats()["launches"])


def _gather(pack: torch.Tensor, stages, group) -> Tuple[torch.Tensor, list, int]:
    world = dist.get_world_size(group)
    # gloo moves host tensors: device packs are staged through host memory
    # (the single-GPU test of the multi-rank path); NCCL gathers in HBM
    host = pack.is_cuda and dist.get_backend(group) == "gloo"

    def all_gather(t):
        src = t.cpu() if host else t
        bufs = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(bufs, src, group=group)
        out = torch.stack(bufs)
        return out.to(t.device) if host else out

    packs = all_gather(pack)
    counts = [int(c) for c in packs[:, 0, 0].cpu().tolist()]
    rounds = 1
    kmax = max(counts)
    if kmax > pack.shape[0] - 1:  # rare: more candidates than the fast path's room
        big = torch.empty((kmax + 1, 3), dtype=pack.dtype, device=pack.device)
        stages.repack(big)
        packs = all_gather(big)
        rounds = 2
    return packs, counts, rounds


def sharded_hull(x: torch.Tensor, y: torch.Tensor, offset: int,
                 group: Optional[dist.ProcessGroup] = None, stages=None,
                 cap: Optional[int] = None) -> torch.Tensor:
    """Global clockwise hull indices (int64, on x's device) of the union of
    every rank's shard.  Called by every rank of `group` with its own shard;
    ranks must hold contiguous shards in rank (= offset) order."""
    stages = stages or DeviceStages()
    cap = GATHER_CAP if cap is None else cap
    floor = 0.0
    retries = 0
    while True:
        pack, k, l_local = stages.local(x, y, int(offset), cap, floor)
        packs, counts, rounds = _gather(pack, stages, group)
        try:
            out, l_merge = stages.merge(packs)
            break
        except Exception as e:  # RetryWithFloor: every rank sees the same headers
            if getattr(e, "floor", None) is None or retries:
                raise
            floor = e.floor
            retries += 1
    _LAST["launches"] = l_local + l_merge
    _LAST["info"] = {"candidates_per_rank": counts, "candidates_total": int(sum(counts)),
                     "gather_rounds": rounds, "margin_retries": retries, "hull": int(out.numel())}
    return out


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous, even split of [0, n_total): (offset, count)."""
    base, rem = divmod(n_total, world)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)
