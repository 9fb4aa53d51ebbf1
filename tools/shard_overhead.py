"""Time of the sharded hull's stages at world size 1 (one GPU, NCCL): the
per-rank cost a multi-GPU run adds on top of the local hull.
usage: python tools/shard_overhead.py KIND N SEED"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2510_09417_b200 as vq  # noqa: E402
from paper_2510_09417_b200 import distributed as D  # noqa: E402

kind, n, seed = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
X = torch.empty(n, dtype=torch.float64, pin_memory=True)
Y = torch.empty(n, dtype=torch.float64, pin_memory=True)
vq.generate(kind, n, seed, out=(X, Y))
X, Y = X.cuda(), Y.cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, r


t_local, h = timed(lambda: vq.hull_device(X, Y, out=out, u32=True))
t_shard, g = timed(lambda: D.sharded_hull(X, Y, 0))
t_cand, pk = timed(lambda: vq.shard_candidates(X, Y, 0, 8192, 0.0))
print(f"{kind} n={n}: local hull {t_local:.3f} ms (h={h.numel()}), sharded_hull (world 1) {t_shard:.3f} ms "
      f"(h={g.numel()}), of which local stage + certificate + pack {t_cand:.3f} ms; info {D.last_info()}")
dist.destroy_process_group()
