"""Headers {count, M_eff, A} of the shards of a sharded disk (debug).
usage: python tools/dbg_shard_hdr.py N SHARDS [SEED]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_09417_b200 as vq  # noqa: E402
from paper_2510_09417_b200.distributed import shard_range  # noqa: E402

n, S = int(float(sys.argv[1])), int(sys.argv[2])
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 5
xs, ys = vq.generate("disk", n, seed)
for rep in range(2):
    for r in range(S):
        off, cnt = shard_range(n, r, S)
        x = torch.from_numpy(xs[off:off + cnt]).cuda()
        y = torch.from_numpy(ys[off:off + cnt]).cuda()
        pack, k = vq.shard_candidates(x, y, off, 8192, 0.0)
        print(rep, r, off, cnt, "k", k, "hdr", pack[0].tolist(), {k_: v for k_, v in vq.stats().items() if "root" in k_ or "shard" in k_})
