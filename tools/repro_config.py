"""Run one generated configuration on the GPU vs the oracle (debug aid)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_09417_b200 as vq
from oracle import Oracle
kind, n, seed = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
xs, ys = vq.generate(kind, n, seed)
ref = Oracle().hull_indices(xs, ys) if n <= 2 * 10**7 else None
for rep in range(int(sys.argv[4]) if len(sys.argv) > 4 else 2):
    try:
        got = vq.hull_device(torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()).cpu().numpy().astype(np.uint64)
        print(kind, n, "rep", rep, "h", got.size, "match", None if ref is None else np.array_equal(got, ref), flush=True)
    except Exception as e:
        print("ERR", e, flush=True)
        break
s = vq.stats(); print({k: s[k] for k in ("levels", "launches", "segments", "finisher_segments", "level_points")})
