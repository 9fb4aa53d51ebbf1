"""Quick GPU parity probe (development aid): random + config cases vs oracle."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2510_09417_b200 as vq
from oracle import Oracle
O = Oracle()
rng = np.random.default_rng(7)
bad = 0
cases = 0
def check(xs, ys, tag):
    global bad, cases
    cases += 1
    ref = O.hull_indices(xs, ys) if len(xs) else np.zeros(0, np.uint64)
    x = torch.from_numpy(np.ascontiguousarray(xs, dtype=np.float64)).cuda()
    y = torch.from_numpy(np.ascontiguousarray(ys, dtype=np.float64)).cuda()
    got = vq.hull_device(x, y).cpu().numpy().astype(np.uint64)
    if not np.array_equal(got, ref):
        bad += 1
        if bad < 6:
            print("MISMATCH", tag, len(xs), "h", len(ref), len(got), ref[:10], got[:10], flush=True)
for it in range(400):
    n = int(rng.integers(0, 3000)) if it % 5 else int(rng.integers(0, 40))
    k = it % 4
    if k == 0: xs = rng.integers(-4, 5, n).astype(float); ys = rng.integers(-4, 5, n).astype(float)
    elif k == 1: xs = rng.uniform(-1, 1, n); ys = rng.uniform(-1, 1, n)
    elif k == 2:
        th = rng.uniform(0, 2*np.pi, n); xs = np.cos(th); ys = np.sin(th)
    else: xs = rng.integers(-1000, 1000, n).astype(float); ys = rng.integers(-1000, 1000, n).astype(float)
    check(xs, ys, f"rand{k}")
print("random cases", cases, "bad", bad, flush=True)
for kind, n, seed in [("disk", 10**6, 1), ("square", 10**7, 2), ("circle", 10**6, 3), ("kuzmin", 10**7, 4), ("circle", 10**7, 3)]:
    xs, ys = vq.generate(kind, n, seed)
    t = time.time(); ref = O.hull_indices(xs, ys); tc = time.time() - t
    x = torch.from_numpy(xs).cuda(); y = torch.from_numpy(ys).cuda()
    got = vq.hull_device(x, y).cpu().numpy().astype(np.uint64)
    torch.cuda.synchronize()
    vq.set_timing(True)
    got = vq.hull_device(x, y).cpu().numpy().astype(np.uint64)
    s = vq.stats()
    vq.set_timing(False)
    print(kind, n, "h", len(ref), "match", np.array_equal(got, ref), "cpu %.2fs" % tc,
          "gpu total %.3f ms" % s["ms_total"], {k: round(v, 3) if isinstance(v, float) else v for k, v in s.items()}, flush=True)
