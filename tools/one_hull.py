"""One hull of a BASELINE config on cuda:0 (for ncu launch lists).
usage: python tools/one_hull.py CONFIG|KIND:N:SEED [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_09417_b200 as vq  # noqa: E402

CONFIGS = {1: ("disk", 10**6, 1), 2: ("square", 10**8, 2), 3: ("circle", 10**7, 3),
           4: ("kuzmin", 10**9, 4), 5: ("disk", 4 * 10**9, 5)}
if ":" in sys.argv[1]:  # KIND:N:SEED
    kind, n, seed = sys.argv[1].split(":")
    n, seed = int(float(n)), int(seed)
else:
    kind, n, seed = CONFIGS[int(sys.argv[1])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
X = torch.empty(n, dtype=torch.float64, pin_memory=True)
Y = torch.empty(n, dtype=torch.float64, pin_memory=True)
vq.generate(kind, n, seed, out=(X, Y))
X, Y = X.cuda(), Y.cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(reps):
    h = vq.hull_device(X, Y, out=out, u32=True)
torch.cuda.synchronize()
print(f"{kind} n={n}: h={h.numel()} stats={vq.stats()}")
