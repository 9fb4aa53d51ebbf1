"""One hull of a generated configuration (for ncu captures): python tools/one_hull.py KIND N SEED [REPS]."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2510_09417_b200 as vq
kind, n, seed = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
xs, ys = vq.generate(kind, n, seed)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
for _ in range(reps):
    out = vq.hull_device(X, Y, u32=True)
torch.cuda.synchronize()
print(kind, n, "h", out.numel())
