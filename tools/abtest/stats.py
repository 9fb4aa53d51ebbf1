"""Survivors / levels / reruns of one configuration (development aid)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2510_09417_b200 as vq
kind, n, seed = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
xs, ys = vq.generate(kind, n, seed)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
out = torch.empty(n, dtype=torch.int32, device='cuda')
vq.hull_device(X, Y, out=out, u32=True)
vq.set_timing(True); h = vq.hull_device(X, Y, out=out, u32=True); s = vq.stats(); vq.set_timing(False)
print(kind, n, {k: s[k] for k in ('hull_size', 'levels', 'survivors_root', 'root_filtered', 'root_filter_on', 'root_reruns', 'tail_levels', 'ms_root_partition', 'ms_total')})
