"""Per-kernel-family device times of one configuration (development aid)."""
import sys, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_09417_b200 as vq
kind, n, seed = sys.argv[1], int(float(sys.argv[2])), int(sys.argv[3])
xs, ys = vq.generate(kind, n, seed)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
out = torch.empty(n, dtype=torch.int32, device='cuda')
for _ in range(3): vq.hull_device(X, Y, out=out, u32=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); K = 5
for _ in range(K): vq.hull_device(X, Y, out=out, u32=True)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
vq.set_timing(True); vq.hull_device(X, Y, out=out, u32=True); s = vq.stats(); vq.set_timing(False)
hh = vq.hull_device(X, Y, out=out, u32=True).long()
sig = int((hh * torch.arange(1, hh.numel() + 1, device='cuda')).sum().item()) & 0xffffffffffff
fam = {k[3:]: round(v, 3) for k, v in s.items() if k.startswith('ms_')}
print(f"{kind} n={n}: {ms:.3f} ms/hull  {n/ms/1e6:.3g} Gpts/s  levels={s['levels']} launches={s['launches']} h={hh.numel()} sig={sig:012x} {fam}")
