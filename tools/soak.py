"""Randomised soak against the oracle: ITERS small random instances (the parity
test's generator) plus 12 mid-size circle / annulus / lattice / integer-disk
inputs from seed SEED.  Run it under VQHULL_TINY=0 VQHULL_KC=0 VQHULL_TAIL=0
for the host-driven levels and the batch finisher, VQHULL_KC=0 for KT.
usage: python tools/soak.py SEED ITERS"""
import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch
import paper_2510_09417_b200 as vq
from oracle import Oracle
from test_gpu_parity import random_instance, gpu_indices
torch.cuda.set_device(0)
O = Oracle()
seed0 = int(sys.argv[1]); iters = int(sys.argv[2])
bad = 0
rng = np.random.default_rng(seed0)
for it in range(iters):
    xs, ys = random_instance(rng, it)
    if len(xs) == 0: continue
    if not np.array_equal(gpu_indices(vq, xs, ys), O.hull_indices(xs, ys)):
        print("MISMATCH random", seed0, it, len(xs)); bad += 1
for s in range(12):
    r = np.random.default_rng(seed0 * 100 + s)
    n = int(r.integers(2000, 400000))
    kind = s % 4
    t = r.uniform(0, 2 * np.pi, n)
    if kind == 0: xs, ys = np.cos(t), np.sin(t)
    elif kind == 1:
        rad = np.where(r.random(n) < 0.5, 1.0, r.uniform(0.95, 1.0, n)); xs, ys = rad * np.cos(t), rad * np.sin(t)
    elif kind == 2:
        xs, ys = np.round(np.cos(t) * 4096) / 4096, np.round(np.sin(t) * 4096) / 4096
    else:
        xs, ys = r.integers(-2000, 2001, n).astype(float), r.integers(-2000, 2001, n).astype(float)
        m = xs * xs + ys * ys <= 2000 * 2000; xs, ys = xs[m], ys[m]
    if not np.array_equal(gpu_indices(vq, xs, ys), O.hull_indices(xs, ys)):
        print("MISMATCH mid", seed0, s, kind, len(xs)); bad += 1
print("soak", seed0, "OK" if bad == 0 else f"FAILED {bad}")
