"""Run one golden hull case on the GPU (debug aid)."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
import golden_io as G
import paper_2510_09417_b200 as vq
name = sys.argv[1]
for c in G.hull_cases():
    if c[0] == name:
        _, xs, ys, idx, hx, hy = c
        rc, got = vq.vqhull_compute(xs, ys)
        print(name, "n", len(xs), "rc", rc, "match", np.array_equal(got, idx), vq.stats())
