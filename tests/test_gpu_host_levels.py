"""The host-driven level path on small inputs: with the one-CTA hull, the
cluster recursion and the persistent tail kernel switched off (VQHULL_TINY=0,
VQHULL_KC=0, VQHULL_TAIL=0 — read once per process, hence the subprocess),
every recursion below the root runs through the level kernels and the batch
finisher (csrc/finisher.cu), which otherwise only see the segments of very
large inputs.  Adversarial small cases reach it this way: exact offset ties,
duplicates, signed zeros, integer lattices, circles, and chains that peel one
vertex per depth.  Bit-exact against the oracle and the golden hull cases.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np, torch
import paper_2510_09417_b200 as vq
import golden_io as G
from oracle import Oracle
from test_gpu_parity import random_instance, gpu_indices
torch.cuda.set_device(0)
O = Oracle()
bad = 0
# golden hull cases (produced by the reference library)
for name, xs, ys, want, _, _ in G.hull_cases():
    if len(xs) == 0:
        continue
    got = gpu_indices(vq, xs, ys)
    if not np.array_equal(got, np.asarray(want).astype(np.uint64)):
        print("MISMATCH golden", name); bad += 1
rng = np.random.default_rng(77)
for it in range(400):
    xs, ys = random_instance(rng, it)
    if len(xs) == 0:
        continue
    if not np.array_equal(gpu_indices(vq, xs, ys), O.hull_indices(xs, ys)):
        print("MISMATCH random", it, len(xs)); bad += 1
# chains that peel one vertex per depth (hundreds of depths in one finisher batch)
for m in (64, 300, 600, 760):
    i = np.arange(m)
    xs, ys = np.ldexp(1.0, i), np.ldexp(1.0, -i)
    if not np.array_equal(gpu_indices(vq, xs, ys), O.hull_indices(xs, ys)):
        print("MISMATCH pow2", m); bad += 1
# larger mixes: many finisher segments per batch, ties across segments
for seed in range(6):
    r = np.random.default_rng(seed)
    n = int(r.integers(3000, 60000))
    t = r.uniform(0, 2 * np.pi, n)
    rad = np.where(r.random(n) < 0.5, 1.0, r.uniform(0.9, 1.0, n))
    xs, ys = rad * np.cos(t), rad * np.sin(t)
    k = n // 7
    xs[:k], ys[:k] = np.round(xs[:k] * 64) / 64, np.round(ys[:k] * 64) / 64   # lattice points: exact ties
    xs[-k:], ys[-k:] = xs[k:2 * k], ys[k:2 * k]                              # duplicates
    if not np.array_equal(gpu_indices(vq, xs, ys), O.hull_indices(xs, ys)):
        print("MISMATCH mix", seed, n); bad += 1
s = vq.stats()
print("STATS", s["tail_launches"], s["finisher_segments"])
print("OK" if bad == 0 else "FAILED %d" % bad)
"""


def test_batch_finisher_small_inputs(tmp_path):
    env = dict(os.environ, VQHULL_TINY="0", VQHULL_KC="0", VQHULL_TAIL="0")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=1500, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    out = p.stdout.strip().splitlines()
    assert out and out[-1] == "OK", "\n".join(out[-20:])
    stats = [l for l in out if l.startswith("STATS")][-1].split()
    assert int(stats[1]) == 0 and int(stats[2]) > 0  # no tail kernel; the last hull used finisher segments
