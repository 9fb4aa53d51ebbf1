"""Golden vector for BASELINE config 5 at full size (disk, n = 4e9, seed 5)
from ONE global run of the reference library (oracle/_ref: the reference's
own convex_hull over all 4e9 points, 16 worker threads) — no chunking and no
merge assumption.  The reference's vqhull_compute would need its N-entry hash
map (~160 GB at 4e9) on top of the input, so the index mapping is restated:
the reference's clockwise vertex coordinates (convex_hull) are mapped to the
first input index holding each of them (vqhull_c.cpp:46-61 semantics: equal
coordinates compare with ==, so +0.0 and -0.0 match) by one chunked pass over
the input.  Peak host memory ~130 GB (the input, the reference's own copy of
it); runs on the GPU box, whose host has ~196 GB:

    gpurun -- python tests/golden/make_config5_global.py   # -> gpurun_out/config5_global.json

and --merge FILE updates tests/golden/configs.json.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

NAME, KIND, N, SEED = "config5_disk_4e9_s5", "disk", 4 * 10**9, 5


def first_occurrence(xs, ys, hx, hy, chunk=1 << 27):
    """For every vertex (hx[k], hy[k]) the smallest i with xs[i] == hx[k] and
    ys[i] == hy[k] (one pass over the input, chunked)."""
    h = hx.size
    order = np.lexsort((hy, hx))  # vertices sorted by (x, y)
    sx, sy = hx[order] + 0.0, hy[order] + 0.0  # (+0.0: -0.0 and +0.0 compare equal)
    found = np.full(h, np.iinfo(np.uint64).max, dtype=np.uint64)
    for a in range(0, xs.size, chunk):
        x = xs[a:a + chunk] + 0.0
        pos = np.minimum(np.searchsorted(sx, x), h - 1)
        cand = np.nonzero(sx[pos] == x)[0]
        if cand.size == 0:
            continue
        for i in cand:
            xi, yi = x[i], ys[a + i] + 0.0
            lo = np.searchsorted(sx, xi, "left")
            hi_ = np.searchsorted(sx, xi, "right")
            for k in range(lo, hi_):
                if sy[k] == yi and found[k] == np.iinfo(np.uint64).max:
                    found[k] = a + i
    out = np.empty(h, dtype=np.uint64)
    out[order] = found
    assert np.all(out != np.iinfo(np.uint64).max), "a hull vertex was not found in the input"
    return out


def fnv1a64(idx):
    from oracle import Oracle
    return f"{Oracle().fnv1a64(idx):016x}"


def main():
    if "--merge" in sys.argv:
        src = sys.argv[sys.argv.index("--merge") + 1]
        new = json.load(open(src))
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs.json")
        data = json.load(open(path))
        data[NAME] = new[NAME]
        json.dump(data, open(path, "w"), indent=1)
        print("merged", NAME)
        return
    from oracle import Reference
    R = Reference()
    threads = os.cpu_count() or 16
    t0 = time.time()
    xs, ys = R.generate(KIND, N, SEED, workers=threads)  # the reference's own generator
    print(f"generated {N} points in {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    hx, hy = R.convex_hull(xs, ys, workers=threads, cap=1 << 20)
    print(f"reference convex_hull: h={hx.size} in {time.time() - t0:.1f}s", flush=True)
    t0 = time.time()
    idx = first_occurrence(xs, ys, hx, hy)
    print(f"first occurrences in {time.time() - t0:.1f}s", flush=True)
    rec = {"kind": KIND, "n": N, "seed": SEED, "h": int(idx.size), "fnv1a64_u64le": fnv1a64(idx),
           "head": idx[:8].tolist(), "tail": idx[-8:].tolist(), "model_bytes": None, "ref_calls": None,
           "first_point": 2, "indices": idx.tolist(),
           "source": "oracle/_ref convex_hull (the reference library) over all 4e9 points in one run, "
                     "16 workers, vertex coordinates mapped to first input indices "
                     "(tests/golden/make_config5_global.py); GPU box"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "config5_global.json"), "w") as f:
        json.dump({NAME: rec}, f)
    old = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs.json"))).get(NAME)
    if old:
        print("matches the previous (chunk-merge) golden:", old.get("indices") == rec["indices"], flush=True)
    print(f"h={rec['h']} fnv={rec['fnv1a64_u64le']}", flush=True)


if __name__ == "__main__":
    main()
