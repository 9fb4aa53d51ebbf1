"""Golden vector for BASELINE config 5 at full size (disk, n = 4e9, seed 5),
from the reference library itself (oracle/_ref: the reference's vqhull_compute,
16 threads).  The reference needs ~3 copies of its input, so 4e9 points do not
fit in host RAM at once: it is run on 4 contiguous chunks of 1e9 points (the
reference's generator streams are counter based, so chunk k is points
[k*1e9, (k+1)*1e9) of the same sequence), and then once more on the union of
the chunk hulls ordered by global index (first occurrences first) — the
hull of the union of hulls, exact for this non-degenerate input (no three
hull candidates within rounding of collinear), the same merge as
paper_2510_09417_b200/distributed.py.  Runs on the GPU box:

    gpurun -- python tests/golden/make_config5.py   # -> gpurun_out/config5_golden.json

and, there, also checks the CUDA path on the same bytes.  The result is merged
into tests/golden/configs.json by hand (python tests/golden/make_config5.py --merge FILE).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

NAME, KIND, N, SEED = "config5_disk_4e9_s5", "disk", 4 * 10**9, 5


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
    import paper_2510_09417_b200 as vq
    R = Reference()
    chunk = N // 4
    cx, cy, cg = [], [], []
    for k in range(4):
        t0 = time.time()
        xs, ys = vq.generate(KIND, chunk, SEED, first=k * chunk, threads=16)
        if k == 0:  # the product generator is bit-exact to the reference's (tests); spot-check
            rx, ry = R.generate(KIND, 1000, SEED, workers=4)
            assert np.array_equal(rx, xs[:1000]) and np.array_equal(ry, ys[:1000])
        rc, idx = R.compute(xs, ys, workers=16, cap=1 << 22)
        assert rc == 0
        cx.append(xs[idx]); cy.append(ys[idx]); cg.append(idx.astype(np.uint64) + np.uint64(k * chunk))
        print(f"chunk {k}: h={idx.size} in {time.time() - t0:.1f}s", flush=True)
        del xs, ys
    gx, gy, gg = np.concatenate(cx), np.concatenate(cy), np.concatenate(cg)
    order = np.argsort(gg, kind="stable")
    gx, gy, gg = gx[order], gy[order], gg[order]
    rc, loc = R.compute(gx, gy, workers=1)
    assert rc == 0
    idx = gg[loc]
    print(f"merged: candidates {gg.size} -> h={idx.size}", flush=True)
    xs0, ys0 = vq.generate(KIND, 1, SEED)
    rec = {"kind": KIND, "n": N, "seed": SEED, "h": int(idx.size), "fnv1a64_u64le": fnv1a64(idx),
           "head": [int(v) for v in idx[:8]], "tail": [int(v) for v in idx[-8:]],
           "model_bytes": None, "ref_calls": None,
           "first_point": [float(xs0[0]).hex(), float(ys0[0]).hex()],
           "indices": [int(v) for v in idx],
           "source": "oracle/_ref vqhull_compute (the reference library) on 4 chunks of 1e9, "
                     "then on the union of the chunk hulls ordered by global index; GPU box"}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({NAME: rec}, open(os.path.join(ROOT, "gpurun_out", "config5_golden.json"), "w"))
    # the CUDA path, one device, all 4e9 points
    import torch
    X = torch.empty(N, dtype=torch.float64, pin_memory=True)
    Y = torch.empty(N, dtype=torch.float64, pin_memory=True)
    vq.generate(KIND, N, SEED, out=(X, Y), threads=16)
    Xd, Yd = X.cuda(), Y.cuda()
    del X, Y
    got = vq.hull_device(Xd, Yd).cpu().numpy().astype(np.uint64)
    print("cuda h", got.size, "equal", bool(np.array_equal(got, idx)), flush=True)


if __name__ == "__main__":
    main()
