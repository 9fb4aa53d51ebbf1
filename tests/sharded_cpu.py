"""TEST INFRASTRUCTURE — CPU stand-ins for the sharded hull's device stages.

``CPUStages`` restates, with numpy and the oracle, what the sm_100a local
stage (``vqhull_cuda_shard_candidates``, csrc/shard.cu) and merge
(``vqhull_cuda_merge_candidates``, csrc/driver.cu Engine::merge) compute, so
that the host protocol of ``paper_2510_09417_b200.distributed`` (packing,
all-gather rounds, the margin retry, global indices) runs over gloo on CPU:

* local: the oracle's hull of the shard; the certificate keeps every point
  not proven deep inside a wedge triangle (c, v_i, v_{i+1}) of that hull by
  the margin 2^-32 max(M, floor) |chord|_1 (plain f64 evaluation: a few
  roundings of |chord| M, far below the margin); candidates sorted by index,
  packed behind the header {count, M_eff, A};
* merge: the header checks (count < 0 -> invalid input; A <= 2^12 min M_eff,
  else RetryWithFloor(A / 2^12)), the candidates in global-index order, the
  oracle's hull of them, mapped to global indices.
"""
from __future__ import annotations

import numpy as np
import torch


def _chord(ux, uy, wx, wy, mu):
    ex, ey = wx - ux, wy - uy
    fa, fb = -ey, ex
    fc = ey * ux - ex * uy
    fg = -mu * (np.abs(ex) + np.abs(ey)) - fc
    deg = (ex == 0) & (ey == 0)
    return fa, fb, np.where(deg, -np.inf, fg)


def certify(xs, ys, hull_idx, floor=0.0):
    """(keep mask, M_eff) — the local certificate."""
    n = xs.size
    hx, hy = xs[hull_idx], ys[hull_idx]
    K = hx.size
    if K < 3:
        return np.ones(n, dtype=bool), np.inf
    cx, cy = hx.mean(), hy.mean()
    M = max(np.abs(hx).max(), np.abs(hy).max(), abs(cx), abs(cy))
    Me = max(M, floor)
    mu = 2.0 ** -32 * Me
    nx, ny = np.roll(hx, -1), np.roll(hy, -1)
    ea, eb, eg = _chord(hx, hy, nx, ny, mu)           # v_j -> v_{j+1}
    ra, rb, rg = _chord(cx, cy, hx, hy, mu)           # c -> v_j
    ba, bb, bg = _chord(hx, hy, cx, cy, mu)           # v_j -> c
    if not np.all(ea * cx + eb * cy < eg):            # c must be inside conv(Q)
        return np.ones(n, dtype=bool), np.inf
    th = np.arctan2(hy - cy, hx - cx)
    order = np.argsort(th, kind="stable")
    phi = np.arctan2(ys - cy, xs - cx)
    t = np.searchsorted(th[order], phi, side="right")
    i = order[t % K]                                   # larger-angle vertex of the wedge
    j = (i + 1) % K
    inside = ((ra[i] * xs + rb[i] * ys < rg[i]) & (ea[i] * xs + eb[i] * ys < eg[i])
              & (ba[j] * xs + bb[j] * ys < bg[j]) & (np.abs(xs) <= M) & (np.abs(ys) <= M))
    return ~inside, Me


class CPUStages:
    def __init__(self):
        from oracle import Oracle

        self.O = Oracle()
        self._last = None

    def local(self, x, y, offset, cap, floor):
        xs, ys = x.numpy(), y.numpy()
        n = xs.size
        hdr = [0.0, np.inf, 0.0]
        rows = np.zeros((0, 3))
        if n:
            if not (np.all(np.isfinite(xs)) and np.all(np.isfinite(ys))):
                hdr[0] = -1.0
            else:
                h = self.O.hull_indices(xs, ys).astype(np.int64)
                keep, me = certify(xs, ys, h, floor)
                idx = np.nonzero(keep)[0]  # ascending = sorted by global index
                rows = np.stack([xs[idx], ys[idx], (idx + offset).astype(np.int64).view(np.float64)], 1)
                hdr = [float(idx.size), me, float(max(np.abs(xs).max(), np.abs(ys).max()))]
        self._last = (hdr, rows)
        return self._pack(cap), int(max(hdr[0], 0)), 0

    def _pack(self, cap):
        hdr, rows = self._last
        pack = np.zeros((cap + 1, 3))
        pack[0] = hdr
        m = min(rows.shape[0], cap)
        pack[1:1 + m] = rows[:m]
        return torch.from_numpy(pack)

    def repack(self, pack):
        pack.copy_(self._pack(pack.shape[0] - 1))

    def merge(self, packs):
        from paper_2510_09417_b200 import RetryWithFloor

        P = packs.numpy()
        counts = P[:, 0, 0]
        if np.any(counts < 0):
            raise ValueError("a shard holds a non-finite coordinate")
        A, Mmin = P[:, 0, 2].max(), P[:, 0, 1].min()
        if not A <= 2.0 ** 12 * Mmin:
            raise RetryWithFloor(A * 2.0 ** -12)
        rows = np.concatenate([P[r, 1:1 + int(c)] for r, c in enumerate(counts)])
        g = rows[:, 2].copy().view(np.int64)
        assert np.all(np.diff(g) > 0)
        h = self.O.hull_indices(rows[:, 0].copy(), rows[:, 1].copy()).astype(np.int64)
        return torch.from_numpy(g[h]), 0
