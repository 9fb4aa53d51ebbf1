"""VQH1 loading (reference: proj/src/io.cpp:67-88; tests: test_dataset_io.cpp:122-199)."""
import os
import struct

import numpy as np
import pytest

from paper_2510_09417_b200.io import LoadError, load_vqh1, load_vqh1_device, save_vqh1


def _pts(n, seed=0):
    r = np.random.default_rng(seed)
    return r.standard_normal(n), r.standard_normal(n)


def test_round_trip_byte_identical(tmp_path):
    xs, ys = _pts(1000)
    a, b = tmp_path / "a.bin", tmp_path / "b.bin"
    save_vqh1(str(a), xs, ys)
    x2, y2 = load_vqh1(str(a))
    save_vqh1(str(b), x2, y2)
    assert a.read_bytes() == b.read_bytes()
    assert np.array_equal(x2, xs) and np.array_equal(y2, ys)
    raw = a.read_bytes()
    assert raw[:4] == b"VQH1" and struct.unpack("<Q", raw[4:12])[0] == 1000
    assert len(raw) == 12 + 16 * 1000


def test_empty_round_trip(tmp_path):
    p = tmp_path / "e.bin"
    save_vqh1(str(p), np.empty(0), np.empty(0))
    xs, ys = load_vqh1(str(p))
    assert xs.size == 0 and ys.size == 0


def test_malformed(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"VQH2" + struct.pack("<Q", 0))
    with pytest.raises(LoadError, match="bad magic"):
        load_vqh1(str(p))
    p.write_bytes(b"VQH1" + b"\0\0")
    with pytest.raises(LoadError, match="truncated header"):
        load_vqh1(str(p))
    xs, ys = _pts(10)
    save_vqh1(str(p), xs, ys)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(LoadError, match="truncated payload"):
        load_vqh1(str(p))
    ys[7] = np.nan
    save_vqh1(str(p), xs, ys)
    with pytest.raises(LoadError, match="non-finite coordinate at point 7"):
        load_vqh1(str(p))
    with pytest.raises(LoadError, match="cannot open"):
        load_vqh1(str(tmp_path / "definitely_missing_file.bin"))


@pytest.mark.gpu
def test_device_load_then_hull(tmp_path):
    import torch

    import paper_2510_09417_b200 as vq

    xs, ys = vq.generate("disk", 200_000, 1)
    p = tmp_path / "d.bin"
    save_vqh1(str(p), xs, ys)
    X, Y = load_vqh1_device(str(p))
    assert X.is_cuda and torch.equal(X.cpu(), torch.from_numpy(xs))
    assert torch.equal(Y.cpu(), torch.from_numpy(ys))
    got = vq.hull_device(X, Y).cpu().numpy()
    rc, ref = vq.vqhull_compute(xs, ys)
    assert rc == 0 and np.array_equal(got.astype(np.int64), ref.astype(np.int64))
    ys[3] = np.inf
    save_vqh1(str(p), xs, ys)
    with pytest.raises(LoadError, match="point 3"):
        load_vqh1_device(str(p))
