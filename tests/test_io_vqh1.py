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


# ---- text format (io.cpp:26-65, 100-121; test_dataset_io.cpp:122-206) ----

from paper_2510_09417_b200.io import format_for_path, read_points, to_chars, write_points  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "to_chars.txt")


def test_to_chars_matches_libstdcxx_golden():
    n = 0
    with open(GOLDEN) as f:
        for line in f:
            h, want = line.split()
            v = struct.unpack("<d", bytes.fromhex(h)[::-1])[0]
            assert to_chars(v) == want, (h, want)
            n += 1
    assert n > 5000


@pytest.mark.parametrize("ext", [".txt", ".pbbs", ".bin"])
def test_text_and_binary_round_trips_byte_identical(tmp_path, ext):
    xs, ys = _pts(500, 3)
    xs[:4] = [0.0, -0.0, 1e22, 123456.0]
    a, b = tmp_path / ("a" + ext), tmp_path / ("b" + ext)
    write_points(str(a), xs, ys)
    x2, y2 = read_points(str(a))
    assert np.array_equal(x2, xs) and np.array_equal(y2, ys)
    write_points(str(b), x2, y2)
    assert a.read_bytes() == b.read_bytes()
    if ext != ".bin":
        assert a.read_bytes().startswith(b"pbbs_sequencePoint2d\n")


def test_text_and_binary_loads_equal(tmp_path):
    xs, ys = _pts(300, 4)
    write_points(str(tmp_path / "x.txt"), xs, ys)
    write_points(str(tmp_path / "x.bin"), xs, ys)
    t = read_points(str(tmp_path / "x.txt"))
    b = read_points(str(tmp_path / "x.bin"))
    assert np.array_equal(t[0], b[0]) and np.array_equal(t[1], b[1])


def test_text_empty_set_and_crlf(tmp_path):
    p = tmp_path / "e.txt"
    write_points(str(p), np.empty(0), np.empty(0))
    assert p.read_bytes() == b"pbbs_sequencePoint2d\n"
    assert read_points(str(p))[0].size == 0
    p.write_bytes(b"pbbs_sequencePoint2d\r\n1 2\r\n\r\n\t-3.5   4e-1\r\n")
    xs, ys = read_points(str(p))
    assert xs.tolist() == [1.0, -3.5] and ys.tolist() == [2.0, 0.4]


def test_text_malformed(tmp_path):
    p = tmp_path / "m.txt"
    p.write_bytes(b"")
    with pytest.raises(LoadError, match="empty file"):
        read_points(str(p))
    p.write_bytes(b"not_a_header\n1 2\n")
    with pytest.raises(LoadError, match='unrecognized header "not_a_header"'):
        read_points(str(p))
    p.write_bytes(b"pbbs_sequencePoint2d\n1 2\n3 x\n")
    with pytest.raises(LoadError, match="malformed coordinate on line 3"):
        read_points(str(p))
    p.write_bytes(b"pbbs_sequencePoint2d\n1 2\n3 inf\n")
    with pytest.raises(LoadError, match="non-finite coordinate at point 1"):
        read_points(str(p))


def test_format_for_path():
    assert format_for_path("points.txt") == "text"
    assert format_for_path("points.pbbs") == "text"
    assert format_for_path("points.bin") == "binary"
    assert format_for_path("points") == "binary"
    assert format_for_path("dir.txt/points") == "binary"


def test_text_writer_matches_reference_library(tmp_path):
    """ref_points.txt was written by the reference's own write_points
    (tests/golden/make_ref_text.py) from ref_points.bin."""
    g = os.path.dirname(GOLDEN)
    xs, ys = read_points(os.path.join(g, "ref_points.bin"))
    out = tmp_path / "ours.txt"
    write_points(str(out), xs, ys)
    with open(os.path.join(g, "ref_points.txt"), "rb") as f:
        assert out.read_bytes() == f.read()
    t = read_points(os.path.join(g, "ref_points.txt"))
    assert np.array_equal(t[0], xs) and np.array_equal(t[1], ys)
    assert np.array_equal(np.signbit(t[0]), np.signbit(xs))
