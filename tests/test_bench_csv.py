"""bench.py --csv: the reference's bench CSV schema (proj/src/bench.cpp:156-199)."""
import csv
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_csv_header_matches_reference_schema():
    b = _bench()
    assert b.CSV_HEADER.split(",") == [
        "kind", "n", "seed", "workers", "block_size", "lanes", "simd", "write_combining", "reps",
        "rep", "seconds", "mean_seconds", "stddev_seconds", "model_bytes",
        "bandwidth_gbps", "baseline_gbps", "hull_vertices", "joules"]


def test_csv_rows(tmp_path):
    b = _bench()
    p = tmp_path / "r.csv"
    rows = [(0.001, 1_600_000_000), (0.003, 1_600_000_000)]
    b.write_csv(str(p), "square", 10**8, 2, 1, rows, 42, 6538.6)
    with open(p) as f:
        recs = list(csv.DictReader(f))
    assert len(recs) == 2
    assert [int(r["rep"]) for r in recs] == [1, 2]
    r = recs[0]
    assert r["kind"] == "square" and r["n"] == "100000000" and r["seed"] == "2"
    assert int(r["reps"]) == 2 and int(r["hull_vertices"]) == 42 and r["joules"] == ""
    assert float(r["mean_seconds"]) == 0.002
    # sample standard deviation, as stddev_of (bench.cpp:84-89)
    assert abs(float(r["stddev_seconds"]) - 0.0014142135623730952) < 1e-15
    assert float(r["bandwidth_gbps"]) == 1_600_000_000 / 0.002 / 1e9
    one = tmp_path / "one.csv"
    b.write_csv(str(one), "disk", 10, 1, 1, rows[:1], 5, 1.0)
    with open(one) as f:
        assert float(next(csv.DictReader(f))["stddev_seconds"]) == 0.0
