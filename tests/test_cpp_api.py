"""The C++ host API (include/vqhull_b200.hpp) builds against the library, and
— on a GPU — passes the reference's own C++ test cases (tests/cpp/)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2510_09417_b200", "lib")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "test_cpp_api")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", LIBDIR, "-lvqhull_b200",
           f"-Wl,-rpath,{LIBDIR}", "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_api_builds(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path, cuda):
    out = subprocess.run([build(tmp_path)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "all checks passed" in out.stdout


@pytest.mark.gpu
def test_plain_c_caller_without_torch(tmp_path, cuda):
    """The drop-in: a C program (no torch, no cudart of its own) calls
    vqhull_compute on tiny and odd sizes; runs in a fresh process."""
    src = os.path.join(str(tmp_path), "c_caller.c")
    with open(src, "w") as f:
        f.write(r'''
#include <stdio.h>
#include "vqhull_b200.h"
int main(void) {
    double xs[] = {0, 4, 4, 0, 2, 0}, ys[] = {0, 0, 4, 4, 2, 0};
    size_t idx[6], cnt = 0;
    if (vqhull_compute(xs, ys, 6, 1, idx, &cnt) || cnt != 4 || idx[0] != 0 || idx[1] != 3) return 2;
    for (size_t n = 1; n <= 6; ++n)
        if (vqhull_compute(xs, ys, n, 1, idx, &cnt)) return 3;
    puts("c caller ok");
    return 0;
}
''')
    exe = os.path.join(str(tmp_path), "c_caller")
    subprocess.run(["gcc", "-O1", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-lvqhull_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "c caller ok" in out.stdout, (out.returncode, out.stderr)


@pytest.mark.gpu
def test_plain_c_caller_sharded_path(tmp_path, cuda, vq, oracle):
    """A plain C caller with VQHULL_GPUS set (the multi-device drop-in path,
    here with 1 and 3 shards) gets the reference's golden list for config 1."""
    import numpy as np

    import golden_io as G

    cfg = G.configs()["config1_disk_1e6_s1"]
    xs, ys = vq.generate(cfg["kind"], cfg["n"], cfg["seed"])
    pts = os.path.join(str(tmp_path), "pts.bin")
    np.concatenate([xs, ys]).tofile(pts)
    src = os.path.join(str(tmp_path), "c_sharded.c")
    with open(src, "w") as f:
        f.write(r'''
#include <stdio.h>
#include <stdlib.h>
#include "vqhull_b200.h"
int main(int argc, char** argv) {
    size_t n = (size_t)atoll(argv[2]);
    double* p = malloc(2 * n * sizeof(double));
    size_t* idx = malloc(n * sizeof(size_t));
    FILE* f = fopen(argv[1], "rb");
    if (!p || !idx || !f || fread(p, sizeof(double), 2 * n, f) != 2 * n) return 2;
    fclose(f);
    size_t cnt = 0;
    int rc = vqhull_compute(p, p + n, n, 1, idx, &cnt);
    if (rc) return 10 + rc;
    FILE* o = fopen(argv[3], "wb");
    fwrite(idx, sizeof(size_t), cnt, o);
    fclose(o);
    return 0;
}
''')
    exe = os.path.join(str(tmp_path), "c_sharded")
    subprocess.run(["gcc", "-O1", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR, "-lvqhull_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    for g in ("1", "3"):
        outp = os.path.join(str(tmp_path), f"idx{g}.bin")
        env = dict(os.environ, VQHULL_GPUS=g)
        r = subprocess.run([exe, pts, str(cfg["n"]), outp], capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, (r.returncode, r.stderr)
        got = np.fromfile(outp, dtype=np.uint64)
        assert got.size == cfg["h"]
        assert f"{oracle.fnv1a64(got):016x}" == cfg["fnv1a64_u64le"]
