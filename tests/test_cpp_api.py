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
