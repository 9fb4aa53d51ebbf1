"""Generate tests/golden/ref_points.{bin,txt}: seeded points (incl. signed
zeros, large integers, tiny and huge magnitudes) as VQH1, and the reference
library's own text rendering of them (make_ref_text.cpp).  Needs
/root/reference and oracle/_ref/libvqhull_ref.so (run `__graft_entry__.build()`
first); the fixtures are committed, so the tests do not."""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2510_09417_b200.io import save_vqh1  # noqa: E402

r = np.random.default_rng(11)
xs = r.standard_normal(400) * 10.0 ** r.integers(-30, 30, 400)
ys = r.uniform(-1, 1, 400) * 10.0 ** r.integers(-8, 24, 400)
xs[:8] = [0.0, -0.0, 1e22, 123456.0, 9007199254740993.0, 5e-324, 0.001, 1e-4]
ys[:8] = [-0.0, 100.0, 1e5, 2.5e10, 0.1, 1.7976931348623157e308, 3.0, -12300.0]
bin_path = os.path.join(HERE, "ref_points.bin")
txt_path = os.path.join(HERE, "ref_points.txt")
save_vqh1(bin_path, xs, ys)
exe = "/tmp/make_ref_text"
lib = os.path.join(ROOT, "oracle", "_ref")
subprocess.check_call(["g++", "-std=c++20", "-O1", os.path.join(HERE, "make_ref_text.cpp"),
                       "-I/root/reference/proj/include", "-L" + lib, "-lvqhull_ref",
                       "-Wl,-rpath," + lib, "-o", exe])
subprocess.check_call([exe, bin_path, txt_path])
print("wrote", bin_path, txt_path)
