"""Builds the native library libvqhull_b200.so in-tree (sm_100a only).

nvcc -gencode arch=compute_100a,code=sm_100a, -O3 -lineinfo, --fmad=false
(no FMA contraction anywhere: the reference builds with -ffp-contract=off,
CMakeLists.txt:17), static cudart, host code with -ffp-contract=off.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libvqhull_b200.so")
LIB_DBG = os.path.join(LIBDIR, "libvqhull_b200_dbg.so")
SOURCES = ["device.cu", "shard.cu", "driver.cu", "dataset.cpp"]  # device.cu includes kernels.cu, partition.cu, tail.cu
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def flags(extra=()):
    return [*ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
            "-Xcompiler", "-fPIC,-ffp-contract=off,-O3", "-I", os.path.join(ROOT, "include"),
            *extra]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "vqhull_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False,
          defines=(), suffix: str = "") -> str:
    """Build lib/libvqhull_b200.so (or lib/libvqhull_b200_dbg.so with device
    bounds checks, -DVQB_DEBUG)."""
    lib = LIB_DBG if debug else LIB
    if suffix:
        lib = os.path.join(LIBDIR, f"libvqhull_b200_{suffix}.so")
    if not force and not debug and not suffix and not stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + (".dbg.o" if debug else ".o"))
        extra = (["-DVQB_DEBUG"] if debug else []) + [f"-D{d}" for d in defines]
        obj = obj.replace(".o", f".{suffix}.o") if suffix else obj
        cmd = [NVCC, *flags(extra), "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "c++"]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs, "-lpthread"],
                   check=True)
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    suf = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--suffix=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                defines=defs, suffix=suf))
