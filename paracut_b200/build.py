"""Build the sm_100a shared library in-tree: paracut_b200/_lib/libparacut_b200.so.

    python -m paracut_b200.build

nvcc cross-compiles for sm_100a without a GPU.  -fmad=false keeps every fp64
multiply and add separately rounded, which the bitwise-parity contract with
the reference's numba kernels needs (no fastmath there, _kernels.py:3-5).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "paracut_b200.cu")
OUT_DIR = os.path.join(HERE, "_lib")
OUT = os.path.join(OUT_DIR, "libparacut_b200.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith((".cu", ".cuh"))]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    hdr = os.path.join(os.path.dirname(HERE), "include", "paracut_b200.h")
    return all(os.path.getmtime(s) <= t for s in sources() + [hdr, __file__])


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(OUT_DIR, exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), "-O3", "-std=c++17", ARCH, "-lineinfo", "-fmad=false",
           "-Xcompiler", "-fPIC", "-shared", "-o", tmp, SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed (%d)" % res.returncode)
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
