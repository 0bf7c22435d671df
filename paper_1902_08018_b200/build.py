"""Build libwhff_b200.so in-tree with nvcc for sm_100a.

The shared library is the product (the C ABI declared in include/whff_b200.h);
Python only binds it with ctypes.  ``python -m paper_1902_08018_b200.build``
or ``__graft_entry__.build()`` runs this.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libwhff_b200.so")
SOURCES = [os.path.join(CSRC, "whff_b200.cu")]
HEADERS = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) + [
    os.path.join(ROOT, "include", "whff_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    # no --use_fast_math: dequantisation relies on IEEE subnormals and
    # the GEMV policies on un-contracted binary32 products
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the B200 extension cannot be built")


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    extra = os.environ.get("WHFF_NVCC_EXTRA", "").split()   # tuning sweeps (-D...)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp",
           *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    env = dict(os.environ)
    # the system gcc is the supported nvcc host compiler in this image
    if os.path.exists("/usr/bin/gcc"):
        env["PATH"] = "/usr/bin:" + env.get("PATH", "")
    subprocess.run(cmd, check=True, env=env)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
