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
SOURCES = [os.path.join(CSRC, f) for f in ("whff_b200.cu", "whff_pack.cu", "whff_packed.cu")]
HEADERS = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) + [
    os.path.join(ROOT, "include", "whff_b200.h")]
OBJDIR = os.path.join(HERE, "build")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    # no --use_fast_math: dequantisation relies on IEEE subnormals and
    # the GEMV policies on un-contracted binary32 products
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the B200 extension cannot be built")


def _obj(src):
    return os.path.join(OBJDIR, os.path.basename(src) + ".o")


def _newer(path, deps):
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    return any(os.path.getmtime(p) > t for p in deps)


def stale():
    if not os.path.exists(LIB):
        return True
    return _newer(LIB, SOURCES + HEADERS)


def build(force=False, verbose=False):
    """Compile each translation unit (only the stale ones) and link the .so."""
    if not force and not stale():
        return LIB
    extra = os.environ.get("WHFF_NVCC_EXTRA", "").split()   # tuning sweeps (-D...)
    env = dict(os.environ)
    # the system gcc is the supported nvcc host compiler in this image
    if os.path.exists("/usr/bin/gcc"):
        env["PATH"] = "/usr/bin:" + env.get("PATH", "")
    os.makedirs(OBJDIR, exist_ok=True)
    procs = []
    for src in SOURCES:
        obj = _obj(src)
        if force or extra or _newer(obj, [src] + HEADERS):
            cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj + ".tmp", src]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            procs.append((subprocess.Popen(cmd, env=env), obj))
    for p, obj in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc " + obj)
        os.replace(obj + ".tmp", obj)
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB + ".tmp",
           *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, env=env)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
