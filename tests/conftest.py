import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libwhff_b200.so")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def hostcheck():
    """The device decoder/encoder headers compiled for the host."""
    import ctypes
    lib = os.path.join(ROOT, "tools", "libhostcheck.so")
    src = os.path.join(ROOT, "tools", "hostcheck.cpp")
    hdrs = [os.path.join(ROOT, "paper_1902_08018_b200", "csrc", h)
            for h in ("whff_decode.cuh", "whff_encode.cuh", "whff_relayout.cuh", "whff_packed.cuh")]
    if not os.path.exists(lib) or any(os.path.getmtime(p) > os.path.getmtime(lib) for p in hdrs + [src]):
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.run([cxx, "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                        "-Wno-unknown-pragmas", "-o", lib, src], check=True)
    L = ctypes.CDLL(lib)
    p, u64, i64, ci = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
    L.hc_decode_blocks.argtypes = [p, u64, p, p, i64, ci, ci] + [p] * 6
    L.hc_decompress.argtypes = [p, u64, p, p, i64, i64, ci, ci, p]
    L.hc_compress.argtypes = [p, i64, i64, ci, ctypes.c_double, p, p]
    L.hc_compress.restype = i64
    L.hc_encode_blocks.argtypes = [p] * 6 + [i64, ci, ci, p, p]
    L.hc_encode_blocks.restype = i64
    L.hc_relayout.argtypes = [p, p, p, p, i64, u64, ci, ci, ci]
    L.hc_decode_blocks_sf.argtypes = [p, u64, p, p, i64, ci, ci] + [p] * 6
    L.hc_pack.argtypes = [p] * 5 + [i64, i64] + [p] * 7 + [ci]
    L.hc_pack.restype = i64
    L.hc_unpack.argtypes = [p, p, p, p, i64, i64, i64, p, ci]
    L.hc_unpack.restype = i64
    return L


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    return load


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def golden_codec_cases(g):
    """Yield dicts of the reference's codec golden cases."""
    for i in range(int(g["n"][0])):
        k = f"c{i:03d}"
        name, kind, _ = g[k + "_meta"]
        yield {
            "name": str(name), "kind": str(kind), "param": float(g[k + "_param"][0]),
            "array": g[k + "_array"], "payload": g[k + "_payload"], "index": g[k + "_index"],
            "total_bits": int(g[k + "_total_bits"][0]),
            "dec": tuple(g[k + "_" + n] for n in ("mag", "neg", "emax", "raw", "raw_words", "consumed")),
            "words": g[k + "_words"], "ok": bool(g[k + "_ok"][0]),
        }


def mode_tuple(case):
    p = case["param"]
    return (case["kind"], int(p) if case["kind"] != "accuracy" else p)
