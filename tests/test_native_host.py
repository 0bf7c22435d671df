"""A non-Python host of the C ABI: examples/whff_gemv_file.c reads a WHFZ
file (the reference's container) and runs the fused decode+GEMV through
include/whff_b200.h only.  CPU: it compiles and links against the library.
GPU: its products equal the Python layer's (same kernels, same order)."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

LIB_DIR = os.path.join(ROOT, "paper_1902_08018_b200")
CUDA = "/usr/local/cuda"


def build(tmp_path):
    cc = shutil.which("gcc") or "/usr/bin/gcc"
    exe = tmp_path / "whff_gemv_file"
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(CUDA, "include"), "-o", str(exe),
                    os.path.join(ROOT, "examples", "whff_gemv_file.c"),
                    "-L", LIB_DIR, "-lwhff_b200", "-L", os.path.join(CUDA, "lib64"), "-lcudart"],
                   check=True)
    return exe


@pytest.mark.skipif(not os.path.exists(os.path.join(LIB_DIR, "libwhff_b200.so")),
                    reason="libwhff_b200.so not built")
def test_native_host_builds(tmp_path):
    assert build(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["rate", "accuracy"])
@pytest.mark.parametrize("evaluation", ["exact", "coefficient"])
def test_native_host_matches_python(tmp_path, kind, evaluation):
    import torch
    from paper_1902_08018_b200 import codec, synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=5000, K=61, M=61, seed=5)
    C = synth.deformation_rows(spec, 1, 0.4, 0, 61)
    mode = codec.FixedRate(8) if kind == "rate" else codec.FixedAccuracy(1e-12)
    s = codec.compress(C, mode)
    path = tmp_path / "slit.whfz"
    codec.save_stream(path, s)
    exe = build(tmp_path)
    env = dict(os.environ, LD_LIBRARY_PATH=f"{LIB_DIR}:{CUDA}/lib64:" + os.environ.get("LD_LIBRARY_PATH", ""))
    args = [str(exe), str(path), "--ramp"] + (["--coefficient"] if evaluation == "coefficient" else [])
    out = subprocess.run(args, capture_output=True, text=True, env=env, timeout=120)
    assert out.returncode == 0, out.stderr
    rows, total, y0, yl = out.stdout.split()
    ds = codec.DeviceStream.from_host(codec.load_stream(path)).relayout("skeleton-first")
    v = torch.tensor([(j % 7 + 1) / 8.0 for j in range(5000)], dtype=torch.float32, device="cuda")
    y = ds.gemv(v, evaluation=evaluation).cpu().numpy()
    assert int(rows) == 61
    # %.9g identifies a binary32 uniquely
    assert np.float32(float(y0)) == y[0] and np.float32(float(yl)) == y[-1]
    assert abs(float(total) - float(y.astype(np.float64).sum())) <= 1e-12 * abs(float(total)) + 1e-30
