"""Profiling driver: one paper-width slit, fused decode+GEMV launched a few
times (run under ncu).  Usage: python tools/prof_fused.py [mode] [eval] [slits]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import codec, synth  # noqa: E402
from paper_1902_08018_b200.executor import GemvPlan  # noqa: E402
from paper_1902_08018_b200 import _lib  # noqa: E402

mode_s = sys.argv[1] if len(sys.argv) > 1 else "rate:8"
ev = sys.argv[2] if len(sys.argv) > 2 else "exact"
nsl = int(sys.argv[3]) if len(sys.argv) > 3 else 4
layout = sys.argv[4] if len(sys.argv) > 4 else "reference"
kind, p = mode_s.split(":")
mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
        "accuracy": codec.FixedAccuracy}[kind](int(p) if kind != "accuracy" else float(p))
spec = synth.Spec(grid_rows=608, grid_cols=608, S=256000, K=378 * nsl, M=378, seed=7)
streams = []
for s in range(nsl):
    rows = synth.deformation_rows(spec, 0, 0.3, s * 378, (s + 1) * 378, device="cuda")
    ds = codec.compress_device(rows, mode)
    if layout != "reference":
        ds.relayout(layout)
    streams.append(ds)
v = torch.rand(256000, device="cuda")
y = torch.zeros(378 * nsl, device="cuda")
plan = GemvPlan([(ds, v, y[i * 378:(i + 1) * 378], 0, 378) for i, ds in enumerate(streams)],
                "mixed", ev)
st = _lib.status_word()
for _ in range(3):
    plan.launch(st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    plan.launch(st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{mode_s} {ev} {layout} slits={nsl}: {ms:.3f} ms/launch, {plan.bytes_read / ms / 1e6:.1f} GB/s, "
      f"blocks={plan.n_blocks}")
