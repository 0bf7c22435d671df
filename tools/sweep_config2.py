"""BASELINE configs[1]: mid-size synthetic compressed matrix (4,096 x 262,144,
1.07 G values) -- one fused decode+GEMV per mode and evaluation on one B200,
against the HBM roofline.  Prints one JSON line per case.
Usage: python tools/sweep_config2.py [rows] [cols] [layout: packed | skeleton-first]

roofline_frac: the launch's own bytes (packed copy, or payload + index) over
the HBM peak; reference_stream_frac: the WHFZ stream bytes over the same time."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import _lib, codec, synth  # noqa: E402
from paper_1902_08018_b200.executor import GemvPlan  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
layout = sys.argv[3] if len(sys.argv) > 3 else "packed"
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    peak = 6650.0   # B200_PROFILING.md fallback
spec = synth.Spec(grid_rows=608, grid_cols=608, S=cols, K=rows, M=378, seed=11)
C = torch.empty((rows, cols), dtype=torch.float32, device="cuda")
for r0 in range(0, rows, 512):                       # generated in row bands
    C[r0:r0 + 512] = synth.deformation_rows(spec, 2, 1.1, r0, min(rows, r0 + 512), device="cuda")
v = torch.rand(cols, device="cuda")
st = _lib.status_word()
modes = [codec.FixedRate(4), codec.FixedRate(8), codec.FixedRate(16), codec.FixedPrecision(17),
         codec.FixedAccuracy(1e-12)]
words = torch.empty_like(C)
for mode in modes:
    ds = codec.compress_device(C, mode)
    if layout == "packed":
        ds.pack()
    else:
        ds.relayout(layout)
    # decode-only (codec.decompress on the device: bit-exact binary32 words to HBM)
    for _ in range(2):
        ds.decode(out=words, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ds.decode(out=words, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    comp = ds.payload_bytes + ds.index_bytes
    print(json.dumps({"config": "configs[1] mid-size sweep", "shape": [rows, cols], "mode": repr(mode),
                      "evaluation": "decode-only (whff_decode)", "compressed_bytes": comp,
                      "bpv": round(8 * comp / (rows * cols), 3), "ms": round(ms, 4),
                      "compressed_gbs": round(comp / ms / 1e6, 1), "gflops": None,
                      "decoded_gbs": round(4 * rows * cols / ms / 1e6, 1),
                      "roofline_frac": round((comp + 4 * rows * cols) / ms / 1e6 / peak, 4)}),
          flush=True)
    for ev in ("coefficient", "exact"):
        y = torch.empty(rows, device="cuda")
        plan = GemvPlan([(ds, v, y, 0, rows)], "mixed", ev)
        for _ in range(3):
            plan.launch(st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for _ in range(n):
            plan.launch(st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        comp = ds.payload_bytes + ds.index_bytes
        print(json.dumps({
            "config": "configs[1] mid-size sweep", "shape": [rows, cols], "mode": repr(mode),
            "evaluation": ev, "compressed_bytes": comp, "bpv": round(8 * comp / (rows * cols), 3),
            "ms": round(ms, 4), "compressed_gbs": round(comp / ms / 1e6, 1),
            "gflops": round(rows * (2 * cols - 1) / ms / 1e6, 1),
            "decoded_gbs": round(4 * rows * cols / ms / 1e6, 1), "layout": layout,
            "roofline_frac": round((plan.bytes_read + plan.bytes_written) / ms / 1e6 / peak, 4),
            "reference_stream_frac": round(comp / ms / 1e6 / peak, 4)}),
            flush=True)
        plan.close()
    ds.close()
