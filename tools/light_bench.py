"""Light-step sized plans (1 and 3 paper slits, 378 x 256,000, skeleton-first):
kernel time from CUDA events (median of 50 launches) and the bits of each
slit's rows against a single whff_decode_gemv call.  One JSON line per
(slits, evaluation).  Usage: python tools/light_bench.py [mode]"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import _lib, codec, synth  # noqa: E402
from paper_1902_08018_b200.executor import GemvPlan  # noqa: E402

mode_s = sys.argv[1] if len(sys.argv) > 1 else "rate:8"
kind, p = mode_s.split(":")
mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
        "accuracy": codec.FixedAccuracy}[kind](int(p) if kind != "accuracy" else float(p))
spec = synth.Spec(grid_rows=608, grid_cols=608, S=256000, K=3 * 378, M=378, seed=7)
streams = []
for a in range(3):
    c = synth.deformation_rows(spec, a, 0.3 + a, a * 378, (a + 1) * 378, device="cuda")
    ds = codec.compress_device(c, mode)
    ds.relayout("skeleton-first")
    streams.append(ds)
    del c
v = torch.rand(256000, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
for ev in ("coefficient", "exact"):
    single = [ds.gemv(v, evaluation=ev).cpu().numpy() for ds in streams]
    for n in (1, 3):
        out = torch.zeros(378 * n, device="cuda")
        plan = GemvPlan([(streams[i], v, out[i * 378:(i + 1) * 378], 0, 378) for i in range(n)],
                        evaluation=ev)
        st = _lib.status_word()
        for _ in range(5):
            plan.launch(st)
        ts = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.launch(st)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        y = out.cpu().numpy()
        ms = statistics.median(ts)
        print(json.dumps({"mode": mode_s, "evaluation": ev, "slits": n, "block_rows": 95 * n,
                          "ms": round(ms, 4), "GBps": round(plan.bytes_read / (ms * 1e-3) / 1e9, 1),
                          "identical_to_single_calls": bool(np.array_equal(
                              y.view(np.uint32), np.concatenate(single[:n]).view(np.uint32)))}),
              flush=True)
        plan.close()
