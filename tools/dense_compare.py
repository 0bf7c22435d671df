"""Compressed vs uncompressed on the B200: the dense binary32 GEMV
(mpgemv "blocked" shape, mixed policy) over paper slits (378 x 256,000, 387 MB
each) against the fused decode+GEMV of the same slits compressed with
FixedRate(8) / FixedAccuracy(1e-12).  CUDA-event medians; inputs far larger
than L2 (distinct slits per launch).  One JSON line per case.
Usage: python tools/dense_compare.py [n_slits]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import _lib, codec, synth  # noqa: E402
from paper_1902_08018_b200.executor import GemvPlan  # noqa: E402
from paper_1902_08018_b200.mpgemv import gemv_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
spec = synth.Spec(grid_rows=608, grid_cols=608, S=256000, K=n * 378, M=378, seed=7)
mats = [synth.deformation_rows(spec, 0, 0.3, i * 378, (i + 1) * 378, device="cuda") for i in range(n)]
v = torch.rand(256000, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
out = torch.empty(n * 378, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def dense():
    for i, m in enumerate(mats):
        gemv_device(m, v, "mixed", "blocked", out=out[i * 378:(i + 1) * 378])


ms = timed(dense)
nbytes = n * 378 * 256000 * 4
print(json.dumps({"case": "dense binary32 GEMV (blocked, mixed)", "slits": n, "ms": round(ms, 3),
                  "matrix_GB": round(nbytes / 1e9, 2), "GBps_read": round(nbytes / ms / 1e6, 1),
                  "ms_per_slit": round(ms / n, 4)}), flush=True)
for mode in (codec.FixedRate(8), codec.FixedAccuracy(1e-12)):
    streams = []
    for m in mats:
        ds = codec.compress_device(m, mode)
        ds.relayout("skeleton-first")
        streams.append(ds)
    for ev in ("coefficient", "exact"):
        plan = GemvPlan([(streams[i], v, out[i * 378:(i + 1) * 378], 0, 378) for i in range(n)],
                        evaluation=ev)
        st = _lib.status_word()
        ms = timed(lambda: plan.launch(st))
        print(json.dumps({"case": f"fused {mode} {ev}", "slits": n, "ms": round(ms, 3),
                          "compressed_GB": round(plan.bytes_read / 1e9, 3),
                          "decoded_equiv_GBps": round(nbytes / ms / 1e6, 1),
                          "ms_per_slit": round(ms / n, 4),
                          "hbm_footprint_vs_dense": round(plan.bytes_read / nbytes, 3)}), flush=True)
        plan.close()
    for ds in streams:
        ds.close()
