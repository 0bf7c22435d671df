"""Small runs of every packed-layout kernel for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the staged coefficient
kernel (mixed, single; single calls, row ranges, a plan), the exact
evaluation, decode-only, the packer -- on smooth and random streams -- and
the bulk-copy staged sequential GEMV (1, 2, 9 and 32 rows per warp, a
strided matrix with a column tail).
Usage: compute-sanitizer --tool <tool> python tools/san_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import _lib, codec, synth  # noqa: E402
from paper_1902_08018_b200.executor import GemvPlan  # noqa: E402


def smooth(rows, cols, seed):
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=cols, K=max(rows, 19656), M=rows, seed=seed)
    return synth.deformation_rows(spec, 0, 0.4 + seed, 5000, 5000 + rows)


rng = np.random.default_rng(3)
streams = []
for rows, cols, mode in ((61, 3000, codec.FixedRate(8)), (37, 9001, codec.FixedAccuracy(1e-12)),
                         (16, 70000, codec.FixedPrecision(17))):
    streams.append(codec.compress_device(smooth(rows, cols, len(streams)), mode).pack())
# adversarial values: raw escapes / exceptions / generic segments
wild = (rng.standard_normal((21, 700)) * np.exp(rng.uniform(-60, 60, (21, 700)))).astype(np.float32)
streams.append(codec.compress_device(wild, codec.FixedAccuracy(0.0)).pack())
for ds in streams:
    v = torch.from_numpy(rng.random(ds.cols).astype(np.float32)).cuda()
    for pol in ("mixed", "single"):
        for ev in ("coefficient", "exact"):
            ds.gemv(v, policy=pol, evaluation=ev)
            ds.gemv(v, policy=pol, evaluation=ev, row_begin=ds.rows // 3, row_end=ds.rows)
    ds.decode()
v = torch.from_numpy(rng.random(streams[0].cols).astype(np.float32)).cuda()
out = torch.zeros(2 * streams[0].rows, device="cuda")
plan = GemvPlan([(streams[0], v, out[:streams[0].rows], 0, streams[0].rows),
                 (streams[0].clone(), v, out[streams[0].rows:], 0, streams[0].rows)], "mixed", "coefficient")
st = _lib.status_word()
plan.launch(st)
torch.cuda.synchronize()
from paper_1902_08018_b200.mpgemv import gemv_device  # noqa: E402
for rows, cols, pad in ((70, 1000, 0), (600, 515, 1), (5000, 260, 0), (19000, 68, 0)):
    base = torch.from_numpy(rng.standard_normal((rows, cols + pad)).astype(np.float32)).cuda()
    vv = torch.from_numpy(rng.standard_normal(cols).astype(np.float32)).cuda()
    for pol in ("mixed", "single", "double"):
        gemv_device(base[:, :cols], vv, pol, "sequential")
torch.cuda.synchronize()
print("san_probe ok")
