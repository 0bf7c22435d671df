"""Paper-scale device scan: run_scan over fields of 52 slits
x 378 x 256,000 per axis (compressed on the GPU), fast schedule (34 light + 36
dark ms, 50 ms budget), paced at 1 ms per step on the device clock and
unpaced; slits resident in HBM, and streamed from pinned host memory through
a 4-slot ring (the reference's stage 1).  One JSON line.
Usage: python tools/scan_bench.py [n_fields] [mode] [evaluation] [ring slots]"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_08018_b200 import codec, model, pipeline, thermal  # noqa: E402

n_fields = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode_s = sys.argv[2] if len(sys.argv) > 2 else "rate:8"
ev = sys.argv[3] if len(sys.argv) > 3 else "coefficient"
depth = int(sys.argv[4]) if len(sys.argv) > 4 else 4      # streaming ring slots
kind, p = mode_s.split(":")
mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
        "accuracy": codec.FixedAccuracy}[kind](int(p) if kind != "accuracy" else float(p))
spec = model.ModelSpec(grid_rows=608, grid_cols=608, S=256000, K=52 * 378 * n_fields, M=378,
                       nnz_target=7, seed=7, n_fields=n_fields)
t0 = time.time()
m = model.generate_model(spec, materialize=False)
hl = thermal.synthetic_heatload(m, seed=0)
sched = model.build_scan_schedule("fast", n_fields)
out = {"workload": f"paper-scale scan: {n_fields} fields x 52 slits x 3 axes x 378x256000, "
                   f"{mode_s}, fast schedule (34 light + 36 dark ms, budget 50 ms)",
       "evaluation": ev, "setup_s": None}
variants = [("paced_1ms", 1e-3, False), ("unpaced", None, False),
            ("streaming_paced_1ms", 1e-3, True), ("streaming_unpaced", None, True)]
for tag, period, streaming in variants:
    cfg = pipeline.PipelineConfig(use_compression=True, codec_mode=mode, evaluation=ev,
                                  step_period_s=period, streaming=streaming,
                                  queue_depth=depth if streaming else 2)
    t1 = time.time()
    res = pipeline.run_scan(m, sched, hl, cfg)
    wall = time.time() - t1
    light = [s.t_compute * 1e3 for s in res.trace.steps if s.phase == "light"]
    dark = [s.t_compute * 1e3 for s in res.trace.steps if s.phase == "dark"]
    light.sort()
    out[tag] = {
        "field_latency_ms": [round(f.latency_s * 1e3, 3) for f in res.trace.fields],
        "deadline_met": [f.deadline_met for f in res.trace.fields],
        "light_step_ms": {"p50": round(statistics.median(light), 4),
                          "p99": round(light[min(len(light) - 1, int(0.99 * len(light)))], 4),
                          "max": round(light[-1], 4)},
        "dark_step_ms_p50": round(statistics.median(dark), 4),
        "bytes_in_per_light_step": res.trace.steps[0].bytes_in,
        "transfer_ms_p50": round(statistics.median(
            [s.t_transfer * 1e3 for s in res.trace.steps if s.phase == "light"]), 4),
        "wall_s_incl_setup": round(wall, 2)}
out["setup_s"] = round(time.time() - t0, 1)
print(json.dumps(out))
