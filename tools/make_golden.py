"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Runs the unmodified reference (oracle/_ref, built by oracle/build_ref.sh from
/root/reference/pkg) -- never this repository's code -- and stores small
input/output vectors the CPU oracle and the GPU kernels are checked against.
Usage: python tools/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
import whff  # noqa: E402
from whff import codec, mpgemv, model, pipeline, thermal  # noqa: E402

assert whff.BACKEND_NAME == "compiled"
OUT = os.path.join(ROOT, "tests", "golden")
os.makedirs(OUT, exist_ok=True)

MODES = [("rate", 1), ("rate", 3), ("rate", 8), ("rate", 16), ("rate", 32),
         ("precision", 5), ("precision", 17), ("precision", 27),
         ("accuracy", 1e-6), ("accuracy", 1e-12), ("accuracy", 0.0)]


def mk_mode(kind, p):
    return {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[kind](p)


def arrays(rng):
    yield "smooth", (1e-8 * (np.exp(-((np.linspace(0, 1, 23)[None, :] - .4) ** 2
                                      + (np.linspace(0, 1, 18)[:, None] - .6) ** 2) * 6)
                             + 1e-3 * rng.standard_normal((18, 23)))).astype(np.float32)
    yield "noise", (1e-8 * rng.standard_normal((13, 29))).astype(np.float32)
    yield "ints", rng.integers(-1000, 1000, (12, 12)).astype(np.float32)
    yield "big", (rng.standard_normal((5, 3)) * 1e20).astype(np.float32)
    a = rng.standard_normal((20, 20)).astype(np.float32)
    a[::3] *= 1e30
    a[1::3] *= 1e-30
    yield "dynrange", a
    yield "zeros", np.zeros((4, 4), np.float32)
    yield "tiny", (rng.standard_normal((1, 1)) * 1e-8).astype(np.float32)
    yield "subnormal", (np.float32(1e-45) * rng.integers(-5, 6, (7, 9))).astype(np.float32)
    spec = model.ModelSpec(grid_rows=16, grid_cols=16, S=256, K=64, M=16, seed=5)
    yield "model", model.generate_model(spec).C["x"][:24]


def codec_cases():
    rng = np.random.default_rng(20240601)
    out = {}
    n = 0
    for name, arr in arrays(rng):
        for kind, p in MODES:
            mode = mk_mode(kind, p)
            s = codec.compress(arr, mode)
            seg = codec._segment_lengths(s)
            pl = min(p, 27) if kind == "precision" else 27
            dec = codec.get_kernels().decode_blocks(s.payload, s.block_index, seg, 27, pl,
                                                    kind == "accuracy")
            try:
                words = codec.decompress(s)
                ok = True
            except whff.errors.CorruptStreamError:
                words, ok = np.zeros(arr.shape, np.float32), False
            key = f"c{n:03d}"
            out[key + "_meta"] = np.array([name, kind, repr(p)])
            out[key + "_param"] = np.array([p], np.float64)
            out[key + "_array"] = arr
            out[key + "_payload"] = s.payload
            out[key + "_index"] = s.block_index
            out[key + "_total_bits"] = np.array([s.total_bits], np.int64)
            for nm, a in zip(("mag", "neg", "emax", "raw", "raw_words", "consumed"), dec):
                out[key + "_" + nm] = a
            out[key + "_words"] = words.view(np.uint32)
            out[key + "_ok"] = np.array([ok])
            n += 1
    out["n"] = np.array([n])
    np.savez_compressed(os.path.join(OUT, "codec_cases.npz"), **out)
    print("codec cases", n)


def gemv_cases():
    rng = np.random.default_rng(1234)
    out = {}
    n = 0
    for dims in ((1, 1), (7, 130), (64, 1031), (3, 5), (5, 37)):
        m = rng.standard_normal(dims).astype(np.float32)
        v = rng.standard_normal(dims[1]).astype(np.float32)
        key = f"g{n:02d}"
        out[key + "_m"], out[key + "_v"] = m, v
        for pol in ("mixed", "single", "double"):
            for shape, fo in (("sequential", 2), ("fixed-tree", 2), ("fixed-tree", 4),
                              ("fixed-tree", 16)):
                r = mpgemv.gemv(mpgemv.GemvRequest(m, v, pol, shape, fo))
                out[f"{key}_{pol}_{shape}_{fo}"] = r
        out[key + "_oracle"] = mpgemv.gemv_oracle(m, v)
        n += 1
    out["n"] = np.array([n])
    np.savez_compressed(os.path.join(OUT, "gemv_cases.npz"), **out)
    print("gemv cases", n)


def thermal_cases():
    spec = model.ModelSpec(grid_rows=16, grid_cols=16, S=128, K=48, M=6, seed=11, n_fields=2)
    m = model.generate_model(spec)
    rng = np.random.default_rng(99)
    out = {}
    A, P = m.A_f64(), m.P_f64()
    out["A_indptr"], out["A_indices"], out["A_data"] = A.indptr, A.indices, A.data
    out["P_indptr"], out["P_indices"], out["P_data"] = P.indptr, P.indices, P.data
    out["B"] = m.B
    for t in range(4):
        tk = rng.standard_normal(m.T).astype(np.float32)
        uk = rng.standard_normal(m.T).astype(np.float32)
        out[f"t{t}_T"], out[f"t{t}_u"] = tk, uk
        out[f"t{t}_next"] = thermal.thermal_step(A, m.B, tk, uk)
        out[f"t{t}_S"] = thermal.thermal_interpolate(P, out[f"t{t}_next"])
    np.savez_compressed(os.path.join(OUT, "thermal_cases.npz"), **out)
    print("thermal cases", 4)


def pipeline_small():
    """Config 1 (SPEC.md:468 small mesh: gen --grid 32x32 --S 256 --K 512 --M 16
    --seed 7), one field of the fast schedule with the pipeline's default
    FixedAccuracy(1e-12) compression: per light step the thermal vector, the
    slit id and the reference deformations."""
    spec = model.ModelSpec(grid_rows=32, grid_cols=32, S=256, K=512, M=16, seed=7)
    m = model.generate_model(spec)
    sched = model.build_scan_schedule("fast", 1, t_l=6, t_d=2)
    load = thermal.synthetic_heatload(m, seed=0)
    cfg = pipeline.PipelineConfig(use_compression=True)
    res = pipeline.run_scan(m, sched, load, cfg)
    out = {}
    # thermal trajectory for the same light steps
    state = thermal.ThermalState.initial(m)
    svecs, slits = [], []
    for k, phase, slit, s_next in thermal.run_field_thermal(m, sched.fields[0], load, state):
        if phase == "light":
            svecs.append(s_next)
            slits.append(slit)
    out["S"] = np.stack(svecs)
    out["slits"] = np.array(slits)
    for a in model.AXES:
        out["D_" + a] = res.deformations[a]
        c_field = m.fetch_field_submatrix(a, 0)
        for s in sorted(set(slits)):
            c = m.fetch_slit_submatrix(c_field, 0, s)
            st = codec.compress(c, codec.FixedAccuracy(1e-12))
            out[f"C_{a}_{s}"] = np.ascontiguousarray(c)
            out[f"payload_{a}_{s}"] = st.payload
            out[f"index_{a}_{s}"] = st.block_index
    np.savez_compressed(os.path.join(OUT, "pipeline_small.npz"), **out)
    print("pipeline steps", len(slits))


def scan_small():
    """Reference run_scan (pipeline.py:164-181, simulated clock) on the
    config-1 model: two fields of a shortened fast schedule, without
    compression, with the default FixedAccuracy(1e-12) and with FixedRate(8).
    Stores the deformations and the timing-independent trace columns."""
    spec = model.ModelSpec(grid_rows=32, grid_cols=32, S=256, K=512, M=16, seed=7)
    m = model.generate_model(spec)
    sched = model.build_scan_schedule("fast", 2, t_l=6, t_d=3)
    load = thermal.synthetic_heatload(m, seed=0)
    out = {}
    for tag, cfg in (("raw", pipeline.PipelineConfig()),
                     ("acc", pipeline.PipelineConfig(use_compression=True)),
                     ("r8", pipeline.PipelineConfig(use_compression=True,
                                                    codec_mode=codec.FixedRate(8)))):
        res = pipeline.run_scan(m, sched, load, cfg)
        for a in model.AXES:
            out[f"{tag}_D_{a}"] = res.deformations[a]
        tr = res.trace.steps
        out[f"{tag}_field"] = np.array([s.field_id for s in tr])
        out[f"{tag}_k"] = np.array([s.k for s in tr])
        out[f"{tag}_light"] = np.array([s.phase == "light" for s in tr])
        out[f"{tag}_slit"] = np.array([s.slit for s in tr])
        out[f"{tag}_bytes_in"] = np.array([s.bytes_in for s in tr])
        # the simulated clock's times (pipeline.py:208-289)
        out[f"{tag}_times"] = np.array([[s.t_transfer, s.t_decode, s.t_compute, s.stage1_start,
                                         s.stage1_end, s.stage2_start, s.stage2_end] for s in tr])
        out[f"{tag}_fields"] = np.array([[f.start, f.end, f.latency_s, f.budget_s,
                                          float(f.deadline_met)] for f in res.trace.fields])
    np.savez_compressed(os.path.join(OUT, "scan_small.npz"), **out)
    print("scan steps", len(tr))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    codec_cases()
    gemv_cases()
    thermal_cases()
    pipeline_small()
