"""Device pipeline mirror (paper_1902_08018_b200/pipeline.py, model.py): the
host-side pieces -- model generation, schedules, heat loads, trace export,
Table-1 algebra, config validation -- against the reference's semantics and
goldens (no GPU)."""

import numpy as np
import pytest

from paper_1902_08018_b200 import model, pipeline, thermal
from paper_1902_08018_b200.errors import WhffError


def config1():
    return model.ModelSpec(grid_rows=32, grid_cols=32, S=256, K=512, M=16, seed=7)


def test_generate_model_matches_reference_slits(golden):
    """model.py:158-186: same rng order -> the reference's C, slit by slit."""
    g = golden("pipeline_small")
    m = model.generate_model(config1())
    assert m.n_fields == 8 and m.n_slits(0) == 4
    for a in model.AXES:
        c_field = m.fetch_field_submatrix(a, 0)
        for s in range(4):
            got = m.fetch_slit_submatrix(c_field, 0, s)
            assert np.array_equal(got, g[f"C_{a}_{s}"])
            assert np.array_equal(m.slit_rows(a, 0, s), got)


def test_lazy_model_has_no_dense_operators():
    spec = model.ModelSpec(grid_rows=64, grid_cols=64, S=4096, K=378 * 8, M=378, seed=1)
    m = model.generate_model(spec, materialize=False)
    assert m.C is None and m.n_fields == 2 and m.n_slits(1) == 4
    with pytest.raises(WhffError):
        m.fetch_field_submatrix("x", 0)
    with pytest.raises(model.ModelTooLargeError):
        model.generate_model(model.ModelSpec(grid_rows=608, grid_cols=608, S=256000,
                                             K=378 * 52, M=378))


def test_schedule_mirror():
    s = model.build_scan_schedule("fast", 3)
    assert s.steps_per_field == 70 and len(s.fields) == 3
    f = s.fields[0]
    assert (f.t_l, f.t_d, f.time_budget_ms) == (34, 36, 50.0)
    assert [f.slit_for_light_step(i, 4) for i in (0, 8, 9, 33)] == [0, 0, 1, 3]
    with pytest.raises(model.ScheduleError):
        f.slit_for_light_step(34, 4)
    with pytest.raises(model.ScheduleError):
        model.build_scan_schedule("medium", 1)
    with pytest.raises(model.ScheduleError):
        model.build_scan_schedule("fast", 1, t_l=0, t_d=0)


def test_synthetic_heatload_shapes_and_validation():
    m = model.generate_model(config1())
    hl = thermal.synthetic_heatload(m, seed=0)
    assert hl.dark_load.shape == (m.T,) and (hl.dark_load < 0).all()
    fp = hl.light_load(1, 2)
    assert fp.shape == (m.T,) and (fp >= 0).all()
    with pytest.raises(WhffError):
        hl.light_load(9, 0)
    with pytest.raises(WhffError):
        thermal.HeatLoad(np.zeros(4), {(0, 0): -np.ones(4)})


def test_config_validation():
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(queue_depth=1)
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(time_source="wallclock")
    pipeline.PipelineConfig(time_source="simulated")
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(evaluation="approximate")
    cfg = pipeline.PipelineConfig(use_compression=True)
    assert cfg.codec_mode.tolerance == 1e-12


def test_table1_algebra():
    assert pipeline.pipeline_period(4.0, 1.0, 0.5, 2.0, True) == 2.0
    assert pipeline.pipeline_period(4.0, 1.0, 0.5, 2.0, False) == 4.0
    assert pipeline.pipeline_latency(4.0, 1.0, 0.5, 2.0, True) == 3.5
    with pytest.raises(WhffError):
        pipeline.pipeline_period(1.0, 1.0, 1.0, 0.5, True)


def test_trace_csv_and_deadline_report(tmp_path):
    steps = [pipeline.StepRecord(0, 1, "light", 2, 100, 0.0, 0.0, 1e-4, 0.0, 0.0, 0.0, 1e-4),
             pipeline.StepRecord(0, 2, "dark", -1, 0, 0.0, 0.0, 1e-4, 1e-3, 1e-3, 1e-3, 1.1e-3),
             pipeline.StepRecord(1, 3, "light", 0, 100, 0.0, 0.0, 1e-4, 2e-3, 2e-3, 2e-3, 9e-2)]
    fields = [pipeline.FieldRecord(0, 0.0, 1.1e-3, 1.1e-3, 0.05, True),
              pipeline.FieldRecord(1, 2e-3, 9e-2, 8.8e-2, 0.05, False)]
    tr = pipeline.PipelineTrace(steps, fields)
    p = tmp_path / "t.csv"
    pipeline.export_trace_csv(tr, p)
    lines = p.read_text().splitlines()
    assert lines[0] == pipeline.TRACE_HEADER
    assert lines[1].startswith("0,1,light,2,100,0.0,0.0,0.0001,") and lines[1].endswith(",true")
    assert lines[3].endswith(",false")
    rep = pipeline.deadline_report(tr)
    assert rep.miss_rate == 0.5 and rep.worst_latency_s == 8.8e-2
    assert pipeline.deadline_report(tr, budgets={0: 1e-4, 1: 1.0}).verdicts[0][1] is False


def test_streaming_config_needs_compression():
    from paper_1902_08018_b200 import codec
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(streaming=True)              # nothing compressed to stage
    pipeline.PipelineConfig(streaming=True, use_compression=True)
    pipeline.PipelineConfig(streaming=True, use_compression=True, codec_mode=codec.FixedRate(8))


def test_layout_defaults():
    """Resident slits default to the tile-packed copy (the k_pk_gemv2 path);
    streaming stages a stream layout (skeleton-first) and rejects packed."""
    assert pipeline.PipelineConfig(use_compression=True).layout == "packed"
    assert pipeline.PipelineConfig(streaming=True, use_compression=True).layout == "skeleton-first"
    assert pipeline.PipelineConfig(layout="reference").layout == "reference"
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(streaming=True, use_compression=True, layout="packed")
    with pytest.raises(WhffError):
        pipeline.PipelineConfig(layout="tiled")
