"""bench.py's command line (no GPU): the driver's default invocation and the
configs[4] preset resolve to the workloads BASELINE.json names."""

import importlib.util
import os
import sys

from conftest import ROOT


def _bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _parse(mod, argv, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"] + argv)
    return mod.parse()


def test_default_is_the_paper_step(monkeypatch):
    mod = _bench()
    a = _parse(mod, [], monkeypatch)
    assert (a.gpus, a.S, a.grid, a.slits, a.rows, a.mode) == (1, 256000, 608, 52, 378, "rate:8")
    assert a.warmup >= 3 and a.latency_steps >= 1000
    assert mod.workload_config(a, 1)["workload"].startswith("paper-scale WHFF step (configs[2])")
    assert "configs[3]" in mod.workload_config(a, 8)["workload"]


def test_mesh4x_preset(monkeypatch):
    mod = _bench()
    a = _parse(mod, ["--preset", "mesh4x", "--gpus", "8", "--latency-steps", "10"], monkeypatch)
    assert (a.S, a.grid, a.latency_steps) == (1024000, 1216, 1000)
    assert mod.workload_config(a, 8)["workload"].startswith("4x paper mesh step (configs[4] workload)")
