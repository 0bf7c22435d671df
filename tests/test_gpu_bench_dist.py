"""bench.py's N>1 path (torchrun, row-sharded field, broadcast + all-gather)
run functionally with two ranks sharing one GPU over gloo: it must finish and
print one well-formed JSON line from rank 0 with the whole field's bytes."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--dist-backend", "gloo", "--slits", "2", "--steps", "3", "--warmup", "3",
           "--latency-steps", "5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "row-shard2"
    # whole field: 3 axes x 2 slits x 378 x 256,000 at FixedRate(8) = 1 byte per value
    assert abs(d["value"] * d["ms_per_step"] * 1e6 - 3 * 2 * 380 * 256000) < 0.01 * 3 * 2 * 378 * 256000
    assert d["latency_ms"]["samples"] == 5
