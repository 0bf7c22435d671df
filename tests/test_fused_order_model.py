"""CPU checks of the fused-order model (tests/fused_order.py) against the
oracle's reference GEMV: identical where the orders coincide (one block
column: the sequential order), within the reference's bound otherwise."""

import numpy as np
import pytest

from fused_order import fused_exact


@pytest.mark.parametrize("policy", ["mixed", "single", "double"])
def test_single_block_column_is_sequential(orc, policy, rng):
    for cols in (1, 2, 3, 4):
        m = rng.standard_normal((7, cols)).astype(np.float32)
        v = rng.random(cols).astype(np.float32)
        want = orc.gemv_kernel(m, v, policy, "sequential")
        got = fused_exact(m, v, policy)
        assert np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).view(np.uint32))


def test_within_reference_bound(orc, rng):
    m = rng.standard_normal((9, 50000)).astype(np.float32)
    v = rng.random(50000).astype(np.float32)
    got = fused_exact(m, v, "mixed").astype(np.float64)
    ref = np.asarray(orc.gemv_kernel(m, v, "mixed", "sequential"), np.float64)
    bound = (m.shape[1] + 1) * np.finfo(np.float32).eps * (np.abs(m).astype(np.float64) @ v)
    assert (np.abs(got - ref) <= bound).all()


def test_coefficient_model_within_reference_bound_smooth(orc, rng):
    """The coefficient-domain model on a smooth operator (the WHFF case)
    stays inside the reference's per-row bound around the sequential GEMV of
    the decoded words (DESIGN §2 tolerance contract)."""
    from fused_order import fused_coefficient
    from paper_1902_08018_b200 import codec, synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=6001, K=13, M=13, seed=4)
    C = synth.deformation_rows(spec, 2, 0.9, 0, 13)
    for mode in (codec.FixedRate(8), codec.FixedAccuracy(1e-12)):
        host = orc.compress(C, mode)
        host.mode = mode
        words = orc.decompress(host)
        v = rng.random(C.shape[1]).astype(np.float32)
        got = fused_coefficient(orc, host, v).astype(np.float64)
        ref = np.asarray(orc.gemv_kernel(words, v, "mixed", "sequential"), np.float64)
        bound = (C.shape[1] + 1) * np.finfo(np.float32).eps * (np.abs(words).astype(np.float64) @ v)
        assert (np.abs(got - ref) <= bound).all()


def test_model_segment_size_matches_the_layout():
    """packed_host.seg_tiles_for restates csrc/whff_packed.cuh seg_tiles_for_mode."""
    import os
    import re
    from conftest import ROOT
    from packed_host import seg_tiles_for
    hdr = open(os.path.join(ROOT, "paper_1902_08018_b200", "csrc", "whff_packed.cuh")).read()
    assert int(re.search(r"kSegTilesRate = (\d+);", hdr).group(1)) == seg_tiles_for("rate")
    assert int(re.search(r"kSegTilesVar = (\d+);", hdr).group(1)) == seg_tiles_for("accuracy")
    assert seg_tiles_for("precision") == seg_tiles_for("accuracy")
