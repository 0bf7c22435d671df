"""Both fused evaluations, bit for bit, against CPU models of their
arithmetic and summation order (tests/fused_order.py) applied to the
oracle's decoded words / fields: every policy, stream variant and layout,
ragged shapes, raw escapes and extreme scales."""

import numpy as np
import pytest

from fused_order import fused_exact

pytestmark = pytest.mark.gpu


def matrix(kind, rows, cols, rng):
    if kind == "smooth":
        from paper_1902_08018_b200 import synth
        spec = synth.Spec(grid_rows=16, grid_cols=16, S=cols, K=rows, M=rows, seed=2)
        return synth.deformation_rows(spec, 1, 0.4, 0, rows)
    m = rng.standard_normal((rows, cols)).astype(np.float32)
    special = np.array([1e30, -1e-30, 3e-38, 0.0, -0.0, 7.5], np.float32)   # wide range / raw escapes
    n = min(6, cols)
    m[rows // 2, cols - n:] = special[:n]
    return m


@pytest.mark.parametrize("kind,rows,cols", [("smooth", 37, 20011), ("noise", 23, 4099),
                                            ("smooth", 8, 131072), ("noise", 5, 3)])
@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("rate", 13), ("precision", 17),
                                             ("accuracy", 1e-12)])
@pytest.mark.parametrize("layout", ["reference", "skeleton-first"])
def test_exact_matches_order_model(orc, kind, rows, cols, mode_kind, param, layout, rng):
    import torch
    from paper_1902_08018_b200 import codec
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    C = matrix(kind, rows, cols, rng)
    host = codec.compress(C, mode)
    words = orc.decompress(host)                     # oracle: bit-exact decoded words
    ds = codec.DeviceStream.from_host(host)
    if layout != "reference":
        ds.relayout(layout)
    v = rng.random(cols).astype(np.float32)
    vd = torch.from_numpy(v).cuda()
    for policy in ("mixed", "single", "double"):
        got = ds.gemv(vd, policy=policy, evaluation="exact").cpu().numpy()
        want = fused_exact(words, v, policy)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (policy, kind, mode_kind)


@pytest.mark.parametrize("kind,rows,cols", [("smooth", 37, 20011), ("noise", 23, 4099),
                                            ("noise", 5, 3)])
@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("precision", 17), ("accuracy", 1e-12)])
@pytest.mark.parametrize("layout", ["reference", "skeleton-first"])
def test_coefficient_matches_order_model(orc, kind, rows, cols, mode_kind, param, layout, rng):
    """The coefficient-domain evaluation (bench default), bit for bit, against
    tests/fused_order.fused_coefficient on the oracle's decoded fields: u = G^T v
    per block column, binary32 FMAs in coefficient order, 2^k scaling, binary64
    lane sums, the exact spatial fallback for raw / extreme blocks, the two
    butterflies and the final G combination."""
    import torch
    from fused_order import fused_coefficient
    from paper_1902_08018_b200 import codec
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    C = matrix(kind, rows, cols, rng)
    host = codec.compress(C, mode)
    ds = codec.DeviceStream.from_host(host)
    if layout != "reference":
        ds.relayout(layout)
    v = rng.random(cols).astype(np.float32)
    vd = torch.from_numpy(v).cuda()
    for policy in ("mixed", "single"):
        got = ds.gemv(vd, policy=policy, evaluation="coefficient").cpu().numpy()
        want = fused_coefficient(orc, host, v, policy)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (policy, kind, mode_kind)


def test_paper_width_rows_match_order_models(orc, rng):
    """Paper slit width (256,000 columns: 2,000 groups, 63 per virtual warp),
    FixedRate(8), skeleton-first: both evaluations bit-exact vs the models."""
    import torch
    from fused_order import fused_coefficient
    from paper_1902_08018_b200 import codec
    C = matrix("smooth", 40, 256000, rng)
    host = codec.compress(C, codec.FixedRate(8))
    ds = codec.DeviceStream.from_host(host).relayout("skeleton-first")
    v = rng.random(256000).astype(np.float32)
    vd = torch.from_numpy(v).cuda()
    got = ds.gemv(vd, evaluation="coefficient").cpu().numpy()
    assert np.array_equal(got.view(np.uint32), fused_coefficient(orc, host, v).view(np.uint32))
    got = ds.gemv(vd, evaluation="exact").cpu().numpy()
    assert np.array_equal(got.view(np.uint32), fused_exact(orc.decompress(host), v).view(np.uint32))
