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
