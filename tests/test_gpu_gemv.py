"""Dense GEMV policies on the GPU vs the reference (goldens, bit-exact for
sequential and fixed-tree; blocked within the reference's own bound)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = (("sequential", 2), ("fixed-tree", 2), ("fixed-tree", 4), ("fixed-tree", 16))


def test_gemv_bit_exact_vs_reference_goldens(golden):
    from paper_1902_08018_b200.mpgemv import GemvRequest, gemv
    g = golden("gemv_cases")
    for i in range(int(g["n"][0])):
        k = f"g{i:02d}"
        m, v = g[k + "_m"], g[k + "_v"]
        for pol in ("mixed", "single", "double"):
            for shape, fo in SHAPES:
                got = gemv(GemvRequest(m, v, pol, shape, fo))
                assert got.dtype == np.float32
                assert np.array_equal(got.view(np.uint32), g[f"{k}_{pol}_{shape}_{fo}"].view(np.uint32)), \
                    (k, pol, shape, fo)


def test_gemv_oracle_matches_reference(golden):
    from paper_1902_08018_b200.mpgemv import gemv_oracle
    g = golden("gemv_cases")
    for i in range(int(g["n"][0])):
        k = f"g{i:02d}"
        assert np.array_equal(gemv_oracle(g[k + "_m"], g[k + "_v"]), g[k + "_oracle"])


def test_blocked_within_reference_bound(rng):
    """tests/test_mpgemv.py:116-130 bound for the B200 blocked order."""
    from paper_1902_08018_b200.mpgemv import GemvRequest, gemv, gemv_oracle
    for dims in ((1, 1), (7, 130), (64, 1031), (378, 16384), (3, 262147)):
        m = rng.standard_normal(dims).astype(np.float32)
        v = rng.standard_normal(dims[1]).astype(np.float32)
        ref = gemv_oracle(m, v)
        scale = np.abs(m).astype(np.float64) @ np.abs(v).astype(np.float64)
        bound = (dims[1] + 1) * np.finfo(np.float32).eps * np.maximum(scale, np.abs(ref))
        for pol in ("mixed", "single", "double"):
            got = gemv(GemvRequest(m, v, pol, "blocked"))
            assert (np.abs(got.astype(np.float64) - ref) <= bound + 1e-300).all(), (dims, pol)


def test_mixed_beats_single_on_wide_rows(rng):
    from paper_1902_08018_b200.mpgemv import GemvRequest, gemv, gemv_oracle, relative_error
    m = rng.standard_normal((32, 8192)).astype(np.float32)
    v = rng.standard_normal(8192).astype(np.float32)
    ref = gemv_oracle(m, v)
    em = relative_error(gemv(GemvRequest(m, v, "mixed", "sequential")), ref)
    es = relative_error(gemv(GemvRequest(m, v, "single", "sequential")), ref)
    assert np.median(em) < np.median(es)


def test_gemv_input_validation(rng):
    from paper_1902_08018_b200.errors import DimensionError, NonFiniteError, WhffError
    from paper_1902_08018_b200.mpgemv import GemvRequest, gemv
    m = rng.standard_normal((2, 3)).astype(np.float32)
    with pytest.raises(DimensionError):
        gemv(GemvRequest(m, np.zeros(4, np.float32)))
    bad = m.copy()
    bad[1, 2] = np.inf
    with pytest.raises(NonFiniteError) as exc:
        gemv(GemvRequest(bad, np.zeros(3, np.float32)))
    assert exc.value.name == "matrix" and exc.value.index == 5
    with pytest.raises(WhffError):
        GemvRequest(m, m[0], "half")
    with pytest.raises(WhffError):
        GemvRequest(m, m[0], "mixed", "fixed-tree", fanout=3)


def test_plugin_gemv_kernel_matches_compiled_reference(golden):
    from paper_1902_08018_b200 import backend
    g = golden("gemv_cases")
    k = "g02"
    got = backend.gemv_kernel(g[k + "_m"], g[k + "_v"], "mixed", "fixed-tree", 16)
    assert np.array_equal(got, g[f"{k}_mixed_fixed-tree_16"])


def test_find_nonfinite_first_index_any_alignment():
    """whff_find_nonfinite returns the smallest flat index of a NaN/inf, for
    aligned (float4 path) and unaligned views (scalar path) alike."""
    import random
    import torch
    from paper_1902_08018_b200.codec import find_nonfinite
    random.seed(0)
    for _ in range(120):
        n = random.randint(1, 5000)
        off = random.randint(0, 3)
        y = torch.rand(n + off, device="cuda")[off:]
        idx = sorted(random.sample(range(n), min(n, random.randint(0, 3))))
        for i in idx:
            y[i] = random.choice([float("nan"), float("inf"), float("-inf")])
        assert find_nonfinite(y) == (idx[0] if idx else None)


def test_gemv_oracle_keeps_binary64_inputs(rng):
    """mpgemv.py:64-69 casts to float64: binary64 inputs (even beyond the
    binary32 range) give the reference's np.cumsum result bit for bit."""
    from paper_1902_08018_b200.mpgemv import gemv_oracle
    m = rng.standard_normal((9, 1031)) * 1e200
    v = rng.standard_normal(1031) * 1e-100
    want = np.cumsum(m * v, axis=1, dtype=np.float64)[:, -1]
    got = gemv_oracle(m, v)
    assert got.dtype == np.float64 and np.array_equal(got, want)


@pytest.mark.parametrize("rows,cols,pad", [
    (70, 1000, 0),       # staged: seven full 128-column stages + a 104-column one
    (33, 128, 0),        # one stage, a row block with a single row
    (5, 3, 0),           # no staged columns: global-memory tail only
    (37, 1003, 0),       # lda % 4 != 0: the per-thread kernel
    (40, 1003, 1),       # strided rows (lda 1004): staged + 3-column tail
    (600, 515, 1),       # 2 rows per warp, strided
    (5000, 260, 0),      # 9 rows per warp, a partial last warp
    (19000, 100, 0),     # 32 rows per warp
    (378, 256000, 0),    # one paper slit
])
def test_sequential_kernels_bit_exact_vs_oracle(orc, rows, cols, pad):
    """K:24-47 strict left-to-right order, on every sequential kernel path
    (the bulk-copy staged kernel at 1..32 rows per warp, and the per-thread
    fallback for unaligned rows)."""
    import torch
    from paper_1902_08018_b200.mpgemv import gemv_device
    g = np.random.default_rng(rows * 7919 + cols)
    base = (g.standard_normal((rows, cols + pad)) * np.exp(g.uniform(-20, 20, (rows, 1)))).astype(np.float32)
    m = np.ascontiguousarray(base[:, :cols])
    v = g.standard_normal(cols).astype(np.float32)
    mt = torch.from_numpy(base).cuda()[:, :cols]
    vt = torch.from_numpy(v).cuda()
    for pol in ("mixed", "single", "double"):
        if cols > 100000 and pol != "mixed":
            continue
        got = gemv_device(mt, vt, pol, "sequential").cpu().numpy()
        want = orc.gemv_kernel(m, v, pol, "sequential")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (rows, cols, pad, pol)
