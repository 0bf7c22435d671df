"""The CPU oracle (oracle/whff_oracle.c) pinned against the reference:
golden vectors produced by the reference itself (tools/make_golden.py) and,
when oracle/_ref is built in this container, the live reference."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_codec_cases, mode_tuple


def test_oracle_codec_matches_reference_goldens(orc, golden):
    g = golden("codec_cases")
    n = 0
    for case in golden_codec_cases(g):
        mode = mode_tuple(case)
        s = orc.compress(case["array"], mode)
        assert np.array_equal(s.payload, case["payload"]), case["name"]
        assert np.array_equal(s.block_index, case["index"])
        assert s.total_bits == case["total_bits"]
        seg = orc.segment_lengths(mode, s.payload.size, s.block_index)
        dec = orc.decode_blocks(s.payload, s.block_index, seg, 27, orc.planes_limit_for(mode),
                                mode[0] == "accuracy")
        for a, b in zip(dec, case["dec"]):
            assert np.array_equal(a, b)
        if case["ok"]:
            w = orc.decompress(s)
            assert np.array_equal(w.view(np.uint32), case["words"])
        n += 1
    assert n >= 90


def test_oracle_gemv_matches_reference_goldens(orc, golden):
    g = golden("gemv_cases")
    for i in range(int(g["n"][0])):
        k = f"g{i:02d}"
        m, v = g[k + "_m"], g[k + "_v"]
        for pol in ("mixed", "single", "double"):
            for shape, fo in (("sequential", 2), ("fixed-tree", 2), ("fixed-tree", 4),
                              ("fixed-tree", 16)):
                got = orc.gemv_kernel(m, v, pol, shape, fo)
                assert np.array_equal(got.view(np.uint32), g[f"{k}_{pol}_{shape}_{fo}"].view(np.uint32))


def test_oracle_thermal_matches_reference_goldens(orc, golden):
    import scipy.sparse as sp
    g = golden("thermal_cases")
    n = g["B"].size
    A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=(n, n))
    P = sp.csr_matrix((g["P_data"], g["P_indices"], g["P_indptr"]), shape=(g["P_indptr"].size - 1, n))
    for t in range(4):
        nxt = orc.thermal_step(A, g["B"], g[f"t{t}_T"], g[f"t{t}_u"])
        assert np.array_equal(nxt.view(np.uint32), g[f"t{t}_next"].view(np.uint32))
        s = orc.thermal_interpolate(P, nxt)
        assert np.array_equal(s.view(np.uint32), g[f"t{t}_S"].view(np.uint32))


def _ref():
    path = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.isdir(os.path.join(path, "whff")):
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    if path not in sys.path:
        sys.path.insert(0, path)
    import whff
    return whff


def test_oracle_against_live_reference_random(orc):
    whff = _ref()
    from whff import codec
    rng = np.random.default_rng(5)
    for trial in range(40):
        r, c = rng.integers(1, 21, 2)
        arr = (rng.standard_normal((r, c)) * 10.0 ** rng.integers(-12, 6)).astype(np.float32)
        for mode in (codec.FixedRate(int(rng.integers(1, 33))),
                     codec.FixedPrecision(int(rng.integers(1, 33))),
                     codec.FixedAccuracy(float(rng.choice([0.0, 1e-6, 1e-9, 1e-12])))):
            s = codec.compress(arr, mode)
            o = orc.compress(arr, mode)
            assert np.array_equal(s.payload, o.payload)
            assert np.array_equal(s.block_index, o.block_index)
            assert np.array_equal(codec.decompress(s).view(np.uint32),
                                  orc.decompress(s).view(np.uint32))


def test_oracle_decoder_on_arbitrary_bits_matches_reference(orc):
    """Corrupt / arbitrary bitstreams: the decoder never errors and both agree."""
    whff = _ref()
    from whff import backend
    kern = backend.get_kernels("compiled")
    rng = np.random.default_rng(11)
    for trial in range(300):
        nb = int(rng.integers(1, 30))
        lens = rng.integers(0, 600, nb).astype(np.uint64)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        nbytes = max(1, int((lens.sum() + 7) // 8))
        payload = np.packbits((rng.random(nbytes * 8) < rng.choice([.5, .15, .85])).astype(np.uint8))
        pl, hr = int(rng.integers(1, 28)), bool(rng.integers(0, 2))
        a = kern.decode_blocks(payload, offs, lens, 27, pl, hr)
        b = orc.decode_blocks(payload, offs, lens, 27, pl, hr)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
