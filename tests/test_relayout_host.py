"""Skeleton-first layout (csrc/whff_relayout.cuh), host-compiled: the forward
permutation + its decoder reproduce the reference decode_blocks outputs
exactly, and the inverse permutation restores the reference bytes."""

import ctypes

import numpy as np

from conftest import golden_codec_cases, mode_tuple


def P(a):
    return ctypes.c_void_p(a.ctypes.data)


def words_of(payload):
    n = (payload.size + 3) // 4 + 16
    w = np.zeros(n * 4, np.uint8)
    w[:payload.size] = payload
    return w.view(np.uint32)


def roundtrip(L, orc, payload, offs, seg, pl, hr):
    nb = offs.size
    pb = payload.size * 8
    win = words_of(payload)
    sf = win.copy()
    L.hc_relayout(P(win), P(sf), P(offs), P(seg), nb, pb, pl, int(hr), 0)
    ref = orc.decode_blocks(payload, offs, seg, 27, pl, hr)
    out = [np.zeros((nb, 16), np.uint32), np.zeros((nb, 16), np.uint8), np.zeros(nb, np.uint16),
           np.zeros(nb, np.uint8), np.zeros((nb, 16), np.uint32), np.zeros(nb, np.uint64)]
    L.hc_decode_blocks_sf(P(sf), pb, P(offs), P(seg), nb, pl, int(hr), *[P(o) for o in out])
    for a, b in zip(ref, out):
        assert np.array_equal(a, b)
    back = sf.copy()
    L.hc_relayout(P(sf), P(back), P(offs), P(seg), nb, pb, pl, int(hr), 1)
    assert np.array_equal(back.view(np.uint8)[:payload.size], payload)
    return sf.view(np.uint8)[:payload.size]


def test_skeleton_first_golden(hostcheck, golden, orc):
    changed = 0
    for case in golden_codec_cases(golden("codec_cases")):
        mode = mode_tuple(case)
        seg = orc.segment_lengths(mode, case["payload"].size, case["index"])
        sf = roundtrip(hostcheck, orc, case["payload"], case["index"], seg,
                       orc.planes_limit_for(mode), mode[0] == "accuracy")
        assert sf.size == case["payload"].size
        changed += int(not np.array_equal(sf, case["payload"]))
    assert changed > 50      # it is a real permutation, not the identity


def test_skeleton_first_fuzz_arbitrary_bits(hostcheck, orc):
    rng = np.random.default_rng(7)
    for trial in range(1200):
        nb = int(rng.integers(1, 40))
        if rng.integers(0, 3) == 0:
            bpv = int(rng.integers(1, 33))
            seg = np.full(nb, 16 * bpv, np.uint64)
            offs = np.arange(nb, dtype=np.uint64) * 16 * bpv
            nbytes = max(1, int(nb * 2 * bpv + rng.integers(-3, 4)))
            pl, hr = 27, False
        else:
            lens = rng.integers(0, 700, nb).astype(np.uint64)
            offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
            nbytes = max(1, int((lens.sum() + 7) // 8 + rng.integers(0, 3)))
            ends = np.empty(nb, np.uint64)
            ends[:-1] = offs[1:]
            ends[-1] = nbytes * 8
            seg = ends - offs
            pl, hr = int(rng.integers(1, 28)), bool(rng.integers(0, 2))
        payload = np.packbits((rng.random(nbytes * 8) < rng.choice([.5, .2, .8, .05])).astype(np.uint8))
        roundtrip(hostcheck, orc, payload, offs, seg, pl, hr)


def test_skeleton_first_real_slit(hostcheck, orc):
    """A paper-shaped smooth slit at every mode: identical decode."""
    from paper_1902_08018_b200 import synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=4096, K=378 * 4, M=378, seed=7)
    C = synth.deformation_rows(spec, 1, 0.7, 378, 756)
    for mode in (("rate", 8), ("rate", 4), ("precision", 17), ("accuracy", 1e-12)):
        s = orc.compress(C, mode)
        seg = orc.segment_lengths(mode, s.payload.size, s.block_index)
        roundtrip(hostcheck, orc, s.payload, s.block_index, seg, orc.planes_limit_for(mode),
                  mode[0] == "accuracy")
