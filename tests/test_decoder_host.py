"""The device decoder and encoder (csrc/whff_decode.cuh, whff_encode.cuh)
compiled for the host and checked against the oracle -- the exact kernel
logic, exercised without a GPU."""

import ctypes

import numpy as np
import pytest

from conftest import golden_codec_cases, mode_tuple


def P(a):
    return ctypes.c_void_p(a.ctypes.data)


def words_of(payload):
    n = (payload.size + 3) // 4 + 16
    w = np.zeros(n * 4, np.uint8)
    w[:payload.size] = payload
    return w.view(np.uint32)


def host_decode_blocks(L, payload, offs, seg, pl, hr):
    nb = offs.size
    out = [np.zeros((nb, 16), np.uint32), np.zeros((nb, 16), np.uint8), np.zeros(nb, np.uint16),
           np.zeros(nb, np.uint8), np.zeros((nb, 16), np.uint32), np.zeros(nb, np.uint64)]
    w = words_of(payload)
    L.hc_decode_blocks(P(w), payload.size * 8, P(offs), P(seg), nb, pl, int(hr), *[P(o) for o in out])
    return out


def test_device_decoder_matches_golden(hostcheck, golden, orc):
    for case in golden_codec_cases(golden("codec_cases")):
        mode = mode_tuple(case)
        payload, index = case["payload"], case["index"]
        seg = orc.segment_lengths(mode, payload.size, index)
        got = host_decode_blocks(hostcheck, payload, index, seg, orc.planes_limit_for(mode),
                                 mode[0] == "accuracy")
        for a, b in zip(got, case["dec"]):
            assert np.array_equal(a, b), case["name"]
        if case["ok"]:
            arr = case["array"]
            d = np.zeros(arr.shape, np.float32)
            w = words_of(payload)
            hostcheck.hc_decompress(P(w), payload.size * 8, P(index), P(seg), arr.shape[0],
                                    arr.shape[1], orc.planes_limit_for(mode),
                                    int(mode[0] == "accuracy"), P(d))
            assert np.array_equal(d.view(np.uint32), case["words"])


def test_device_decoder_fuzz_arbitrary_bits(hostcheck, orc):
    rng = np.random.default_rng(7)
    for trial in range(1500):
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
        bits = (rng.random(nbytes * 8) < rng.choice([0.5, 0.2, 0.8, 0.05])).astype(np.uint8)
        payload = np.packbits(bits)
        ref = orc.decode_blocks(payload, offs, seg, 27, pl, hr)
        got = host_decode_blocks(hostcheck, payload, offs, seg, pl, hr)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)


def test_device_encoder_matches_golden(hostcheck, golden):
    for case in golden_codec_cases(golden("codec_cases")):
        kind, p = mode_tuple(case)
        code = {"rate": 0, "precision": 1, "accuracy": 2}[kind]
        a = np.ascontiguousarray(case["array"], np.float32)
        offs = np.zeros(case["index"].size, np.uint64)
        tot = hostcheck.hc_compress(P(a), a.shape[0], a.shape[1], code, float(p), P(offs), None)
        w = np.zeros((tot + 7) // 8 // 4 + 8, np.uint32)
        hostcheck.hc_compress(P(a), a.shape[0], a.shape[1], code, float(p), P(offs), P(w))
        assert tot == case["total_bits"]
        assert np.array_equal(offs, case["index"])
        assert np.array_equal(w.view(np.uint8)[:(tot + 7) // 8], case["payload"])


def test_device_encoder_random_vs_oracle(hostcheck, orc):
    rng = np.random.default_rng(3)
    for trial in range(60):
        r, c = (int(x) for x in rng.integers(1, 24, 2))
        a = (rng.standard_normal((r, c)) * 10.0 ** rng.integers(-40, 30, (r, c))).astype(np.float32)
        for kind, p in (("rate", int(rng.integers(1, 33))), ("precision", int(rng.integers(1, 33))),
                        ("accuracy", float(rng.choice([0.0, 1e-6, 1e-12, 1e-30])))):
            code = {"rate": 0, "precision": 1, "accuracy": 2}[kind]
            o = orc.compress(a, (kind, p))
            offs = np.zeros(o.block_index.size, np.uint64)
            tot = hostcheck.hc_compress(P(a), r, c, code, float(p), P(offs), None)
            w = np.zeros((tot + 7) // 8 // 4 + 8, np.uint32)
            hostcheck.hc_compress(P(a), r, c, code, float(p), P(offs), P(w))
            assert tot == o.total_bits
            assert np.array_equal(w.view(np.uint8)[:(tot + 7) // 8], o.payload)


def test_lift_range_fits_int32():
    """Every intermediate of codec.py:_inv_lift (cols then rows) is, up to
    floor rounding, a linear form of the 16 coefficients; with |coef| < 2^27
    the worst case is 15*(2^27-1) < 2^31, so the int32 device lift is exact."""
    peak = [0.0]

    def tr(v):
        peak[0] = max(peak[0], np.abs(v).sum())

    def inv_lift(x, y, z, w):
        y = y + w / 2; tr(y); w = w - y / 2; tr(w)
        y = y + w; tr(y); w = 2 * w; tr(w); w = w - y; tr(w)
        z = z + x; tr(z); x = 2 * x; tr(x); x = x - z; tr(x)
        y = y + z; tr(y); z = 2 * z; tr(z); z = z - y; tr(z)
        w = w + x; tr(w); x = 2 * x; tr(x); x = x - w; tr(x)
        return x, y, z, w

    E = np.eye(16)
    t = [[E[4 * i + j] for j in range(4)] for i in range(4)]
    for j in range(4):
        col = inv_lift(*[t[i][j] for i in range(4)])
        for i in range(4):
            t[i][j] = col[i]
    for i in range(4):
        t[i] = list(inv_lift(*t[i]))
    bound = peak[0] * (2 ** 27 - 1) + 64      # + generous floor-rounding slack
    assert peak[0] == 15.0
    assert bound < 2 ** 31 - 1


def test_device_encode_blocks_matches_oracle(hostcheck, orc):
    """K:228-283 from coefficient arrays, including raw blocks truncated to a
    fixed-rate budget (K:266-270)."""
    rng = np.random.default_rng(1234)
    for t in range(200):
        nb = int(rng.integers(1, 50))
        hr = bool(rng.integers(0, 2))
        budget = int(rng.choice([0, 16 * int(rng.integers(1, 33))]))
        mag = (rng.integers(0, 2 ** 27, (nb, 16)) >> rng.integers(0, 27, (nb, 16))).astype(np.uint32)
        neg = rng.integers(0, 2, (nb, 16)).astype(np.uint8)
        emax = rng.integers(0, 300, nb).astype(np.uint16)
        emax[rng.random(nb) < .2] = 0
        planes = rng.integers(0, 28, nb).astype(np.uint8)
        raw = (rng.random(nb) < .2).astype(np.uint8)
        rw = rng.integers(0, 2 ** 32, (nb, 16), dtype=np.uint64).astype(np.uint32)
        want = orc.encode_blocks(mag, neg, emax, planes, raw, rw, 27, budget, hr)
        offs = np.zeros(nb, np.uint64)
        args = [P(mag), P(neg), P(emax), P(planes), P(raw), P(rw), nb, budget, int(hr), P(offs)]
        tot = hostcheck.hc_encode_blocks(*args, None)
        w = np.zeros(tot // 32 + 8, np.uint32)
        hostcheck.hc_encode_blocks(*args, P(w))
        assert tot == want[2]
        assert np.array_equal(offs, want[1])
        assert np.array_equal(w.view(np.uint8)[:(tot + 7) // 8], want[0])
