"""GPU codec parity: decode_blocks / decompress / decode_block / compress /
encode_blocks against the reference's golden vectors and the oracle --
bit-exact (uint32 / byte equality)."""

import dataclasses
import ctypes

import numpy as np
import pytest

from conftest import golden_codec_cases, mode_tuple

pytestmark = pytest.mark.gpu


def as_mode(case):
    from paper_1902_08018_b200 import codec
    kind, p = mode_tuple(case)
    return {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[kind](p)


def host_stream(case):
    from paper_1902_08018_b200 import codec
    arr = case["array"]
    return codec.CompressedStream(mode=as_mode(case), rows=arr.shape[0], cols=arr.shape[1],
                                  payload=case["payload"], block_index=case["index"],
                                  total_bits=case["total_bits"])


def test_decode_blocks_plugin_matches_reference(golden, orc):
    from paper_1902_08018_b200 import backend
    for case in golden_codec_cases(golden("codec_cases")):
        mode = mode_tuple(case)
        seg = orc.segment_lengths(mode, case["payload"].size, case["index"])
        got = backend.decode_blocks(case["payload"], case["index"], seg, 27,
                                    orc.planes_limit_for(mode), mode[0] == "accuracy")
        for a, b in zip(got, case["dec"]):
            assert np.array_equal(a, b), case["name"]


def test_stream_decode_blocks_all_index_kinds(golden):
    from paper_1902_08018_b200 import codec
    for case in golden_codec_cases(golden("codec_cases")):
        ds = codec.DeviceStream.from_host(host_stream(case))
        got = [t.cpu().numpy() for t in ds.decode_blocks()]
        assert np.array_equal(got[0].view(np.uint32), case["dec"][0])
        assert np.array_equal(got[1], case["dec"][1])
        assert np.array_equal(got[2].view(np.uint16), case["dec"][2])
        assert np.array_equal(got[3], case["dec"][3])
        assert np.array_equal(got[4].view(np.uint32), case["dec"][4])
        assert np.array_equal(got[5].view(np.uint64), case["dec"][5])


def test_decompress_bit_exact(golden):
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    n = 0
    for case in golden_codec_cases(golden("codec_cases")):
        s = host_stream(case)
        if case["ok"]:
            out = codec.decompress(s)
            assert out.dtype == np.float32 and out.shape == case["array"].shape
            assert np.array_equal(out.view(np.uint32), case["words"]), case["name"]
            n += 1
        else:
            with pytest.raises(CorruptStreamError):
                codec.decompress(s)
    assert n > 80


def test_compress_byte_identical(golden):
    from paper_1902_08018_b200 import codec
    for case in golden_codec_cases(golden("codec_cases")):
        s = codec.compress(case["array"], as_mode(case))
        assert np.array_equal(s.payload, case["payload"]), (case["name"], case["kind"])
        assert np.array_equal(s.block_index, case["index"])
        assert s.total_bits == case["total_bits"]


def test_compress_random_vs_oracle(orc, rng):
    from paper_1902_08018_b200 import codec
    for trial in range(25):
        r, c = (int(x) for x in rng.integers(1, 40, 2))
        a = (rng.standard_normal((r, c)) * 10.0 ** rng.integers(-30, 20, (r, c))).astype(np.float32)
        for mode in (codec.FixedRate(int(rng.integers(1, 33))),
                     codec.FixedPrecision(int(rng.integers(1, 33))),
                     codec.FixedAccuracy(float(rng.choice([0.0, 1e-6, 1e-12])))):
            o = orc.compress(a, mode)
            s = codec.compress(a, mode)
            assert np.array_equal(s.payload, o.payload)
            assert np.array_equal(s.block_index, o.block_index)
            assert s.total_bits == o.total_bits
            assert np.array_equal(codec.decompress(s).view(np.uint32),
                                  orc.decompress(o).view(np.uint32))


def test_encode_blocks_plugin_matches_oracle(orc, rng):
    from paper_1902_08018_b200 import backend
    for t in range(60):
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
        a = backend.encode_blocks(mag, neg, emax, planes, raw, rw, 27, budget, hr)
        b = orc.encode_blocks(mag, neg, emax, planes, raw, rw, 27, budget, hr)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_decode_block_independence(golden):
    """test_codec.py:165-177: one block through the index == full decode window."""
    from paper_1902_08018_b200 import codec
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"]:
            continue
        s = host_stream(case)
        full = codec.decompress(s)
        pr, pc = s.padded_shape
        gc = pc // 4
        for index in sorted({0, min(3, s.n_blocks - 1), s.n_blocks - 1}):
            blk = codec.decode_block(s, index)
            br, bc = divmod(index, gc)
            win = full[br * 4:(br + 1) * 4, bc * 4:(bc + 1) * 4]
            assert np.array_equal(blk[:win.shape[0], :win.shape[1]].view(np.uint32), win.view(np.uint32))
        with pytest.raises(codec.CorruptStreamError):
            codec.decode_block(s, s.n_blocks)


def test_prefix_property():
    """test_codec.py:107-118: a deep stream re-read with a shallow plane limit
    equals the shallow encoding."""
    from paper_1902_08018_b200 import codec
    x = np.linspace(0, 1, 16)
    arr = (1e-8 * (np.exp(-((x[None, :] - .4) ** 2 + (x[:, None] - .6) ** 2) * 6)
                   + 0.2 * np.cos(4 * np.pi * x)[None, :])).astype(np.float32)
    deep = codec.compress(arr, codec.FixedPrecision(20))
    shallow = codec.compress(arr, codec.FixedPrecision(8))
    reread = dataclasses.replace(deep, mode=codec.FixedPrecision(8))
    assert np.array_equal(codec.decompress(reread), codec.decompress(shallow))


def test_stream_file_round_trip_and_corruption(tmp_path, rng):
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    arr = (1e-8 * rng.standard_normal((30, 50))).astype(np.float32)
    for mode in (codec.FixedRate(6), codec.FixedPrecision(17), codec.FixedAccuracy(1e-11)):
        s = codec.compress(arr, mode)
        path = tmp_path / "s.whfz"
        codec.save_stream(path, s)
        back = codec.load_stream(path)
        assert back.mode == s.mode
        assert np.array_equal(back.payload, s.payload)
        assert np.array_equal(codec.decompress(back), codec.decompress(s))
    raw = bytearray(path.read_bytes())
    raw[0:4] = b"JUNK"
    path.write_bytes(bytes(raw))
    with pytest.raises(CorruptStreamError):
        codec.load_stream(path)


def test_fuzz_arbitrary_bits_match_oracle(orc, rng):
    from paper_1902_08018_b200 import backend
    for trial in range(150):
        nb = int(rng.integers(1, 64))
        lens = rng.integers(0, 700, nb).astype(np.uint64)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        nbytes = max(1, int((lens.sum() + 7) // 8))
        payload = np.packbits((rng.random(nbytes * 8) < rng.choice([.5, .15, .85])).astype(np.uint8))
        pl, hr = int(rng.integers(1, 28)), bool(rng.integers(0, 2))
        a = backend.decode_blocks(payload, offs, lens, 27, pl, hr)
        b = orc.decode_blocks(payload, offs, lens, 27, pl, hr)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_accuracy_bound_property(rng):
    """test_codec.py:236-249 on the GPU codec."""
    from paper_1902_08018_b200 import codec
    for trial in range(20):
        r, c = (int(x) for x in rng.integers(1, 21, 2))
        tol = float(rng.choice([1e-6, 1e-9, 1e-12, 0.0]))
        arr = (rng.standard_normal((r, c)) * 10.0 ** rng.integers(-12, 6)).astype(np.float32)
        dec = codec.decompress(codec.compress(arr, codec.FixedAccuracy(tol)))
        assert np.abs(dec.astype(np.float64) - arr.astype(np.float64)).max() <= tol


@pytest.mark.parametrize("kind", ["rate", "precision", "accuracy"])
def test_fuzz_skeleton_first_on_device(orc, rng, kind):
    """Arbitrary bits through the device relayout + skeleton-first decoder
    (event walk, closed-form endings, general walker) vs the oracle's
    decode_blocks: identical arrays, and the inverse layout restores the
    bytes.  One block-row of nb blocks per trial."""
    import torch
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    for trial in range(60):
        nb = int(rng.integers(1, 80))
        if kind == "rate":
            bpv = 8 if trial % 2 == 0 else int(rng.integers(1, 33))   # 8: the 128-bit kernel
            mode = codec.FixedRate(bpv)
            lens = np.full(nb, 16 * bpv, np.uint64)
        else:
            mode = codec.FixedPrecision(int(rng.integers(1, 28))) if kind == "precision" \
                else codec.FixedAccuracy(float(rng.choice([0.0, 1e-12])))
            lens = rng.integers(1, 600, nb).astype(np.uint64)
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        total = int(lens.sum())
        nbytes = max(1, (total + 7) // 8) + int(kind != "rate")
        bits = (rng.random(nbytes * 8) < rng.choice([.5, .12, .88])).astype(np.uint8)
        payload = np.packbits(bits)
        s = codec.CompressedStream(mode=mode, rows=4, cols=4 * nb, payload=payload,
                                   block_index=offs, total_bits=total if kind == "rate" else nbytes * 8)
        mk = (kind, mode.bpv if kind == "rate" else mode.planes if kind == "precision" else mode.tolerance)
        seg = orc.segment_lengths(mk, payload.size, offs)
        ref = orc.decode_blocks(payload, offs, seg, 27, orc.planes_limit_for(mk), kind == "accuracy")
        ds = codec.DeviceStream.from_host(s).relayout("skeleton-first")
        got = ds.decode_blocks()
        for a, b in zip(got, ref):
            a = a.cpu().numpy() if hasattr(a, "cpu") else a
            assert np.array_equal(a.reshape(b.shape).astype(b.dtype), b), (trial, kind)
        assert np.array_equal(ds.to_host().payload, payload)
        # the fused kernels' variants (in-register window, sink-only magnitudes)
        # on the same bits: identical to the reference-layout products
        rl = codec.DeviceStream.from_host(s)
        v = torch.rand(4 * nb, device="cuda")
        for ev in ("exact", "coefficient"):
            outs = []
            for d in (rl, ds):
                try:
                    outs.append(d.gemv(v, evaluation=ev).cpu().numpy().view(np.uint32))
                except CorruptStreamError:
                    outs.append("corrupt")
            if isinstance(outs[0], str) or isinstance(outs[1], str):
                assert isinstance(outs[0], str) and isinstance(outs[1], str), (trial, ev)
            else:
                assert np.array_equal(outs[0], outs[1]), (trial, ev)
        rl.close()
        ds.close()
