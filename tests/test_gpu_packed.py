"""The tile-packed device layout (whff_dstream_pack, csrc/whff_packed.cuh) on
the B200: the device packer is byte-identical to the host packer
(tests/packed_host.py), decode from the packed copy is bit-exact with the
oracle's codec.decompress on every reference golden stream and on arbitrary
bit streams, and the fused decode + GEMV over it is bit-exact against a CPU
model of its arithmetic (tests/fused_order.py packed_model) and within the
reference's bound (tests/test_mpgemv.py:116-130, test_acceptance.py:195-197).
"""

import numpy as np
import pytest

from conftest import golden_codec_cases
import packed_host as ph

pytestmark = pytest.mark.gpu
EPS32 = np.finfo(np.float32).eps


def bound(C, v):
    scale = np.abs(C).astype(np.float64) @ np.abs(v).astype(np.float64)
    return (C.shape[1] + 1) * EPS32 * scale


def host_stream(case):
    from test_gpu_codec import host_stream as hs
    return hs(case)


def download_packed(ds):
    """(segs, body, exc_block, exc_words) of a packed device stream."""
    import ctypes
    from paper_1902_08018_b200 import _lib
    info = _lib.DStreamInfo()
    _lib.call("whff_dstream_get_info", ds.handle, ctypes.byref(info))
    nseg, words, nexc = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _lib.call("whff_dstream_packed_download", ds.handle, None, None, None, None,
              ctypes.byref(nseg), ctypes.byref(words), ctypes.byref(nexc))
    segs = np.zeros(nseg.value * 48, np.uint8)
    body = np.zeros(words.value, np.uint32)
    xb = np.zeros(max(nexc.value, 1), np.uint64)
    xw = np.zeros((max(nexc.value, 1), 16), np.uint32)
    _lib.call("whff_dstream_packed_download", ds.handle, _lib.ptr(segs), _lib.ptr(body),
              _lib.ptr(xb), _lib.ptr(xw), ctypes.byref(nseg), ctypes.byref(words), ctypes.byref(nexc))
    return segs, body, xb[:nexc.value], xw[:nexc.value]


def test_device_packer_matches_host_packer_on_goldens(golden, hostcheck):
    from paper_1902_08018_b200 import codec
    n = 0
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"]:
            continue
        s = host_stream(case)
        mag, neg, emax, raw, raw_words, _ = case["dec"]
        hp = ph.pack(hostcheck, mag, neg, emax, raw, raw_words, s.rows, s.cols, s.mode)
        ds = codec.DeviceStream.from_host(s).pack()
        assert ds.packed and ds.packed_exceptions == hp["exc_block"].size
        segs, body, xb, xw = download_packed(ds)
        assert np.array_equal(segs, hp["segs"]), case["name"]
        assert np.array_equal(body, hp["body"][:body.size]), case["name"]
        assert np.array_equal(xb, hp["exc_block"]) and np.array_equal(xw, hp["exc_words"])
        ds.close()
        n += 1
    assert n > 50


@pytest.mark.parametrize("layout", ["reference", "skeleton-first"])
def test_packed_decode_bitexact_every_golden_stream(golden, orc, layout):
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    for case in golden_codec_cases(golden("codec_cases")):
        s = host_stream(case)
        ds = codec.DeviceStream.from_host(s)
        if layout != "reference":
            ds.relayout(layout)
        ds.pack()
        if case["ok"]:
            got = ds.decode().cpu().numpy()
            assert np.array_equal(got.view(np.uint32), case["words"].view(np.uint32)), case["name"]
        else:
            with pytest.raises(CorruptStreamError):
                ds.decode()
        ds.close()


def test_packed_decode_arbitrary_bits(orc):
    """Random payloads (any emax, raw escapes, truncated planes): exceptions,
    generic segments, zero blocks; words equal the oracle's bit for bit."""
    import torch
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    rng = np.random.default_rng(11)
    for trial in range(40):
        rows, cols = int(rng.integers(1, 40)), int(rng.integers(1, 2100))
        nb = ((rows + 3) // 4) * ((cols + 3) // 4)
        kind = ("precision", int(rng.integers(1, 28))) if trial % 2 else ("accuracy", 1e-6)
        seg = int(rng.integers(12, 160))
        payload = rng.integers(0, 256, nb * seg // 8 + 16, dtype=np.uint8)
        index = np.arange(nb, dtype=np.uint64) * np.uint64(seg)
        mode = codec.FixedPrecision(kind[1]) if kind[0] == "precision" else codec.FixedAccuracy(kind[1])
        s = codec.CompressedStream(mode=mode, rows=rows, cols=cols, payload=payload, block_index=index,
                                   total_bits=int(payload.size * 8))
        try:
            ref = orc.decompress(s)
        except ValueError:
            ref = None
        ds = codec.DeviceStream.from_host(s).pack()
        if ref is None:
            with pytest.raises(CorruptStreamError):
                ds.decode()
        else:
            got = ds.decode().cpu().numpy()
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), trial
        ds.close()
    torch.cuda.synchronize()


def _packed_gemv(s, v, policy, evaluation):
    import torch
    from paper_1902_08018_b200 import codec
    ds = codec.DeviceStream.from_host(s).pack()
    y = ds.gemv(torch.from_numpy(v).cuda(), policy=policy, evaluation=evaluation).cpu().numpy()
    ds.close()
    return y


@pytest.mark.parametrize("evaluation", ["exact", "coefficient"])
@pytest.mark.parametrize("policy", ["mixed", "single", "double"])
def test_packed_gemv_bitexact_model_goldens(golden, orc, evaluation, policy, rng):
    """Every golden stream (raw escapes, extreme scales -> the exception
    list; ragged shapes; zero blocks): device == CPU model, bit for bit."""
    from fused_order import packed_model
    if evaluation == "coefficient" and policy == "double":
        pytest.skip("coefficient evaluation: mixed and single policies")
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"]:
            continue
        s = host_stream(case)
        v = rng.standard_normal(s.cols).astype(np.float32)
        got = _packed_gemv(s, v, policy, evaluation)
        want = packed_model(orc, s, v, policy, evaluation)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), case["name"]


def smooth_matrix(rows, cols, seed=0, S=None):
    from paper_1902_08018_b200 import synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=S or cols, K=max(rows, 19656), M=rows, seed=seed)
    phase = np.random.default_rng(seed).random() * 2 * np.pi
    return synth.deformation_rows(spec, 0, phase, 5000, 5000 + rows)[:, :cols].copy()


@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("rate", 4), ("rate", 16),
                                             ("precision", 17), ("accuracy", 1e-12)])
def test_packed_gemv_paper_like_slit(orc, mode_kind, param, rng):
    """378 x 8192 smooth slit: bit-exact vs the model (both evaluations),
    within the reference's bound vs oracle decompress + gemv(mixed,
    sequential), and >= 97 % of rows bit-identical with the exact products."""
    from fused_order import packed_model
    from paper_1902_08018_b200 import codec
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    C0 = smooth_matrix(378, 8192)
    s = codec.compress(C0, mode)
    C = orc.decompress(s)
    v = rng.random(8192).astype(np.float32)
    ref = orc.gemv_kernel(C, v, "mixed", "sequential")
    for ev in ("exact", "coefficient"):
        got = _packed_gemv(s, v, "mixed", ev)
        want = packed_model(orc, s, v, "mixed", ev)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), ev
        err = np.abs(got.astype(np.float64) - ref)
        assert (err <= bound(C, v)).all(), ev
        scale = np.abs(C).astype(np.float64) @ v.astype(np.float64)
        assert (err / scale).max() <= 1e-6, (ev, (err / scale).max())
        if ev == "exact":
            assert np.mean(got.view(np.uint32) == ref.view(np.uint32)) >= 0.97


def test_packed_row_ranges_plans_and_clone(orc, rng):
    """Row ranges (band edges and mid-band), plans over several jobs and a
    clone of a packed stream give the single-call bits."""
    import torch
    from paper_1902_08018_b200 import codec, _lib
    from paper_1902_08018_b200.executor import GemvPlan
    C0 = smooth_matrix(61, 3000)
    ds = codec.DeviceStream.from_host(codec.compress(C0, codec.FixedRate(8))).pack()
    v = torch.from_numpy(rng.random(3000).astype(np.float32)).cuda()
    for ev in ("exact", "coefficient"):
        full = ds.gemv(v, evaluation=ev).cpu().numpy()
        for rb, re in ((0, 61), (4, 20), (3, 9), (16, 32), (60, 61), (8, 8), (15, 17)):
            part = ds.gemv(v, evaluation=ev, row_begin=rb, row_end=re).cpu().numpy()
            assert np.array_equal(part, full[rb:re]), (ev, rb, re)
        c = ds.clone()
        assert c.packed
        assert np.array_equal(c.gemv(v, evaluation=ev).cpu().numpy(), full)
        out = torch.zeros(61 + 17, device="cuda")
        plan = GemvPlan([(ds, v, out[:40], 0, 40), (c, v, out[40:61], 40, 61),
                         (ds, v, out[61:], 4, 21)], evaluation=ev)
        st = _lib.status_word()
        plan.launch(st)
        o = out.cpu().numpy()
        assert np.array_equal(o[:61], full) and np.array_equal(o[61:], full[4:21])
        assert _lib.read_status(st) is None
        c.close()


def test_packed_flags_nonfinite():
    """codec.py:312-313 through the packed copy: decode raises, fused too."""
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    bits = [int(b) for b in format(200, "09b")] + [1]
    for w in [0x7F800000] + [0x3F800000] * 15:
        bits += [int(b) for b in format(w, "032b")]
    payload = np.packbits(np.array(bits, np.uint8))
    s = codec.CompressedStream(mode=codec.FixedAccuracy(0.0), rows=4, cols=4, payload=payload,
                               block_index=np.zeros(1, np.uint64), total_bits=len(bits))
    import torch
    ds = codec.DeviceStream.from_host(s).pack()
    assert ds.packed_exceptions == 1
    with pytest.raises(CorruptStreamError):
        ds.decode()
    with pytest.raises(CorruptStreamError):
        ds.gemv(torch.ones(4, device="cuda"))


def test_packed_rebind_drops_copy(rng):
    from paper_1902_08018_b200 import codec
    C0 = smooth_matrix(8, 512)
    s = codec.compress(C0, codec.FixedPrecision(17))
    ds = codec.DeviceStream.from_host(s).pack()
    assert ds.packed
    ds.rebind(ds.payload_bytes)
    assert not ds.packed


@pytest.mark.parametrize("policy", ["mixed", "single"])
def test_staged_kernel_wide_bands(orc, policy, rng):
    """Over 16 segments per virtual warp (1.1 M columns: the staged kernel's
    16-entry header ring wraps): bit-exact vs the CPU model."""
    from fused_order import packed_model
    from paper_1902_08018_b200 import codec
    C0 = smooth_matrix(9, 1_100_003, S=1_100_003)
    s = codec.compress(C0, codec.FixedRate(8))
    v = rng.random(C0.shape[1]).astype(np.float32)
    got = _packed_gemv(s, v, policy, "coefficient")
    want = packed_model(orc, s, v, policy, "coefficient")
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("evaluation", ["coefficient", "exact"])
def test_staged_kernel_runs_of_generic_segments(orc, evaluation, rng):
    """Long runs of generic segments (random data at a high rate: fields too
    wide for the fast path) between fast ones: the producer skips far ahead
    of the consumer through the header ring.  Every virtual warp sees a fast
    segment, 18 generic ones, then fast ones again; bit-exact vs the model."""
    from fused_order import packed_model
    from paper_1902_08018_b200 import codec
    seg_cols, vws = 4 * 32 * ph.seg_tiles_for("rate"), 32
    cols = 20 * vws * seg_cols
    C0 = smooth_matrix(6, cols, S=cols)
    wild = rng.standard_normal((6, 18 * vws * seg_cols)).astype(np.float32) * np.float32(1e-8)
    C0[:, vws * seg_cols:19 * vws * seg_cols] = wild
    s = codec.compress(C0, codec.FixedRate(24))
    v = rng.random(cols).astype(np.float32)
    got = _packed_gemv(s, v, "mixed", evaluation)
    want = packed_model(orc, s, v, "mixed", evaluation)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
