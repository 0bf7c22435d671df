"""Fused decompress + GEMV (the hot path) against the CPU oracle's
decompress -> gemv(mixed, sequential) on identical inputs.

Tolerance (stated in DESIGN.md, the reference's own bound from
tests/test_mpgemv.py:116-130 and tests/test_acceptance.py:195-197):
    |y_gpu - y_ref| <= (W+1) * 2^-24 * sum_j |C_ij v_j|   per row.
The exact evaluation must additionally match bit-for-bit on (almost) every
row: products are the reference's binary32 products and the binary64 sum
only changes order."""

import numpy as np
import pytest

from conftest import golden_codec_cases, mode_tuple

pytestmark = pytest.mark.gpu
EPS32 = np.finfo(np.float32).eps


def bound(C, v):
    scale = np.abs(C).astype(np.float64) @ np.abs(v).astype(np.float64)
    return (C.shape[1] + 1) * EPS32 * scale


def check(got, ref, C, v, min_identical=None):
    b = bound(C, v)
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    assert (err <= b + 1e-300).all(), float((err - b).max())
    ident = float(np.mean(got.view(np.uint32) == ref.view(np.uint32)))
    if min_identical is not None:
        assert ident >= min_identical, ident
    return ident


def host_stream(case):
    from test_gpu_codec import host_stream as hs
    return hs(case)


@pytest.mark.parametrize("policy", ["mixed", "single", "double"])
def test_fused_exact_all_golden_streams(golden, orc, policy, rng):
    from paper_1902_08018_b200.mpgemv import gemv_compressed
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"]:
            continue
        s = host_stream(case)
        C = orc.decompress(s)
        v = rng.standard_normal(C.shape[1]).astype(np.float32)
        ref = orc.gemv_kernel(C, v, policy, "sequential")
        got = gemv_compressed(s, v, policy=policy)
        check(got, ref, C, v, min_identical=0.9 if policy != "single" else None)


def test_fused_coefficient_domain_within_bound(golden, orc, rng):
    from paper_1902_08018_b200.mpgemv import gemv_compressed
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"] or case["name"] in ("big", "dynrange", "subnormal"):
            continue
        s = host_stream(case)
        C = orc.decompress(s)
        v = rng.standard_normal(C.shape[1]).astype(np.float32)
        ref = orc.gemv_kernel(C, v, "mixed", "sequential")
        for pol in ("mixed", "single"):
            got = gemv_compressed(s, v, policy=pol, evaluation="coefficient")
            check(got, ref, C, v)


def smooth_matrix(rows, cols, seed=0):
    from paper_1902_08018_b200 import synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=cols, K=rows, M=rows, seed=seed)
    ops_phase = np.random.default_rng(seed).random() * 2 * np.pi
    return synth.deformation_rows(spec, 0, ops_phase, 0, rows)


@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("rate", 4), ("rate", 16), ("rate", 5),
                                             ("precision", 17), ("accuracy", 1e-12)])
def test_fused_paper_like_slit(orc, mode_kind, param, rng):
    """378 x 8192 smooth slit (the paper's slit shape, narrowed): every mode,
    both evaluations, vs oracle decompress + mixed sequential GEMV."""
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.mpgemv import gemv_compressed
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    C0 = smooth_matrix(378, 8192)
    s = codec.compress(C0, mode)
    C = orc.decompress(s)
    v = rng.random(8192).astype(np.float32)
    ref = orc.gemv_kernel(C, v, "mixed", "sequential")
    ident = check(gemv_compressed(s, v), ref, C, v, min_identical=0.97)
    check(gemv_compressed(s, v, evaluation="coefficient"), ref, C, v)
    # acceptance-3 style: median relative error vs binary64 <= 1e-7
    exact = C.astype(np.float64) @ v.astype(np.float64)
    rel = np.abs(gemv_compressed(s, v, evaluation="coefficient") - exact) / np.abs(exact)
    assert np.median(rel) <= 1e-7


def test_fused_row_ranges_and_plan(orc, rng):
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.executor import GemvPlan
    import torch
    C0 = smooth_matrix(61, 1000)
    ds = codec.DeviceStream.from_host(codec.compress(C0, codec.FixedRate(8)))
    v = torch.from_numpy(rng.random(1000).astype(np.float32)).cuda()
    full = ds.gemv(v).cpu().numpy()
    for rb, re in ((0, 61), (4, 20), (3, 9), (60, 61), (8, 8)):
        part = ds.gemv(v, row_begin=rb, row_end=re).cpu().numpy()
        assert np.array_equal(part, full[rb:re])
    out = torch.zeros(61 + 17, device="cuda")
    plan = GemvPlan([(ds, v, out[:40], 0, 40), (ds, v, out[40:61], 40, 61),
                     (ds, v, out[61:], 4, 21)])
    from paper_1902_08018_b200 import _lib
    st = _lib.status_word()
    plan.launch(st)
    o = out.cpu().numpy()
    assert np.array_equal(o[:61], full) and np.array_equal(o[61:], full[4:21])
    assert _lib.read_status(st) is None


def test_fused_flags_nonfinite_decoded_values():
    """codec.py:312-313: a stream that decodes to inf raises CorruptStreamError."""
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.errors import CorruptStreamError
    from paper_1902_08018_b200.mpgemv import gemv_compressed
    bits = [int(b) for b in format(200, "09b")] + [1]        # emax, raw flag
    for w in [0x7F800000] + [0x3F800000] * 15:                 # inf then ones
        bits += [int(b) for b in format(w, "032b")]
    payload = np.packbits(np.array(bits, np.uint8))
    s = codec.CompressedStream(mode=codec.FixedAccuracy(0.0), rows=4, cols=4, payload=payload,
                               block_index=np.zeros(1, np.uint64), total_bits=len(bits))
    with pytest.raises(CorruptStreamError):
        codec.decompress(s)
    with pytest.raises(CorruptStreamError):
        gemv_compressed(s, np.ones(4, np.float32))


def test_fused_checksum_property_mid_size(rng):
    """Mid-size (1024 x 65536, rate 8) size-independent property: the fused
    product equals GPU decompress followed by the GPU dense GEMV within the
    bound, and the column-sum identity sum_i y_i = (1^T C) v holds."""
    import torch
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.mpgemv import gemv_device
    C0 = torch.from_numpy(smooth_matrix(1024, 65536))
    ds = codec.compress_device(C0, codec.FixedRate(8))
    v = torch.from_numpy(rng.random(65536).astype(np.float32)).cuda()
    y = ds.gemv(v).double().cpu().numpy()
    C = ds.decode()
    y2 = gemv_device(C, v, "mixed", "blocked").double().cpu().numpy()
    Cn = C.cpu().numpy()
    b = bound(Cn, v.cpu().numpy())
    assert (np.abs(y - y2) <= 2 * b).all()
    colsum = Cn.astype(np.float64).sum(0)
    assert abs(y.sum() - colsum @ v.cpu().numpy().astype(np.float64)) <= 1e-6 * np.abs(y).sum()


@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("rate", 3), ("precision", 17),
                                             ("accuracy", 1e-12), ("accuracy", 0.0)])
def test_skeleton_first_layout_identical(orc, mode_kind, param, rng):
    """whff_dstream_relayout: same decoded words, same decode_blocks arrays,
    bit-identical fused products, reference bytes restored on download."""
    import torch
    from paper_1902_08018_b200 import codec
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    C0 = smooth_matrix(130, 3000) if param != 0.0 else rng.standard_normal((37, 91)).astype(np.float32)
    host = codec.compress(C0, mode)
    ref = codec.DeviceStream.from_host(host)
    sf = codec.DeviceStream.from_host(host).relayout("skeleton-first")
    assert sf.layout == "skeleton-first"
    assert torch.equal(ref.decode(), sf.decode())
    for a, b in zip(ref.decode_blocks(), sf.decode_blocks()):
        assert torch.equal(a, b)
    v = torch.from_numpy(rng.random(C0.shape[1]).astype(np.float32)).cuda()
    for ev in ("exact", "coefficient"):
        assert torch.equal(ref.gemv(v, evaluation=ev), sf.gemv(v, evaluation=ev))
    back = sf.to_host()
    assert np.array_equal(back.payload, host.payload)
    assert np.array_equal(back.block_index, host.block_index)
    sf.relayout("reference")
    assert torch.equal(ref.decode(), sf.decode())


def coefficient_bound(orc, s, C, v):
    """Error bound of the coefficient-domain evaluation: it applies the real
    inverse lift G to the block's coefficients instead of the integer lift, so
    each block contributes up to K quantisation steps 2^(e-26) per row times
    sum_j |v_j| over its columns (K = 16 covers the two lift passes' floors),
    on top of the reference's (W+1) 2^-24 sum|C v|."""
    mode = mode_of(s)
    seg = orc.segment_lengths(mode, s.payload.size, s.block_index)
    mag, neg, emax, raw, rw, _ = orc.decode_blocks(s.payload, s.block_index, seg, 27,
                                                   orc.planes_limit_for(mode), mode[0] == "accuracy")
    rows, cols = C.shape
    bc = (cols + 3) // 4
    vb = np.zeros(bc * 4)
    vb[:cols] = np.abs(v.astype(np.float64))
    vsum = vb.reshape(bc, 4).sum(1)
    step = np.where((emax > 0) & (raw == 0), np.ldexp(1.0, emax.astype(np.int64) - 160 - 26), 0.0)
    per_brow = (16 * step.reshape(-1, bc) * vsum[None, :]).sum(1)
    return bound(C, v) + np.repeat(per_brow, 4)[:rows]


def mode_of(s):
    m = s.mode
    kind = {"FixedRate": "rate", "FixedPrecision": "precision", "FixedAccuracy": "accuracy"}[type(m).__name__]
    return (kind, m.bpv if kind == "rate" else m.planes if kind == "precision" else m.tolerance)


@pytest.mark.parametrize("evaluation", ["exact", "coefficient"])
def test_skeleton_first_all_golden_streams(golden, orc, evaluation, rng):
    """The bench's layout on every golden stream of the reference (ragged
    shapes, raw escapes, zero blocks, extreme and subnormal scales -- the
    coefficient kernel's out-of-line exact fallback).  Exact: within the
    reference's bound; coefficient: within its own (documented) bound, which
    equals the reference's for blocks without a large intra-block dynamic
    range (the smooth WHFF operators) and is looser for adversarial ones."""
    import torch
    from paper_1902_08018_b200 import codec
    for case in golden_codec_cases(golden("codec_cases")):
        if not case["ok"]:
            continue
        s = host_stream(case)
        C = orc.decompress(s)
        v = rng.standard_normal(C.shape[1]).astype(np.float32)
        ref = orc.gemv_kernel(C, v, "mixed", "sequential")
        ds = codec.DeviceStream.from_host(s).relayout("skeleton-first")
        got = ds.gemv(torch.from_numpy(v).cuda(), evaluation=evaluation).cpu().numpy()
        ds.close()
        if evaluation == "exact":
            check(got, ref, C, v, min_identical=0.9)
        else:
            err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
            assert (err <= coefficient_bound(orc, s, C, v) + 1e-300).all(), case["name"]
