"""Launch-independent row sums: every block-row runs on 4 CTAs of 8 warps
whose 32 virtual-warp partials the last warp to finish adds with a fixed
butterfly.

A row's result must therefore be bit-identical whichever launch computes it:
a single call, a single call over a row sub-range, a one-job plan, or a plan
batching it with other streams -- in every stream variant (FixedRate(8),
another implicit rate, indexed, indexed with raw escapes), both layouts and
both evaluations -- and stay so across repeated launches (the per-row
arrival counters reset themselves)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def smooth_matrix(rows, cols, seed=0):
    from paper_1902_08018_b200 import synth
    spec = synth.Spec(grid_rows=16, grid_cols=16, S=cols, K=rows, M=rows, seed=seed)
    phase = np.random.default_rng(seed).random() * 2 * np.pi
    return synth.deformation_rows(spec, 0, phase, 0, rows)


def plan_out(jobs, evaluation, launches=2):
    import torch
    from paper_1902_08018_b200 import _lib
    from paper_1902_08018_b200.executor import GemvPlan
    outs = [torch.full((re - rb,), float("nan"), device="cuda") for _, _, rb, re in jobs]
    plan = GemvPlan([(ds, v, o, rb, re) for (ds, v, rb, re), o in zip(jobs, outs)],
                    evaluation=evaluation)
    res = []
    for _ in range(launches):
        st = _lib.status_word()
        plan.launch(st)
        torch.cuda.synchronize()
        assert _lib.read_status(st) is None
        res.append([o.cpu().numpy().copy() for o in outs])
    plan.close()
    return res


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.mark.parametrize("mode_kind,param", [("rate", 8), ("rate", 12), ("precision", 17),
                                             ("accuracy", 1e-12)])
@pytest.mark.parametrize("layout", ["reference", "skeleton-first"])
def test_rows_identical_across_launches(mode_kind, param, layout, rng):
    import torch
    from paper_1902_08018_b200 import codec
    mode = {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[mode_kind](param)
    # 5,003 block-columns = 157 groups: every virtual warp has 4-5 groups
    C = smooth_matrix(37, 20011, seed=3)
    C[5, 7:11] = 1e30               # one extreme-scale block (coefficient fallback)
    D = smooth_matrix(90, 20011, seed=4)
    streams = []
    for M in (C, D):
        ds = codec.DeviceStream.from_host(codec.compress(M, mode))
        if layout != "reference":
            ds.relayout(layout)
        streams.append(ds)
    a, b = streams
    v = torch.from_numpy(rng.random(C.shape[1]).astype(np.float32)).cuda()
    for ev in ("exact", "coefficient"):
        full_a = a.gemv(v, evaluation=ev).cpu().numpy()
        full_b = b.gemv(v, evaluation=ev).cpu().numpy()
        assert np.isfinite(full_a).all() and np.isfinite(full_b).all()
        assert same(a.gemv(v, evaluation=ev, row_begin=5, row_end=22).cpu().numpy(), full_a[5:22])
        for got in plan_out([(a, v, 0, 37)], ev):
            assert same(got[0], full_a), ev
        batched = [(b, v, 0, 90), (a, v, 5, 22), (b, v, 13, 14), (a, v, 0, 37), (a, v, 36, 37)]
        for got in plan_out(batched, ev):
            assert same(got[0], full_b) and same(got[1], full_a[5:22]), ev
            assert same(got[2], full_b[13:14]) and same(got[3], full_a), ev
            assert same(got[4], full_a[36:37]), ev


def test_plan_relaunch_and_single_call_workspace(rng):
    """Repeated plan launches and single calls reusing one workspace agree."""
    import torch
    from paper_1902_08018_b200 import codec
    C = smooth_matrix(64, 9000, seed=5)
    ds = codec.DeviceStream.from_host(codec.compress(C, codec.FixedRate(8))).relayout("skeleton-first")
    v = torch.from_numpy(rng.random(C.shape[1]).astype(np.float32)).cuda()
    ref = ds.gemv(v, evaluation="coefficient").cpu().numpy()
    for got in plan_out([(ds, v, 0, 64)], "coefficient", launches=4):
        assert same(got[0], ref)
    import ctypes
    from paper_1902_08018_b200 import _lib
    n = ctypes.c_size_t()
    _lib.call("whff_decode_gemv_workspace_size", ds.handle, _lib.EVAL["coefficient"], ctypes.byref(n))
    ws = torch.full((n.value // 4 + 4,), -1.0, device="cuda")   # arbitrary contents
    for rb, re in ((0, 64), (8, 40), (0, 64)):
        got = ds.gemv(v, evaluation="coefficient", row_begin=rb, row_end=re, workspace=ws)
        assert same(got.cpu().numpy(), ref[rb:re])
    ws_small = torch.zeros(4, device="cuda")
    from paper_1902_08018_b200.errors import WhffError
    with pytest.raises(WhffError):
        y = torch.empty(64, device="cuda")
        st = _lib.status_word()
        _lib.call("whff_decode_gemv", ds.handle, _lib.ptr(v), _lib.ptr(y), _lib.POLICY["mixed"],
                  _lib.EVAL["exact"], 0, 64, _lib.ptr(ws_small), 16, _lib.ptr(st), _lib.cur_stream())


def test_concurrent_plans_on_two_streams(rng):
    """Distinct plans (own partials and counters) over one resident stream,
    launched concurrently on two CUDA streams: each gives the single-call bits."""
    import torch
    from paper_1902_08018_b200 import _lib, codec
    from paper_1902_08018_b200.executor import GemvPlan
    C = smooth_matrix(96, 30011, seed=8)
    ds = codec.DeviceStream.from_host(codec.compress(C, codec.FixedRate(8))).relayout("skeleton-first")
    v1 = torch.from_numpy(rng.random(C.shape[1]).astype(np.float32)).cuda()
    v2 = torch.from_numpy(rng.random(C.shape[1]).astype(np.float32)).cuda()
    ref1 = ds.gemv(v1, evaluation="coefficient").cpu().numpy()
    ref2 = ds.gemv(v2, evaluation="coefficient").cpu().numpy()
    o1, o2 = torch.zeros(96, device="cuda"), torch.zeros(96, device="cuda")
    p1 = GemvPlan([(ds, v1, o1, 0, 96)], evaluation="coefficient")
    p2 = GemvPlan([(ds, v2, o2, 0, 96)], evaluation="coefficient")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    st1, st2 = _lib.status_word(), _lib.status_word()
    torch.cuda.synchronize()
    for _ in range(20):
        with torch.cuda.stream(s1):
            p1.launch(st1)
        with torch.cuda.stream(s2):
            p2.launch(st2)
    torch.cuda.synchronize()
    assert same(o1.cpu().numpy(), ref1) and same(o2.cpu().numpy(), ref2)
    p1.close()
    p2.close()
