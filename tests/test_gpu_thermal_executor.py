"""Thermal step (bit-exact vs the reference) and the field-step executor vs
the reference pipeline's deformations (config 1, small mesh)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_thermal_step_bit_exact(golden):
    import scipy.sparse as sp
    from paper_1902_08018_b200 import thermal
    g = golden("thermal_cases")
    n = g["B"].size
    A = sp.csr_matrix((g["A_data"], g["A_indices"], g["A_indptr"]), shape=(n, n))
    P = sp.csr_matrix((g["P_data"], g["P_indices"], g["P_indptr"]), shape=(g["P_indptr"].size - 1, n))
    for t in range(4):
        nxt = thermal.thermal_step(A, g["B"], g[f"t{t}_T"], g[f"t{t}_u"])
        assert np.array_equal(nxt.view(np.uint32), g[f"t{t}_next"].view(np.uint32))
        s = thermal.thermal_interpolate(P, nxt)
        assert np.array_equal(s.view(np.uint32), g[f"t{t}_S"].view(np.uint32))


def test_thermal_validation():
    import scipy.sparse as sp
    from paper_1902_08018_b200 import thermal
    from paper_1902_08018_b200.errors import DimensionError, NonFiniteError
    A = sp.identity(8, format="csr", dtype=np.float64)
    B = np.ones(8, np.float32)
    u = np.zeros(8, np.float32)
    u[7] = np.nan
    with pytest.raises(NonFiniteError) as e:
        thermal.thermal_step(A, B, np.zeros(8, np.float32), u)
    assert e.value.index == 7
    with pytest.raises(DimensionError):
        thermal.thermal_step(A, B, np.zeros(7, np.float32), np.zeros(8, np.float32))


def test_light_steps_match_reference_pipeline(golden):
    """Config 1 (small mesh, FixedAccuracy(1e-12), pipeline defaults): the
    reference's per-light-step deformations vs the GPU fused products of the
    GPU-compressed slits (streams byte-identical to the reference's)."""
    from paper_1902_08018_b200 import codec
    from paper_1902_08018_b200.mpgemv import gemv_compressed
    g = golden("pipeline_small")
    eps = np.finfo(np.float32).eps
    ident = []
    for i, slit in enumerate(g["slits"]):
        S = g["S"][i]
        for a in "xyz":
            C = g[f"C_{a}_{slit}"]
            s = codec.compress(C, codec.FixedAccuracy(1e-12))
            assert np.array_equal(s.payload, g[f"payload_{a}_{slit}"])
            assert np.array_equal(s.block_index, g[f"index_{a}_{slit}"])
            want = g["D_" + a][i]
            got = gemv_compressed(s, S)
            Cd = codec.decompress(s)
            b = (Cd.shape[1] + 1) * eps * (np.abs(Cd).astype(np.float64) @ np.abs(S).astype(np.float64))
            assert (np.abs(got.astype(np.float64) - want) <= b + 1e-300).all()
            ident.append(np.mean(got.view(np.uint32) == want.view(np.uint32)))
    assert np.mean(ident) >= 0.95


def _small_field(seed=3):
    from paper_1902_08018_b200 import synth
    spec = synth.Spec(grid_rows=24, grid_cols=24, S=256, K=96, M=12, seed=seed, n_fields=2)
    return spec, synth.generate(spec)


def test_field_step_matches_oracle_and_graph_replay(orc):
    import torch
    from paper_1902_08018_b200 import codec, synth, thermal
    from paper_1902_08018_b200.executor import FieldStep
    spec, ops = _small_field()
    fields, slits = synth.windows(spec)
    f0, f1 = fields[0]
    n_slits = len(slits[0])
    mode = codec.FixedAccuracy(1e-12)
    streams, mats = [], []
    for ai, a in enumerate(synth.AXES):
        C = synth.deformation_rows(spec, ai, ops.phases[a], f0, f1)
        mats.append(C)
        streams.append([codec.compress_device(C[s * spec.M:(s + 1) * spec.M], mode)
                        for s in range(n_slits)])
    dark, fps, dose = synth.heatload(spec, len(fields), n_slits, seed=4)
    A, P = thermal.DeviceCSR(ops.A64()), thermal.DeviceCSR(ops.P64())
    B = torch.from_numpy(ops.B).cuda()
    fs = FieldStep(A, B, P, streams, spec.M, n_slits, torch.from_numpy(dark).cuda(),
                   torch.from_numpy(fps[(0, 0)]).cuda(), dose)
    # oracle: two steps of thermal + decompress/gemv(mixed, sequential)
    T = np.zeros(spec.T, np.float32)
    for step in range(2):
        fs.step()
        u = (np.float32(dose) * fps[(0, 0)] + dark).astype(np.float32)
        T = orc.thermal_step(ops.A64(), ops.B, T, u)
        S = orc.thermal_interpolate(ops.P64(), T)
        assert np.array_equal(fs.S.cpu().numpy(), S)
        D = fs.deformations()
        for ai in range(3):
            want = np.concatenate([orc.gemv_kernel(codec.decompress(streams[ai][s]).cpu().numpy(), S,
                                                   "mixed", "sequential") for s in range(n_slits)])
            assert np.abs(D[ai] - want).max() <= 1e-6 * np.abs(want).max()
    fs.check()
    # CUDA graph replay == eager
    d_eager = fs.deformations()
    fs.capture()
    fs.T.zero_()
    fs.replay()
    fs.replay()
    torch.cuda.synchronize()
    d_graph = fs.deformations()
    fs.T.zero_()
    fs.step_local()
    fs.step_local()
    torch.cuda.synchronize()
    d_eager2 = fs.deformations()
    for ai in range(3):
        assert np.array_equal(d_graph[ai], d_eager2[ai])
