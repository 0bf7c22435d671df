"""Row-sharded field step with 2 ranks on one GPU (gloo transport: NCCL will
not put two ranks on one device).  The gathered deformations must equal the
single-rank step bit-for-bit (sharding never splits a row's reduction)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _field(rank, world, port, q, mode_vec, mode="rate", layout="skeleton-first"):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1902_08018_b200 import codec, synth, thermal
    from paper_1902_08018_b200.executor import FieldStep, shard_units
    spec = synth.Spec(grid_rows=24, grid_cols=24, S=512, K=7 * 13, M=13, seed=3, n_fields=1)
    ops = synth.generate(spec)
    cmode = codec.FixedRate(8) if mode == "rate" else codec.FixedAccuracy(1e-12)
    weights = None
    streams = [[None] * 7 for _ in range(3)]

    def make(a, s):
        rows = synth.deformation_rows(spec, a, ops.phases[synth.AXES[a]], s * 13, (s + 1) * 13)
        ds = codec.compress_device(rows, cmode)
        return ds.pack() if layout == "packed" else ds.relayout(layout)
    if mode != "rate":
        # byte-balanced shards: every rank sizes every slit stream
        from paper_1902_08018_b200.executor import unit_weights
        for a in range(3):
            for s in range(7):
                streams[a][s] = make(a, s)
        weights = unit_weights(streams, 3, 7)
    jobs, _ = shard_units(3, 7, 13, world, rank, weights)
    need = {(a, s) for a, s, _, _ in jobs}
    for a in range(3):
        for s in range(7):
            if (a, s) in need and streams[a][s] is None:
                streams[a][s] = make(a, s)
            elif (a, s) not in need and streams[a][s] is not None:
                streams[a][s].close()
                streams[a][s] = None
    dark, fps, dose = synth.heatload(spec, 1, 7, seed=1)
    fs = FieldStep(thermal.DeviceCSR(ops.A64()), torch.from_numpy(ops.B).cuda(),
                   thermal.DeviceCSR(ops.P64()), streams, 13, 7, torch.from_numpy(dark).cuda(),
                   torch.from_numpy(fps[(0, 0)]).cuda(), dose, world=world, rank=rank,
                   vector_mode=mode_vec, weights=weights,
                   evaluation="coefficient" if layout == "packed" else "exact")
    out = []
    for _ in range(3):
        fs.step()
        torch.cuda.synchronize()
        d = fs.deformations()
        out.append(np.concatenate([d[a] for a in range(3)]))
    fs.check()
    q.put((rank, np.stack(out)))
    if world > 1:
        dist.destroy_process_group()


def _run(world, mode_vec, mode="rate", layout="skeleton-first"):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_field, args=(r, world, port, q, mode_vec, mode, layout)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("mode_vec", ["broadcast", "replicate"])
def test_two_rank_field_step_equals_single_rank(mode_vec):
    single = _run(1, mode_vec)[0]
    two = _run(2, mode_vec)
    assert np.array_equal(two[0], single)
    assert np.array_equal(two[1], single)


def test_byte_balanced_accuracy_split_equals_single_rank():
    """FixedAccuracy(1e-12) streams (variable rate), tile-packed, coefficient
    evaluation, split by compressed bytes over 2 ranks: bit-identical to one
    rank."""
    single = _run(1, "replicate", "accuracy", "packed")[0]
    two = _run(2, "replicate", "accuracy", "packed")
    assert np.array_equal(two[0], single)
    assert np.array_equal(two[1], single)
