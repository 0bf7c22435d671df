"""Row sharding of the field products across ranks (host logic) and the
gather/unpad path, including a world_size-2 gloo run."""

import os

import numpy as np
import pytest

from paper_1902_08018_b200.executor import shard_row_counts, shard_units


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n_slits,rows", [(52, 378), (4, 16), (3, 6), (1, 1), (5, 13)])
def test_shards_cover_every_row_once_in_order(world, n_slits, rows):
    n_axes = 3
    seen = []
    for r in range(world):
        jobs, (u0, u1) = shard_units(n_axes, n_slits, rows, world, r)
        for axis, slit, r0, r1 in jobs:
            assert 0 <= r0 < r1 <= rows
            assert r0 % 4 == 0
            seen.extend((axis, slit, i) for i in range(r0, r1))
    want = [(a, s, i) for a in range(n_axes) for s in range(n_slits) for i in range(rows)]
    assert seen == want


def test_shards_are_balanced():
    counts = shard_row_counts(3, 52, 378, 8)
    tot = [sum(c) for c in counts]
    assert max(tot) - min(tot) <= 8          # at most one 4-row unit apart
    assert sum(tot) == 3 * 52 * 378


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_axes, n_slits, rows = 3, 5, 13
    counts = shard_row_counts(n_axes, n_slits, rows, world)
    rank_rows = [sum(c) for c in counts]
    mx = max(rank_rows)
    jobs, _ = shard_units(n_axes, n_slits, rows, world, rank)
    # each rank "computes" rows = global row id, padded to mx
    local = torch.full((mx,), -1.0)
    off = 0
    for axis, slit, r0, r1 in jobs:
        for i in range(r0, r1):
            local[off] = axis * n_slits * rows + slit * rows + i
            off += 1
    gathered = torch.zeros(mx * world)
    dist.all_gather_into_tensor(gathered, local)
    parts = [gathered[r * mx: r * mx + rank_rows[r]] for r in range(world)]
    flat = torch.cat(parts).numpy()
    q.put((rank, flat.tolist()))
    dist.destroy_process_group()


def test_gloo_two_rank_gather_reassembles_field():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = list(range(3 * 5 * 13))
    assert res[0] == want and res[1] == want


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_byte_balanced_shards(world):
    """Variable-rate modes split by compressed bytes: contiguous,
    covering, and every rank within one unit's weight of total / world."""
    from paper_1902_08018_b200.executor import unit_bounds
    rng = np.random.default_rng(world)
    n_axes, n_slits, rows = 3, 7, 30
    bpr = (rows + 3) // 4
    w = rng.integers(20, 400, n_axes * n_slits * bpr)
    w[5:40] *= 9                                   # a heavy region
    b = unit_bounds(w.size, world, w)
    assert b[0] == 0 and b[-1] == w.size and all(x <= y for x, y in zip(b, b[1:]))
    loads = [int(w[b[r]:b[r + 1]].sum()) for r in range(world)]
    assert max(loads) - w.sum() / world <= w.max()
    seen = []
    for r in range(world):
        jobs, (u0, u1) = shard_units(n_axes, n_slits, rows, world, r, w)
        assert (u0, u1) == (b[r], b[r + 1])
        for axis, slit, r0, r1 in jobs:
            seen.extend((axis, slit, i) for i in range(r0, r1))
    assert seen == [(a, s, i) for a in range(n_axes) for s in range(n_slits) for i in range(rows)]
    assert unit_bounds(10, 3, np.ones(10)) == unit_bounds(10, 3)
