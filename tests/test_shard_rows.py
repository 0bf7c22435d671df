"""codec.shard_rows: a block-row range cut out of a stream's payload is
byte-identical to compressing that row window (every mode, ragged shapes,
the padded last block-row), with the oracle encoder as the reference."""

import numpy as np
import pytest

from paper_1902_08018_b200 import codec
from paper_1902_08018_b200.errors import DimensionError

MODES = [("rate", 8), ("rate", 5), ("precision", 17), ("accuracy", 1e-12), ("accuracy", 0.0)]


def as_mode(kind, p):
    return {"rate": codec.FixedRate, "precision": codec.FixedPrecision,
            "accuracy": codec.FixedAccuracy}[kind](p)


@pytest.mark.parametrize("kind,p", MODES)
def test_shard_equals_compressed_window(orc, kind, p):
    rng = np.random.default_rng(3)
    for rows, cols in ((37, 45), (64, 19), (9, 130), (4, 4)):
        C = (1e-8 * (np.cumsum(rng.standard_normal((rows, cols)), axis=1)
                     + rng.standard_normal((rows, cols)))).astype(np.float32)
        full = orc.compress(C, (kind, p))
        s = codec.CompressedStream(mode=as_mode(kind, p), rows=rows, cols=cols,
                                   payload=full.payload, block_index=full.block_index,
                                   total_bits=int(full.total_bits))
        cuts = sorted({0, rows} | {4 * int(x) for x in rng.integers(0, (rows + 3) // 4, 3)})
        for r0, r1 in zip(cuts[:-1], cuts[1:]):
            if r0 >= r1:
                continue
            sh = codec.shard_rows(s, r0, r1)
            ref = orc.compress(C[r0:r1], (kind, p))
            assert np.array_equal(sh.payload, ref.payload), (rows, cols, r0, r1)
            assert np.array_equal(sh.block_index, ref.block_index)
            assert sh.total_bits == int(ref.total_bits)
            assert np.array_equal(orc.decompress(sh).view(np.uint32), orc.decompress(ref).view(np.uint32))


def test_shard_rows_validation():
    s = codec.CompressedStream(mode=codec.FixedRate(8), rows=10, cols=4,
                               payload=np.zeros(48, np.uint8),
                               block_index=np.arange(3, dtype=np.uint64) * 128, total_bits=384)
    with pytest.raises(DimensionError):
        codec.shard_rows(s, 2, 8)
    with pytest.raises(DimensionError):
        codec.shard_rows(s, 0, 7)
    with pytest.raises(DimensionError):
        codec.shard_rows(s, 8, 12)
    assert codec.shard_rows(s, 8, 10).rows == 2
