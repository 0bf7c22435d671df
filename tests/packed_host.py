"""Host form of the tile-packed layout (test infrastructure).

Wraps tools/hostcheck.cpp's hc_pack / hc_unpack: the packer rules of
paper_1902_08018_b200/csrc/whff_packed.cuh compiled for the CPU, fed with
decode_blocks arrays (the oracle's or the reference's), and an unpacker that
reads every fast-path record with the kernels' funnel / magic-number
extraction.  The GPU tests compare the device packer byte-for-byte with
pack() and the device decode with the oracle.
"""

import numpy as np


def _p(a):
    import ctypes
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


MODE_CODE = {"rate": 0, "precision": 1, "accuracy": 2}


def _kind(mode):
    """("rate", 8) / "rate" / codec.FixedRate(8) -> "rate" (and so on)."""
    if isinstance(mode, str):
        return mode
    if isinstance(mode, tuple):
        return mode[0]
    return {"FixedRate": "rate", "FixedPrecision": "precision", "FixedAccuracy": "accuracy"}[type(mode).__name__]


def seg_tiles_for(mode):
    """Tiles per segment of a stream of codec mode `mode`:
    csrc/whff_packed.cuh seg_tiles_for_mode."""
    return 8 if _kind(mode) == "rate" else 16


def _code(mode):
    return MODE_CODE[_kind(mode)]


def pack(hc, mag, neg, emax, raw, raw_words, rows, cols, mode):
    """-> dict(segs uint8[nseg*48], body uint32, exc_block uint64, exc_words uint32[., 16],
    generic int): the packed representation of a stream's decoded blocks
    (`mode`: the stream's codec mode, which sets the segment size)."""
    import ctypes
    mag = np.ascontiguousarray(mag, np.uint32)
    neg = np.ascontiguousarray(neg, np.uint8)
    emax = np.ascontiguousarray(emax, np.uint16)
    raw = np.ascontiguousarray(raw, np.uint8)
    raw_words = np.ascontiguousarray(raw_words, np.uint32)
    nseg, nexc, gen = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    args = [_p(mag), _p(neg), _p(emax), _p(raw), _p(raw_words), int(rows), int(cols)]
    words = hc.hc_pack(*args, None, None, None, None, ctypes.byref(nseg), ctypes.byref(nexc),
                       ctypes.byref(gen), _code(mode))
    segs = np.zeros(nseg.value * 48, np.uint8)
    body = np.zeros(words + 4 * 16 * 32 + 64, np.uint32)      # the device's readable slack
    xb = np.zeros(max(nexc.value, 1), np.uint64)
    xw = np.zeros((max(nexc.value, 1), 16), np.uint32)
    hc.hc_pack(*args, _p(segs), _p(body), _p(xb), _p(xw), ctypes.byref(nseg), ctypes.byref(nexc),
               ctypes.byref(gen), _code(mode))
    return {"segs": segs, "body": body, "body_words": int(words), "exc_block": xb[:nexc.value],
            "exc_words": xw[:nexc.value], "generic": int(gen.value), "nseg": int(nseg.value),
            "mode": _code(mode)}


def unpack(hc, pk, rows, cols):
    """-> (float32 words (rows, cols), number of fast-path extraction mismatches)."""
    out = np.zeros((rows, cols), np.float32)
    xb = np.ascontiguousarray(pk["exc_block"], np.uint64)
    xw = np.ascontiguousarray(pk["exc_words"], np.uint32)
    bad = hc.hc_unpack(_p(pk["segs"]), _p(pk["body"]), _p(xb) if xb.size else None,
                       _p(xw) if xw.size else None, int(xb.size), int(rows), int(cols), _p(out),
                       pk["mode"])
    return out, int(bad)


def packed_bytes(pk):
    return pk["body_words"] * 4 + pk["segs"].size + pk["exc_block"].size * 72
