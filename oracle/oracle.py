"""ctypes front end of the CPU oracle (oracle/whff_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the parity checker, never by the product
package (paper_1902_08018_b200).  Functions mirror the reference API so the
parity tests read like the reference's own tests:

* decode_blocks   <- whff._kernels.decode_blocks   (K:371-408)
* decompress      <- whff.codec.decompress         (codec.py:296-314, :335-357)
* compress        <- whff.codec.compress           (codec.py:225-293, K:228-283)
* gemv_kernel     <- whff._kernels.gemv_kernel     (K:80-132)
* thermal_step    <- whff.thermal.thermal_step     (thermal.py:98-109)
* thermal_interpolate <- whff.thermal.thermal_interpolate (thermal.py:112-117)

Modes are duck-typed: any object whose class is named FixedRate /
FixedPrecision / FixedAccuracy with the reference's field names (bpv /
planes / tolerance), or a tuple ("rate"|"precision"|"accuracy", param).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liborc.so")
N_PLANES = 27
_lib = None


def build():
    """Compile oracle/liborc.so (the checker; building it is not using it)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        L.orc_decode_blocks.argtypes = [p, i64, p, p, i64, ci, ci, ci, p, p, p, p, p, p]
        L.orc_decode_blocks.restype = None
        L.orc_reconstruct_blocks.argtypes = [p, p, p, p, p, i64, p]
        L.orc_reconstruct_blocks.restype = None
        L.orc_decompress.argtypes = [p, i64, p, p, i64, i64, ci, ci, p]
        L.orc_decompress.restype = i64
        L.orc_gemv.argtypes = [p, p, i64, i64, ci, ci, ci, p]
        L.orc_gemv.restype = ci
        L.orc_compress.argtypes = [p, i64, i64, ci, ctypes.c_double, p, p]
        L.orc_compress.restype = i64
        L.orc_thermal_step.argtypes = [p, p, p, i64, p, p, p, p]
        L.orc_thermal_step.restype = None
        L.orc_csr_matvec_f32out.argtypes = [p, p, p, i64, p, p]
        L.orc_csr_matvec_f32out.restype = None
        L.orc_num_threads.restype = ci
        L.orc_encode_blocks.argtypes = [p, p, p, p, p, p, i64, ci, ci, p, p]
        L.orc_encode_blocks.restype = i64
        _lib = L
    return _lib


def num_threads():
    return int(lib().orc_num_threads())


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def mode_kind(mode):
    """-> (code, param): 0 rate, 1 precision, 2 accuracy (codec.py:35-37)."""
    if isinstance(mode, tuple):
        kind, param = mode
    else:
        kind = {"FixedRate": "rate", "FixedPrecision": "precision",
                "FixedAccuracy": "accuracy"}[type(mode).__name__]
        param = {"rate": "bpv", "precision": "planes", "accuracy": "tolerance"}[kind]
        param = getattr(mode, param)
    return {"rate": 0, "precision": 1, "accuracy": 2}[kind], param


# ---------------------------------------------------------------------------
# decode side
# ---------------------------------------------------------------------------

def decode_blocks(payload, offsets, seglens, n_planes, planes_limit, has_raw_flag):
    """K:371-408; returns (mag, neg, emax_code, raw, raw_words, consumed)."""
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    seglens = np.ascontiguousarray(seglens, dtype=np.uint64)
    nb = offsets.shape[0]
    mag = np.zeros((nb, 16), np.uint32)
    neg = np.zeros((nb, 16), np.uint8)
    emax = np.zeros(nb, np.uint16)
    raw = np.zeros(nb, np.uint8)
    raw_words = np.zeros((nb, 16), np.uint32)
    consumed = np.zeros(nb, np.uint64)
    lib().orc_decode_blocks(_ptr(payload), payload.size, _ptr(offsets), _ptr(seglens),
                            nb, int(n_planes), int(planes_limit), int(bool(has_raw_flag)),
                            _ptr(mag), _ptr(neg), _ptr(emax), _ptr(raw),
                            _ptr(raw_words), _ptr(consumed))
    return mag, neg, emax, raw, raw_words, consumed


def reconstruct_blocks(mag, neg, emax, raw, raw_words):
    """codec.py:209-218 -> float32 (nb, 4, 4)."""
    nb = mag.shape[0]
    out = np.empty((nb, 4, 4), np.float32)
    mag = np.ascontiguousarray(mag, np.uint32)
    neg = np.ascontiguousarray(neg, np.uint8)
    emax = np.ascontiguousarray(emax, np.uint16)
    raw = None if raw is None else np.ascontiguousarray(raw, np.uint8)
    raw_words = np.ascontiguousarray(
        np.zeros((nb, 16), np.uint32) if raw_words is None else raw_words, np.uint32)
    lib().orc_reconstruct_blocks(_ptr(mag), _ptr(neg), _ptr(emax), _ptr(raw),
                                 _ptr(raw_words), nb, _ptr(out))
    return out


def segment_lengths(mode, payload_size, block_index):
    """codec.py:335-344."""
    code, param = mode_kind(mode)
    nb = block_index.shape[0]
    if code == 0:
        return np.full(nb, int(param) * 16, dtype=np.uint64)
    ends = np.empty(nb, dtype=np.uint64)
    ends[:-1] = block_index[1:]
    ends[-1] = payload_size * 8
    if (ends < block_index).any():
        raise ValueError("block index offsets are not nondecreasing")
    return ends - block_index


def planes_limit_for(mode):
    """codec.py:301-303."""
    code, param = mode_kind(mode)
    return min(int(param), N_PLANES) if code == 1 else N_PLANES


def decompress(stream):
    """codec.py:296-314 (stream validation is the caller's business)."""
    code, _ = mode_kind(stream.mode)
    payload = np.ascontiguousarray(stream.payload, np.uint8)
    index = np.ascontiguousarray(stream.block_index, np.uint64)
    seg = segment_lengths(stream.mode, payload.size, index)
    out = np.empty((stream.rows, stream.cols), np.float32)
    bad = lib().orc_decompress(_ptr(payload), payload.size, _ptr(index), _ptr(seg),
                               stream.rows, stream.cols, planes_limit_for(stream.mode),
                               int(code == 2), _ptr(out))
    if bad >= 0:
        raise ValueError("decoded array contains non-finite values")
    return out


# ---------------------------------------------------------------------------
# encode side
# ---------------------------------------------------------------------------

def compress(array, mode):
    """codec.py:225-268 -> SimpleNamespace(mode, rows, cols, payload, block_index, total_bits)."""
    a = np.ascontiguousarray(array, dtype=np.float32)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"codec input must be 2D and nonempty, got shape {a.shape}")
    if not np.isfinite(a).all():
        raise ValueError("codec input contains non-finite values")
    rows, cols = a.shape
    nb = ((rows + 3) // 4) * ((cols + 3) // 4)
    code, param = mode_kind(mode)
    offsets = np.zeros(nb, np.uint64)
    total = lib().orc_compress(_ptr(a), rows, cols, code, float(param), _ptr(offsets), None)
    if total < 0:
        raise ValueError("internal error: transform coefficient overflow")
    payload = np.zeros((total + 7) // 8, np.uint8)
    total2 = lib().orc_compress(_ptr(a), rows, cols, code, float(param), _ptr(offsets),
                                _ptr(payload))
    assert total2 == total
    return SimpleNamespace(mode=mode, rows=rows, cols=cols, payload=payload,
                           block_index=offsets, total_bits=int(total), block_size=4)


def encode_blocks(mag, neg, emax_code, planes, raw_mask, raw_words, n_planes, budget_bits,
                  has_raw_flag):
    """K:228-283 -> (payload uint8, offsets uint64, total_bits)."""
    assert int(n_planes) == N_PLANES
    mag = np.ascontiguousarray(mag, np.uint32)
    neg = np.ascontiguousarray(neg, np.uint8)
    emax = np.ascontiguousarray(emax_code, np.uint16)
    planes = np.ascontiguousarray(planes, np.uint8)
    raw_mask = np.ascontiguousarray(raw_mask, np.uint8)
    raw_words = np.ascontiguousarray(raw_words, np.uint32)
    nb = emax.size
    offsets = np.zeros(nb, np.uint64)
    args = [_ptr(mag), _ptr(neg), _ptr(emax), _ptr(planes), _ptr(raw_mask), _ptr(raw_words), nb,
            int(budget_bits), int(bool(has_raw_flag)), _ptr(offsets)]
    total = lib().orc_encode_blocks(*args, None)
    payload = np.zeros((total + 7) // 8, np.uint8)
    lib().orc_encode_blocks(*args, _ptr(payload))
    return payload, offsets, int(total)


# ---------------------------------------------------------------------------
# GEMV and thermal
# ---------------------------------------------------------------------------

_POL = {"mixed": 0, "single": 1, "double": 2}
_SHAPE = {"sequential": 0, "fixed-tree": 1}


def gemv_kernel(m, v, policy, shape, fanout=0):
    """K:80-132."""
    m = np.ascontiguousarray(m, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    h, w = m.shape
    out = np.empty(h, np.float32)
    err = lib().orc_gemv(_ptr(m), _ptr(v), h, w, _POL[policy], _SHAPE[shape],
                         int(fanout), _ptr(out))
    if err:
        raise MemoryError()
    return out


def gemv_mixed_seq(m, v):
    return gemv_kernel(m, v, "mixed", "sequential")


def _csr_parts(A64):
    indptr = np.ascontiguousarray(A64.indptr, np.int64)
    indices = np.ascontiguousarray(A64.indices, np.int32)
    data = np.ascontiguousarray(A64.data, np.float64)
    return indptr, indices, data


def thermal_step(A64, B, T_k, u_k):
    """thermal.py:98-109 (fp64 CSR accumulate in CSR order, fp32 store)."""
    indptr, indices, data = _csr_parts(A64)
    n = indptr.size - 1
    B = np.ascontiguousarray(B, np.float32)
    T_k = np.ascontiguousarray(T_k, np.float32)
    u_k = np.ascontiguousarray(u_k, np.float32)
    out = np.empty(n, np.float32)
    lib().orc_thermal_step(_ptr(indptr), _ptr(indices), _ptr(data), n, _ptr(B),
                           _ptr(T_k), _ptr(u_k), _ptr(out))
    return out


def thermal_interpolate(P64, T_next):
    """thermal.py:112-117."""
    indptr, indices, data = _csr_parts(P64)
    n = indptr.size - 1
    T_next = np.ascontiguousarray(T_next, np.float32)
    out = np.empty(n, np.float32)
    lib().orc_csr_matvec_f32out(_ptr(indptr), _ptr(indices), _ptr(data), n,
                                _ptr(T_next), _ptr(out))
    return out
