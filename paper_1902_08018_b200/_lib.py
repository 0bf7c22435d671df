"""ctypes binding of libwhff_b200.so (the C ABI in include/whff_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present every call raises.  Device buffers are torch tensors (PyTorch is the
allocator and stream provider); the library only ever sees raw pointers.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import CorruptStreamError, DimensionError, NonFiniteError, WhffError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WHFF_LIB", os.path.join(HERE, "libwhff_b200.so"))

OK, E_DIM, E_NONFINITE, E_CORRUPT, E_ARG, E_OVERFLOW, E_NOMEM, E_CUDA = range(8)
MODE_RATE, MODE_PRECISION, MODE_ACCURACY = 0, 1, 2
POLICY = {"mixed": 0, "single": 1, "double": 2}
SHAPE = {"sequential": 0, "fixed-tree": 1, "blocked": 2}
EVAL = {"exact": 0, "coefficient": 1}
INDEX_KIND = {0: "implicit", 1: "compact", 2: "full"}
LAYOUT = {"reference": 0, "skeleton-first": 1}
LAYOUT_NAME = {v: k for k, v in LAYOUT.items()}
STATUS_CLEAR = -1  # UINT64_MAX viewed as int64


class DStreamInfo(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("index_kind", ctypes.c_int32),
                ("param", ctypes.c_double), ("rows", ctypes.c_uint64),
                ("cols", ctypes.c_uint64), ("n_blocks", ctypes.c_uint64),
                ("payload_bytes", ctypes.c_uint64), ("total_bits", ctypes.c_uint64),
                ("index_bytes", ctypes.c_uint64),
                ("device_bytes", ctypes.c_uint64), ("planes_limit", ctypes.c_int32),
                ("has_raw_flag", ctypes.c_int32), ("layout", ctypes.c_int32),
                ("packed", ctypes.c_int32), ("packed_bytes", ctypes.c_uint64),
                ("packed_exceptions", ctypes.c_uint64), ("device", ctypes.c_int32)]


_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I = ctypes.c_int
_SIG = {
    "whff_abi_version": ([], _I),
    "whff_status_string": ([_I], ctypes.c_char_p),
    "whff_last_error": ([], ctypes.c_char_p),
    "whff_dstream_create": ([_I, _I, ctypes.c_double, _U64, _U64, _P, _U64, _P, _U64, _P], _I),
    "whff_dstream_create_segments": ([_I, _P, _U64, _P, _P, _U64, _I, _I, _P], _I),
    "whff_dstream_destroy": ([_P], _I),
    "whff_dstream_clone": ([_P, _P], _I),
    "whff_dstream_relayout": ([_P, _I, _P], _I),
    "whff_dstream_pack": ([_P, _P], _I),
    "whff_dstream_packed_download": ([_P, _P, _P, _P, _P, _P, _P, _P], _I),
    "whff_dstream_get_info": ([_P, _P], _I),
    "whff_dstream_block_row_bits": ([_P, _P], _I),
    "whff_dstream_download": ([_P, _P, _P], _I),
    "whff_dstream_export": ([_P, _P, _P, _P, _P], _I),
    "whff_dstream_reserve": ([_P, _U64], _I),
    "whff_dstream_rebind": ([_P, _U64], _I),
    "whff_dstream_import_async": ([_P, _P, _U64, _P, _U64, _P], _I),
    "whff_compress": ([_P, _U64, _U64, _U64, _I, ctypes.c_double, _P, _P], _I),
    "whff_encode_blocks_size": ([_P, _P, _P, _P, _P, _P, _U64, _I, _I, _I, _P, _P, _P], _I),
    "whff_encode_blocks_emit": ([_P, _P, _P, _P, _P, _P, _U64, _I, _I, _I, _P, _P, _P], _I),
    "whff_decode_blocks": ([_P, _U64, _U64, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "whff_decode_block_words": ([_P, _U64, _U64, _P, _P], _I),
    "whff_decode": ([_P, _P, _U64, _P, _P], _I),
    "whff_decode_gemv_workspace_size": ([_P, _I, _P], _I),
    "whff_decode_gemv": ([_P, _P, _P, _I, _I, _U64, _U64, _P, ctypes.c_size_t, _P, _P], _I),
    "whff_gemv_plan_create": ([_I, _P, _P, _P, _P, _P, _I, _I, _P], _I),
    "whff_gemv_plan_launch": ([_P, _P, _P], _I),
    "whff_gemv_plan_traffic": ([_P, _P, _P, _P], _I),
    "whff_gemv_plan_destroy": ([_P], _I),
    "whff_gemv_workspace_size": ([_U64, _U64, _I, _I, _I, _P], _I),
    "whff_gemv": ([_P, _U64, _U64, _U64, _P, _P, _I, _I, _I, _P, ctypes.c_size_t, _P], _I),
    "whff_gemv_oracle": ([_P, _U64, _U64, _U64, _P, _P, _P], _I),
    "whff_gemv_oracle_f64": ([_P, _U64, _U64, _U64, _P, _P, _P], _I),
    "whff_find_nonfinite": ([_P, _U64, _P, _P], _I),
    "whff_csr_matvec": ([_P, _P, _P, _U64, _P, _P, _P, _P, _P], _I),
    "whff_source_term": ([_P, _P, ctypes.c_float, _U64, _P, _P], _I),
    "whff_device_timestamp": ([_P, _P], _I),
    "whff_wait_until": ([_P, _U64, _P], _I),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the extension; raise loudly if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is not built; run `python -m paper_1902_08018_b200.build` "
                        "(there is no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (args, res) in _SIG.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = res
                _lib = L
    return _lib


def exported_symbols():
    return sorted(_SIG)


def check(status, what=""):
    """Map a whff_status_t onto the errors.py classes."""
    if status == OK:
        return
    L = lib()
    msg = (L.whff_last_error() or b"").decode(errors="replace")
    base = (L.whff_status_string(status) or b"").decode()
    text = f"{what}: {msg or base}" if what else (msg or base)
    if status == E_DIM:
        raise DimensionError(msg or base)
    if status == E_CORRUPT:
        raise CorruptStreamError(msg or base)
    if status in (E_ARG, E_OVERFLOW):
        raise WhffError(msg or base)
    if status == E_NOMEM:
        raise MemoryError(text)
    if status == E_NONFINITE:
        raise NonFiniteError(what or "value", -1)
    raise RuntimeError(f"CUDA failure in {text}")


def call(name, *args):
    check(getattr(lib(), name)(*args), name)


def ptr(t):
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)


def cur_stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1902_08018_b200 needs a CUDA device (no CPU fallback)")
    return torch


def status_word(device=None):
    torch = require_cuda()
    return torch.full((1,), STATUS_CLEAR, dtype=torch.int64,
                      device=device if device is not None else "cuda")


def read_status(word):
    """-> None if clear, else the flat index recorded by the device."""
    v = int(word.item())
    return None if v == STATUS_CLEAR else v
