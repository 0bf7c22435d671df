"""The C ABI: every symbol include/whff_b200.h declares is exported by the
built library and bound by the Python layer (no compute calls: CPU-safe)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "whff_b200.h")
LIB = os.path.join(ROOT, "paper_1902_08018_b200", "libwhff_b200.so")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(whff_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("whff_dstream_create", "whff_decode_blocks", "whff_decode", "whff_decode_gemv",
                 "whff_gemv", "whff_compress", "whff_encode_blocks_size", "whff_encode_blocks_emit",
                 "whff_gemv_plan_create", "whff_gemv_plan_launch", "whff_csr_matvec"):
        assert must in names


def test_python_binding_covers_header():
    from paper_1902_08018_b200 import _lib
    assert sorted(_lib.exported_symbols()) == declared()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libwhff_b200.so not built")
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(L, name), name
    L.whff_abi_version.restype = ctypes.c_int
    assert L.whff_abi_version() == 2
    L.whff_status_string.restype = ctypes.c_char_p
    L.whff_status_string.argtypes = [ctypes.c_int]
    assert L.whff_status_string(3) == b"corrupt stream"


@pytest.mark.skipif(not os.path.exists(LIB), reason="libwhff_b200.so not built")
def test_library_validates_without_gpu():
    """Argument validation happens before any device work."""
    from paper_1902_08018_b200 import _lib
    from paper_1902_08018_b200.errors import CorruptStreamError, WhffError
    import numpy as np
    L = _lib.lib()
    h = ctypes.c_void_p()
    payload = np.zeros(4, np.uint8)
    index = np.zeros(3, np.uint64)           # wrong block count for 4x4
    st = L.whff_dstream_create(0, 0, 8.0, 4, 4, _lib.ptr(payload), 4, _lib.ptr(index), 3, ctypes.byref(h))
    with pytest.raises(CorruptStreamError):
        _lib.check(st)
    st = L.whff_dstream_create(0, 0, 40.0, 4, 4, _lib.ptr(payload), 4, _lib.ptr(index), 1, ctypes.byref(h))
    with pytest.raises(WhffError):
        _lib.check(st)
    big = np.array([64], np.uint64)          # offset past the payload
    st = L.whff_dstream_create(0, 1, 8.0, 4, 4, _lib.ptr(payload), 4, _lib.ptr(big), 1, ctypes.byref(h))
    with pytest.raises(CorruptStreamError):
        _lib.check(st)


def test_backend_plugin_surface():
    """whff/backend.py:36-46 contract: NAME, gemv_kernel, encode_blocks, decode_blocks."""
    from paper_1902_08018_b200 import backend
    assert backend.NAME == "b200"
    for fn in ("gemv_kernel", "encode_blocks", "decode_blocks"):
        assert callable(getattr(backend, fn))
    assert backend.get_kernels() is backend
    with pytest.raises(ImportError):
        backend.get_kernels("python")
