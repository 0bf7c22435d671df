"""The kernel plugin module (whff/backend.py:36-46 contract): NAME,
gemv_kernel, encode_blocks, decode_blocks -- backed by libwhff_b200.so.

A reference maintainer selects it exactly like the compiled backend; see
INTEGRATION.md.  There is no fallback: import succeeds, calls raise loudly
without the extension or a CUDA device.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

NAME = "b200"


def gemv_kernel(m, v, policy, shape, fanout=0):
    """K:80-132: float32 (H, W) C-contiguous, float32 (W,) -> float32 (H,)."""
    torch = _lib.require_cuda()
    from .mpgemv import gemv_device
    mt = torch.from_numpy(np.ascontiguousarray(m, dtype=np.float32)).cuda()
    vt = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
    return gemv_device(mt, vt, policy, shape, fanout if fanout else 2).cpu().numpy()


def decode_blocks(payload, offsets, seglens, n_planes, planes_limit, has_raw_flag):
    """K:371-408 -> (mag u32 (nb,16), neg u8 (nb,16), emax u16, raw u8,
    raw_words u32 (nb,16), consumed u64)."""
    torch = _lib.require_cuda()
    if int(n_planes) != 27:
        raise ValueError("n_planes must be 27")
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    seglens = np.ascontiguousarray(seglens, dtype=np.uint64)
    nb = offsets.size
    empty = (np.zeros((0, 16), np.uint32), np.zeros((0, 16), np.uint8), np.zeros(0, np.uint16),
             np.zeros(0, np.uint8), np.zeros((0, 16), np.uint32), np.zeros(0, np.uint64))
    if nb == 0:
        return empty
    h = ctypes.c_void_p()
    _lib.call("whff_dstream_create_segments", torch.cuda.current_device(), _lib.ptr(payload),
              payload.size, _lib.ptr(offsets), _lib.ptr(seglens), nb, int(planes_limit),
              int(bool(has_raw_flag)), ctypes.byref(h))
    from .codec import DeviceStream
    ds = DeviceStream(h, None)
    try:
        mag, neg, emax, raw, raw_words, consumed = ds.decode_blocks(0, nb, int(planes_limit))
        return (mag.cpu().numpy().view(np.uint32), neg.cpu().numpy(),
                emax.cpu().numpy().view(np.uint16), raw.cpu().numpy(),
                raw_words.cpu().numpy().view(np.uint32), consumed.cpu().numpy().view(np.uint64))
    finally:
        ds.close()


def encode_blocks(mag, neg, emax_code, planes, raw_mask, raw_words, n_planes, budget_bits,
                  has_raw_flag):
    """K:228-283 -> (payload uint8, bit offsets uint64 (nb,), total_bits)."""
    torch = _lib.require_cuda()
    nb = int(np.asarray(emax_code).shape[0])
    if nb == 0:
        return np.zeros(0, np.uint8), np.zeros(0, np.uint64), 0

    def dev(a, dt, tdt):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(dt)).view(tdt)).cuda()

    m = dev(mag, np.uint32, np.int32)
    n_ = dev(neg, np.uint8, np.uint8)
    e = dev(emax_code, np.uint16, np.int16)
    p = dev(planes, np.uint8, np.uint8)
    r = dev(raw_mask, np.uint8, np.uint8)
    w = dev(raw_words, np.uint32, np.int32)
    offs = torch.empty(nb, dtype=torch.int64, device="cuda")
    total = ctypes.c_uint64()
    args = (_lib.ptr(m), _lib.ptr(n_), _lib.ptr(e), _lib.ptr(p), _lib.ptr(r), _lib.ptr(w), nb,
            int(n_planes), int(budget_bits), int(bool(has_raw_flag)))
    _lib.call("whff_encode_blocks_size", *args, _lib.ptr(offs), ctypes.byref(total),
              _lib.cur_stream())
    nbytes = (total.value + 7) // 8
    payload = torch.zeros(((nbytes + 15) // 16) * 16 + 64, dtype=torch.uint8, device="cuda")
    _lib.call("whff_encode_blocks_emit", *args, _lib.ptr(offs), _lib.ptr(payload),
              _lib.cur_stream())
    return (payload[:nbytes].cpu().numpy(), offs.cpu().numpy().view(np.uint64),
            int(total.value))


# whff/backend.py:20-46 selector surface: one backend, no fallback
BACKEND_NAME = NAME


def available_backends():
    import sys
    return {NAME: sys.modules[__name__]}


def get_kernels(name=None):
    if name not in (None, NAME):
        raise ImportError(f"unknown backend {name!r} (only {NAME!r})")
    import sys
    return sys.modules[__name__]
