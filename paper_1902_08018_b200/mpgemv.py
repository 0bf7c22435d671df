"""Mixed-precision dense matrix-vector products on the B200.

Mirrors whff.mpgemv (mpgemv.py): GemvRequest, gemv, gemv_oracle,
reduction_bits_lost, relative_error; adds gemv_compressed, the fused
decompress + GEMV over an HBM-resident compressed stream.

Policies (mpgemv.py:1-7): mixed = binary32 products, binary64 sum; single =
binary32 both; double = binary64 products and sum.  Reduction shapes:
"sequential" and "fixed-tree" are bit-exact with the reference
(_kernels.pyx:24-77); "blocked" is the B200 fast path (fixed per-warp split +
xor butterfly, deterministic) used by the fused kernel.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CorruptStreamError, DimensionError, NonFiniteError, WhffError

POLICIES = ("mixed", "single", "double")
SHAPES = ("sequential", "fixed-tree", "blocked")
EVALUATIONS = ("exact", "coefficient")


@dataclass(frozen=True)
class GemvRequest:
    matrix: object
    vector: object
    precision_policy: str = "mixed"
    reduction_shape: str = "sequential"
    fanout: int = 2

    def __post_init__(self):
        if self.precision_policy not in POLICIES:
            raise WhffError(f"unknown precision policy {self.precision_policy!r}")
        if self.reduction_shape not in SHAPES:
            raise WhffError(f"unknown reduction shape {self.reduction_shape!r}")
        if self.reduction_shape == "fixed-tree":
            f = self.fanout
            if f < 2 or (f & (f - 1)) != 0:
                raise WhffError(f"tree fanout must be a power of two >= 2, got {f}")


def _to_device(x, ndim):
    torch = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=torch.float32)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float32)).cuda()
    return t.contiguous()


def _check_inputs(m, v):
    """mpgemv.py:42-51 on the device (shape checks + first non-finite index)."""
    from .codec import find_nonfinite
    if m.dim() != 2 or v.dim() != 1 or m.shape[1] != v.shape[0]:
        raise DimensionError(
            f"gemv shapes do not agree: matrix {tuple(m.shape)}, vector {tuple(v.shape)}")
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise DimensionError("gemv operands must be nonempty")
    bad = find_nonfinite(m)
    if bad is not None:
        raise NonFiniteError("matrix", bad)
    bad = find_nonfinite(v)
    if bad is not None:
        raise NonFiniteError("vector", bad)


def gemv_device(m, v, policy="mixed", shape="sequential", fanout=2, out=None):
    """K:80-132 on CUDA tensors (no input checks)."""
    torch = _lib.require_cuda()
    rows, cols = m.shape
    if out is None:
        out = torch.empty(rows, dtype=torch.float32, device=m.device)
    ws_bytes = ctypes.c_size_t()
    _lib.call("whff_gemv_workspace_size", rows, cols, _lib.POLICY[policy], _lib.SHAPE[shape],
              int(fanout), ctypes.byref(ws_bytes))
    ws = None
    if ws_bytes.value:
        ws = torch.empty(ws_bytes.value // 8 + 8, dtype=torch.float64, device=m.device)
    _lib.call("whff_gemv", _lib.ptr(m), m.stride(0), rows, cols, _lib.ptr(v), _lib.ptr(out),
              _lib.POLICY[policy], _lib.SHAPE[shape], int(fanout), _lib.ptr(ws), ws_bytes.value,
              _lib.cur_stream())
    return out


def gemv(req, backend=None):
    """Evaluate a GemvRequest (mpgemv.py:54-61).  numpy in -> numpy out,
    CUDA tensors in -> CUDA tensor out."""
    torch = _lib.require_cuda()
    on_device = isinstance(req.matrix, torch.Tensor) and req.matrix.is_cuda
    m = _to_device(req.matrix, 2)
    v = _to_device(req.vector, 1)
    _check_inputs(m, v)
    out = gemv_device(m, v, req.precision_policy, req.reduction_shape, req.fanout)
    return out if on_device else out.cpu().numpy()


def gemv_oracle(matrix, vector):
    """Binary64 ground truth, sequential order (mpgemv.py:64-69), on device.
    Binary64 inputs stay binary64 (the reference casts to float64 first)."""
    torch = _lib.require_cuda()
    if _is_f64(matrix) or _is_f64(vector):
        m = _to_device_f64(matrix, 2)
        v = _to_device_f64(vector, 1)
        if m.shape[1] != v.shape[0] or m.shape[0] < 1 or m.shape[1] < 1:
            raise DimensionError(
                f"gemv shapes do not agree: matrix {tuple(m.shape)}, vector {tuple(v.shape)}")
        if not bool(torch.isfinite(m).all()):
            raise NonFiniteError("matrix", int(torch.nonzero(~torch.isfinite(m.reshape(-1)))[0]))
        if not bool(torch.isfinite(v).all()):
            raise NonFiniteError("vector", int(torch.nonzero(~torch.isfinite(v))[0]))
        out = torch.empty(m.shape[0], dtype=torch.float64, device=m.device)
        _lib.call("whff_gemv_oracle_f64", _lib.ptr(m), m.stride(0), m.shape[0], m.shape[1], _lib.ptr(v),
                  _lib.ptr(out), _lib.cur_stream())
        return out.cpu().numpy()
    m = _to_device(matrix, 2)
    v = _to_device(vector, 1)
    _check_inputs(m, v)
    out = torch.empty(m.shape[0], dtype=torch.float64, device=m.device)
    _lib.call("whff_gemv_oracle", _lib.ptr(m), m.stride(0), m.shape[0], m.shape[1], _lib.ptr(v),
              _lib.ptr(out), _lib.cur_stream())
    return out.cpu().numpy()


def _is_f64(x):
    torch = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        return x.dtype == torch.float64
    return np.asarray(x).dtype == np.float64


def _to_device_f64(x, ndim):
    torch = _lib.require_cuda()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=torch.float64)
    else:
        a = np.asarray(x, dtype=np.float64)
        if a.ndim != ndim:
            raise DimensionError(f"expected a {ndim}-D array, got shape {a.shape}")
        t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.contiguous()


def gemv_compressed(stream, vector, policy="mixed", evaluation="exact", row_begin=0,
                    row_end=None, out=None):
    """Fused decompress + GEMV: C(stream) @ vector without materialising C.

    Equivalent to gemv(GemvRequest(decompress(stream), vector, policy)) with
    the blocked reduction order; evaluation="coefficient" applies the block
    transform to the vector instead of the matrix (within the mixed-policy
    bound).  Host stream/vector -> numpy, device -> tensor.
    """
    torch = _lib.require_cuda()
    from .codec import DeviceStream, find_nonfinite
    if policy not in POLICIES:
        raise WhffError(f"unknown precision policy {policy!r}")
    if evaluation not in EVALUATIONS:
        raise WhffError(f"unknown evaluation {evaluation!r}")
    host = not isinstance(stream, DeviceStream)
    ds = DeviceStream.from_host(stream) if host else stream
    try:
        v = _to_device(vector, 1)
        if v.dim() != 1 or v.shape[0] != ds.cols:
            raise DimensionError(
                f"gemv shapes do not agree: matrix ({ds.rows}, {ds.cols}), vector {tuple(v.shape)}")
        bad = find_nonfinite(v)
        if bad is not None:
            raise NonFiniteError("vector", bad)
        y = ds.gemv(v, policy=policy, evaluation=evaluation, row_begin=row_begin,
                    row_end=row_end, out=out)
        return y.cpu().numpy() if host else y
    finally:
        if host:
            ds.close()


def reduction_bits_lost(width):
    """mpgemv.py:72-80."""
    if width < 1:
        raise WhffError(f"reduction width must be >= 1, got {width}")
    return int(math.floor(math.log2(width)))


def relative_error(result, reference):
    """mpgemv.py:83-89."""
    ref = np.asarray(reference, dtype=np.float64)
    res = np.asarray(result, dtype=np.float64)
    denom = np.abs(ref)
    denom[denom == 0] = 1.0
    return np.abs(res - ref) / denom
