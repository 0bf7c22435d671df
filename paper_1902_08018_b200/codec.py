"""Block bit-plane codec, device side.  Mirrors whff.codec (codec.py) so it is a
drop-in: same mode classes, CompressedStream, compress / decompress /
decode_block / codec_metrics / save_stream / load_stream, same errors.

Compression and decompression run on the B200 through libwhff_b200.so:
  * compress       -> whff_compress        (GPU encoder, byte-identical to
                      codec.py:225-293 + _kernels.pyx:139-283)
  * decompress     -> whff_decode          (bit-exact words, codec.py:296-314)
  * decode_block   -> whff_decode_block_words (codec.py:317-332)
The WHFZ file container (save_stream / load_stream, codec.py:388-450) and the
error metrics (codec.py:359-381) are host-side bookkeeping.

`DeviceStream` is the HBM-resident form the fused decode+GEMV consumes.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import CorruptStreamError, DimensionError, NonFiniteError, WhffError

BLOCK = 4
N_PLANES = 27
QUANT_BITS = 26
EMAX_BIAS = 160

MAGIC = b"WHFZ"
VERSION = 1

_MODE_RATE = 0
_MODE_PRECISION = 1
_MODE_ACCURACY = 2

# total-sequency coefficient order inside a 4x4 block, ties by row (codec.py:40)
SEQUENCY = sorted(range(16), key=lambda k: (k // 4 + k % 4, k // 4))


@dataclass(frozen=True)
class FixedRate:
    bpv: int

    def __post_init__(self):
        if not (isinstance(self.bpv, int) and 1 <= self.bpv <= 32):
            raise WhffError(f"fixed-rate bits per value must be in 1..32, got {self.bpv}")


@dataclass(frozen=True)
class FixedPrecision:
    planes: int

    def __post_init__(self):
        if not (isinstance(self.planes, int) and 1 <= self.planes <= 32):
            raise WhffError(f"fixed-precision planes must be in 1..32, got {self.planes}")


@dataclass(frozen=True)
class FixedAccuracy:
    tolerance: float

    def __post_init__(self):
        if not (self.tolerance >= 0.0):
            raise WhffError(f"tolerance must be nonnegative, got {self.tolerance}")


def mode_code(mode):
    if isinstance(mode, FixedRate):
        return _MODE_RATE, float(mode.bpv)
    if isinstance(mode, FixedPrecision):
        return _MODE_PRECISION, float(mode.planes)
    if isinstance(mode, FixedAccuracy):
        return _MODE_ACCURACY, float(mode.tolerance)
    # accept the reference's own mode objects (duck typing on the class name)
    name = type(mode).__name__
    if name == "FixedRate":
        return _MODE_RATE, float(mode.bpv)
    if name == "FixedPrecision":
        return _MODE_PRECISION, float(mode.planes)
    if name == "FixedAccuracy":
        return _MODE_ACCURACY, float(mode.tolerance)
    raise WhffError(f"unknown codec mode {mode!r}")


def mode_from_code(code, param):
    if code == _MODE_RATE:
        return FixedRate(int(param))
    if code == _MODE_PRECISION:
        return FixedPrecision(int(param))
    return FixedAccuracy(float(param))


@dataclass
class CompressedStream:
    """Host form of a stream (codec.py:71-91)."""
    mode: object
    rows: int
    cols: int
    payload: np.ndarray          # uint8
    block_index: np.ndarray      # uint64 bit offsets, one per block
    total_bits: int
    block_size: int = BLOCK
    version: int = VERSION
    exact_bits: bool = True

    @property
    def n_blocks(self):
        return self.block_index.shape[0]

    @property
    def padded_shape(self):
        r = (self.rows + BLOCK - 1) // BLOCK * BLOCK
        c = (self.cols + BLOCK - 1) // BLOCK * BLOCK
        return r, c


@dataclass
class CodecMetrics:
    bits_per_value: float
    ratio: float
    rmse: float
    nrmse: float
    max_pointwise_error: float
    psnr: float

    def as_dict(self):
        return {"bits_per_value": self.bits_per_value, "ratio": self.ratio,
                "rmse": self.rmse, "nrmse": self.nrmse,
                "max_pointwise_error": self.max_pointwise_error, "psnr": self.psnr}


# ---------------------------------------------------------------------------
# device-resident stream
# ---------------------------------------------------------------------------

class DeviceStream:
    """A compressed stream resident in HBM (handle of whff_dstream_t)."""

    def __init__(self, handle, mode, total_bits=None):
        self._h = handle
        info = _lib.DStreamInfo()
        _lib.call("whff_dstream_get_info", handle, ctypes.byref(info))
        self.mode = mode
        self.rows = int(info.rows)
        self.cols = int(info.cols)
        self.n_blocks = int(info.n_blocks)
        self.payload_bytes = int(info.payload_bytes)
        self.index_bytes = int(info.index_bytes)
        self.device_bytes = int(info.device_bytes)
        self.index_kind = _lib.INDEX_KIND[int(info.index_kind)]
        self.planes_limit = int(info.planes_limit)
        self.has_raw_flag = bool(info.has_raw_flag)
        self.layout = _lib.LAYOUT_NAME[int(info.layout)]
        self.total_bits = total_bits if total_bits is not None else int(info.total_bits)
        import torch
        self.device = torch.device("cuda", int(info.device))
        self._refresh()

    def _refresh(self):
        info = _lib.DStreamInfo()
        _lib.call("whff_dstream_get_info", self._h, ctypes.byref(info))
        self.packed = bool(info.packed)
        self.packed_bytes = int(info.packed_bytes)
        self.packed_exceptions = int(info.packed_exceptions)
        self.device_bytes = int(info.device_bytes)

    @property
    def handle(self):
        return self._h

    @property
    def block_rows(self):
        return (self.rows + 3) // 4

    @property
    def block_cols(self):
        return (self.cols + 3) // 4

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().whff_dstream_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- conversions -------------------------------------------------------
    @classmethod
    def from_host(cls, stream, device=None):
        """Upload a CompressedStream (validates like codec.py:347-356)."""
        torch = _lib.require_cuda()
        _validate_stream(stream)
        code, param = mode_code(stream.mode)
        payload = np.ascontiguousarray(stream.payload, dtype=np.uint8)
        index = np.ascontiguousarray(stream.block_index, dtype=np.uint64)
        dev = torch.cuda.current_device() if device is None else int(device)
        h = ctypes.c_void_p()
        _lib.call("whff_dstream_create", dev, code, param, int(stream.rows), int(stream.cols),
                  _lib.ptr(payload), payload.size, _lib.ptr(index), index.size, ctypes.byref(h))
        return cls(h, stream.mode, total_bits=int(stream.total_bits))

    def relayout(self, layout="skeleton-first"):
        """Permute the device payload in place (whff_dstream_relayout): same
        bytes and index, decodes to the same words; to_host() restores the
        reference bytes."""
        _lib.call("whff_dstream_relayout", self._h, _lib.LAYOUT[layout], _lib.cur_stream())
        self.layout = layout
        return self

    def pack(self):
        """Build the tile-packed device copy (whff_dstream_pack; csrc/whff_packed.cuh):
        the decoded coefficients re-coded losslessly as fixed-width fields per
        segment -- decode / gemv / plans then read it (words stay bit-exact)."""
        _lib.call("whff_dstream_pack", self._h, _lib.cur_stream())
        self._refresh()
        return self

    def block_row_bytes(self):
        """Compressed bytes of every block-row (whff_dstream_block_row_bits):
        the weights of the byte-balanced row sharding (executor.shard_units)."""
        out = np.zeros(self.block_rows + 1, dtype=np.uint64)
        _lib.call("whff_dstream_block_row_bits", self._h, _lib.ptr(out))
        return (np.diff(out.astype(np.int64)) + 7) // 8

    def clone(self):
        """A physically distinct HBM copy (whff_dstream_clone)."""
        h = ctypes.c_void_p()
        _lib.call("whff_dstream_clone", self._h, ctypes.byref(h))
        c = DeviceStream(h, self.mode, total_bits=self.total_bits)
        c.layout = self.layout
        return c

    def to_host(self):
        payload = np.empty(self.payload_bytes, dtype=np.uint8)
        index = np.empty(self.n_blocks, dtype=np.uint64)
        _lib.call("whff_dstream_download", self._h, _lib.ptr(payload), _lib.ptr(index))
        return CompressedStream(mode=self.mode, rows=self.rows, cols=self.cols, payload=payload,
                                block_index=index, total_bits=int(self.total_bits))

    # -- streaming (device-layout contents to / from host memory) -----------
    def export(self, pinned=True):
        """(payload, index blob) exactly as held on the device (device layout),
        as (pinned) host uint8 tensors: the staging form of the streaming scan."""
        import torch
        pb, ib = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.call("whff_dstream_export", self._h, None, ctypes.byref(pb), None, ctypes.byref(ib))
        payload = torch.empty(pb.value, dtype=torch.uint8, pin_memory=pinned)
        index = torch.empty(ib.value, dtype=torch.uint8, pin_memory=pinned)
        _lib.call("whff_dstream_export", self._h, _lib.ptr(payload), None, _lib.ptr(index), None)
        return payload, index

    def reserve(self, payload_capacity):
        _lib.call("whff_dstream_reserve", self._h, int(payload_capacity))

    def rebind(self, payload_bytes):
        """Set the payload size alone (for plans built before the bytes arrive)."""
        _lib.call("whff_dstream_rebind", self._h, int(payload_bytes))
        self.payload_bytes = int(payload_bytes)
        self._refresh()

    def import_async(self, payload, index):
        """Rebind to a same-geometry stream's exported contents (async H2D on
        the current stream; the payload size changes at once for new plans)."""
        _lib.call("whff_dstream_import_async", self._h, _lib.ptr(payload), int(payload.numel()),
                  _lib.ptr(index) if index.numel() else None, int(index.numel()), _lib.cur_stream())
        self.payload_bytes = int(payload.numel())
        self._refresh()

    # -- device operations -------------------------------------------------
    def decode(self, out=None, check=True):
        """Bit-exact binary32 words as a (rows, cols) CUDA tensor."""
        torch = _lib.require_cuda()
        if out is None:
            out = torch.empty((self.rows, self.cols), dtype=torch.float32, device=self.device)
        st = _lib.status_word(self.device)
        _lib.call("whff_decode", self._h, _lib.ptr(out), out.stride(0), _lib.ptr(st),
                  _lib.cur_stream())
        if check and _lib.read_status(st) is not None:
            raise CorruptStreamError("decoded array contains non-finite values")
        return out

    def decode_block_words(self, first, count):
        torch = _lib.require_cuda()
        out = torch.empty((count, 4, 4), dtype=torch.float32, device=self.device)
        _lib.call("whff_decode_block_words", self._h, int(first), int(count), _lib.ptr(out),
                  _lib.cur_stream())
        return out

    def decode_blocks(self, first=0, count=None, planes_limit=-1):
        """K:371-408 outputs for a block range, as CUDA tensors."""
        torch = _lib.require_cuda()
        count = self.n_blocks - first if count is None else count
        d = self.device
        mag = torch.empty((count, 16), dtype=torch.int32, device=d)
        neg = torch.empty((count, 16), dtype=torch.uint8, device=d)
        emax = torch.empty((count,), dtype=torch.int16, device=d)
        raw = torch.empty((count,), dtype=torch.uint8, device=d)
        raw_words = torch.empty((count, 16), dtype=torch.int32, device=d)
        consumed = torch.empty((count,), dtype=torch.int64, device=d)
        _lib.call("whff_decode_blocks", self._h, int(first), int(count), int(planes_limit),
                  _lib.ptr(mag), _lib.ptr(neg), _lib.ptr(emax), _lib.ptr(raw),
                  _lib.ptr(raw_words), _lib.ptr(consumed), _lib.cur_stream())
        return mag, neg, emax, raw, raw_words, consumed

    def gemv(self, vector, policy="mixed", evaluation="exact", row_begin=0, row_end=None,
             out=None, status=None, workspace=None):
        """Fused decompress + GEMV (whff_decode_gemv); returns a CUDA tensor."""
        torch = _lib.require_cuda()
        row_end = self.rows if row_end is None else row_end
        if out is None:
            out = torch.empty(row_end - row_begin, dtype=torch.float32, device=self.device)
        ws_bytes = ctypes.c_size_t()
        _lib.call("whff_decode_gemv_workspace_size", self._h, _lib.EVAL[evaluation],
                  ctypes.byref(ws_bytes))
        if workspace is None and ws_bytes.value:
            workspace = torch.empty(ws_bytes.value // 4 + 4, dtype=torch.float32, device=self.device)
        own_status = status is None
        if own_status:
            status = _lib.status_word(self.device)
        _lib.call("whff_decode_gemv", self._h, _lib.ptr(vector), _lib.ptr(out),
                  _lib.POLICY[policy], _lib.EVAL[evaluation], int(row_begin), int(row_end),
                  _lib.ptr(workspace), ws_bytes.value, _lib.ptr(status), _lib.cur_stream())
        if own_status and _lib.read_status(status) is not None:
            raise CorruptStreamError("decoded array contains non-finite values")
        return out


def to_device(stream, device=None, layout="reference"):
    """Upload (if needed) and lay out: "reference" / "skeleton-first" permute
    the WHFZ payload; "packed" adds the tile-packed copy the kernels read."""
    ds = stream if isinstance(stream, DeviceStream) else DeviceStream.from_host(stream, device)
    if layout == "packed":
        return ds.pack()
    if layout != ds.layout:
        ds.relayout(layout)
    return ds


# ---------------------------------------------------------------------------
# public operations (codec.py:225-357)
# ---------------------------------------------------------------------------

def _as_device_matrix(array):
    torch = _lib.require_cuda()
    if isinstance(array, torch.Tensor):
        t = array
        if t.dim() != 2 or t.shape[0] < 1 or t.shape[1] < 1:
            raise DimensionError(f"codec input must be 2D and nonempty, got shape {tuple(t.shape)}")
        t = t.to(device="cuda", dtype=torch.float32)
        if t.stride(1) != 1:
            t = t.contiguous()
        return t
    a = np.asarray(array)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise DimensionError(f"codec input must be 2D and nonempty, got shape {a.shape}")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def find_nonfinite(t):
    """First flat index of a non-finite element of a CUDA float32 tensor, or None."""
    st = _lib.status_word(t.device)
    _lib.call("whff_find_nonfinite", _lib.ptr(t), t.numel(), _lib.ptr(st), _lib.cur_stream())
    return _lib.read_status(st)


def compress_device(array, mode):
    """GPU compress into an HBM-resident DeviceStream (codec.py:225-268)."""
    code, param = mode_code(mode)
    t = _as_device_matrix(array)
    if t.stride(0) != t.shape[1]:
        t = t.contiguous()
    if find_nonfinite(t) is not None:
        raise WhffError("codec input contains non-finite values")
    h = ctypes.c_void_p()
    _lib.call("whff_compress", _lib.ptr(t), t.stride(0), t.shape[0], t.shape[1], code, param,
              _lib.cur_stream(), ctypes.byref(h))
    return DeviceStream(h, mode)


def compress(array, mode, backend=None):
    """codec.py:225-268 on the GPU; returns a host CompressedStream."""
    ds = compress_device(array, mode)
    try:
        return ds.to_host()
    finally:
        ds.close()


def decompress(stream, backend=None):
    """codec.py:296-314: bit-exact decode on the GPU.  Host streams return a
    numpy array (drop-in); DeviceStreams return a CUDA tensor."""
    if isinstance(stream, DeviceStream):
        return stream.decode()
    ds = DeviceStream.from_host(stream)
    try:
        return ds.decode().cpu().numpy()
    finally:
        ds.close()


def decode_block(stream, index, backend=None):
    """codec.py:317-332: one 4x4 block through the block index."""
    _validate_stream(stream) if not isinstance(stream, DeviceStream) else None
    if not (0 <= index < stream.n_blocks):
        raise CorruptStreamError(f"block index {index} out of range")
    if isinstance(stream, DeviceStream):
        return stream.decode_block_words(index, 1)[0]
    ds = DeviceStream.from_host(stream)
    try:
        return ds.decode_block_words(index, 1)[0].cpu().numpy()
    finally:
        ds.close()


def _segment_lengths(stream):
    """codec.py:335-344."""
    nb = stream.n_blocks
    code, param = mode_code(stream.mode)
    if code == _MODE_RATE:
        return np.full(nb, int(param) * 16, dtype=np.uint64)
    ends = np.empty(nb, dtype=np.uint64)
    ends[:-1] = stream.block_index[1:]
    ends[-1] = stream.payload.size * 8
    if (ends < stream.block_index).any():
        raise CorruptStreamError("block index offsets are not nondecreasing")
    return ends - stream.block_index


def _validate_stream(stream):
    """codec.py:347-356."""
    if stream.block_size != BLOCK:
        raise CorruptStreamError(f"unsupported block size {stream.block_size}")
    pr, pc = stream.padded_shape
    nb = (pr // BLOCK) * (pc // BLOCK)
    if stream.block_index.shape[0] != nb:
        raise CorruptStreamError("block index length does not match dimensions")
    if stream.block_index.size and int(stream.block_index.max()) >= max(stream.payload.size * 8, 1):
        raise CorruptStreamError("block index offsets point past the payload")
    _segment_lengths(stream)


def codec_metrics(original, decoded, stream):
    """codec.py:359-381 (host metrics)."""
    original = np.asarray(original, dtype=np.float32)
    decoded = np.asarray(decoded.cpu() if hasattr(decoded, "cpu") else decoded, dtype=np.float32)
    if original.shape != decoded.shape:
        raise DimensionError(f"metric shapes differ: {original.shape} vs {decoded.shape}")
    diff = original.astype(np.float64) - decoded.astype(np.float64)
    rmse = float(np.sqrt(np.mean(diff * diff)))
    vrange = float(original.max() - original.min())
    max_err = float(np.abs(diff).max())
    pr, pc = stream.padded_shape if hasattr(stream, "padded_shape") else (
        stream.block_rows * 4, stream.block_cols * 4)
    bpv = stream.total_bits / (pr * pc)
    ratio = 32.0 / bpv if bpv > 0 else float("inf")
    if rmse == 0.0:
        psnr, nrmse = float("inf"), 0.0
    else:
        nrmse = rmse / vrange if vrange > 0 else float("inf")
        psnr = float(20.0 * np.log10(vrange / (2.0 * rmse))) if vrange > 0 else float("-inf")
    return CodecMetrics(bits_per_value=bpv, ratio=ratio, rmse=rmse, nrmse=nrmse,
                        max_pointwise_error=max_err, psnr=psnr)


# ---------------------------------------------------------------------------
# block-row shards (a rank uploads only its rows)
# ---------------------------------------------------------------------------

def shard_rows(stream, row_begin, row_end):
    """The stream of rows [row_begin, row_end) of `stream`, cut out of its
    payload without decoding.  Blocks are independent and stored row-major
    over (block-row, block-col) (codec.py:157-164), so a block-row range is
    one contiguous bit range; the result is byte-identical to compressing the
    row window itself (tests/test_shard_rows.py).  row_begin must be a
    multiple of 4, row_end a multiple of 4 or the stream's last row."""
    if isinstance(stream, DeviceStream):
        stream = stream.to_host()
    rows, cols = stream.rows, stream.cols
    if not (0 <= row_begin < row_end <= rows):
        raise DimensionError(f"row range [{row_begin}, {row_end}) outside [0, {rows})")
    if row_begin % BLOCK or (row_end % BLOCK and row_end != rows):
        raise DimensionError("shard rows must start (and end, except at the last row) on a "
                             "block-row boundary (multiples of 4)")
    bc = (cols + BLOCK - 1) // BLOCK
    b0 = (row_begin // BLOCK) * bc
    b1 = ((row_end + BLOCK - 1) // BLOCK) * bc
    index = np.asarray(stream.block_index, dtype=np.uint64)
    start = int(index[b0])
    end = int(index[b1]) if b1 < index.size else int(stream.total_bits)
    nbits = end - start
    nbytes = (nbits + 7) // 8
    src = np.asarray(stream.payload, dtype=np.uint8)
    lo = start // 8
    sh = start % 8
    chunk = np.zeros(nbytes + 1, dtype=np.uint16)
    take = src[lo: lo + nbytes + 1]
    chunk[:take.size] = take
    out = ((chunk[:-1] << sh) | (chunk[1:] >> (8 - sh))).astype(np.uint8) if sh else \
        chunk[:-1].astype(np.uint8)
    if nbits % 8:                            # the encoder pads the last byte with zeros
        out[-1] &= np.uint8((0xFF << (8 - nbits % 8)) & 0xFF)
    return CompressedStream(mode=stream.mode, rows=row_end - row_begin, cols=cols, payload=out,
                            block_index=index[b0:b1] - np.uint64(start), total_bits=nbits,
                            block_size=stream.block_size, version=stream.version,
                            exact_bits=stream.exact_bits)


# ---------------------------------------------------------------------------
# WHFZ container (codec.py:388-450)
# ---------------------------------------------------------------------------

def save_stream(path, stream):
    if isinstance(stream, DeviceStream):
        stream = stream.to_host()
    code, param = mode_code(stream.mode)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<H", stream.version))
        if code == _MODE_ACCURACY:
            fh.write(struct.pack("<Bd", code, param))
        else:
            fh.write(struct.pack("<BI", code, int(param)))
        fh.write(struct.pack("<QQBQ", stream.rows, stream.cols, stream.block_size, stream.n_blocks))
        fh.write(np.asarray(stream.block_index, dtype="<u8").tobytes())
        fh.write(np.asarray(stream.payload, dtype=np.uint8).tobytes())


def _read_exact(fh, n, what):
    buf = fh.read(n)
    if len(buf) != n:
        raise CorruptStreamError(f"truncated stream: missing {what}")
    return buf


def load_stream(path):
    with open(path, "rb") as fh:
        magic = _read_exact(fh, 4, "magic")
        if magic != MAGIC:
            raise CorruptStreamError(f"bad stream magic {magic!r}")
        (version,) = struct.unpack("<H", _read_exact(fh, 2, "version"))
        if version != VERSION:
            raise CorruptStreamError(f"unsupported stream version {version}")
        (code,) = struct.unpack("<B", _read_exact(fh, 1, "mode"))
        if code == _MODE_RATE:
            (p,) = struct.unpack("<I", _read_exact(fh, 4, "mode parameter"))
            mode = FixedRate(p)
        elif code == _MODE_PRECISION:
            (p,) = struct.unpack("<I", _read_exact(fh, 4, "mode parameter"))
            mode = FixedPrecision(p)
        elif code == _MODE_ACCURACY:
            (tol,) = struct.unpack("<d", _read_exact(fh, 8, "mode parameter"))
            mode = FixedAccuracy(tol)
        else:
            raise CorruptStreamError(f"unknown mode code {code}")
        rows, cols, block_size, nb = struct.unpack("<QQBQ", _read_exact(fh, 25, "dimensions"))
        block_index = np.frombuffer(_read_exact(fh, nb * 8, "block index"), dtype="<u8").copy()
        payload = np.frombuffer(fh.read(), dtype=np.uint8).copy()
    if isinstance(mode, FixedRate):
        total_bits, exact = nb * mode.bpv * 16, True
        if payload.size * 8 < total_bits:
            raise CorruptStreamError("truncated stream payload")
    else:
        total_bits, exact = payload.size * 8, False
    stream = CompressedStream(mode=mode, rows=rows, cols=cols, payload=payload,
                              block_index=block_index, total_bits=total_bits,
                              block_size=block_size, version=version, exact_bits=exact)
    _validate_stream(stream)
    return stream
