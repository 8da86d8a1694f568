"""ctypes binding of liblzb.so (the sm_100a kernels behind include/lzb.h).

This is the ONLY way the package reaches compute: there is no CPU fallback.
Importing a compute entry point without a CUDA device or without the built
library raises ``RuntimeError`` -- loudly, by design.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import CompressionError, CorruptArchiveError, DataError, QuantOverflowError

_HERE = os.path.dirname(os.path.abspath(__file__))
# LZB_LIB: another build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("LZB_LIB") or os.path.join(_HERE, "_lib", "liblzb.so")

LZB_OK, LZB_E_ARG, LZB_E_DATA, LZB_E_OVERFLOW = 0, 1, 2, 3
LZB_E_CORRUPT, LZB_E_CUDA, LZB_E_ASSERT, LZB_E_CAPACITY = 4, 5, 6, 7
LZB_E_RETRY = 8  # the fast decoder could not resolve the stream: run the robust one
LZB_MAXLEN_DEVICE = 0xFFFFFFFF  # lzb_huff_encode: the code book is still on the device

STATUS_BYTES = 64


class Geom(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_uint64), ("ny", ctypes.c_uint64), ("nz", ctypes.c_uint64),
                ("cx", ctypes.c_uint64), ("cy", ctypes.c_uint64), ("cz", ctypes.c_uint64),
                ("ndim", ctypes.c_int32), ("reserved", ctypes.c_int32)]


# name -> (restype, argtypes); every entry is declared in include/lzb.h
_P, _U64, _I, _U32, _D, _SZ = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                               ctypes.c_double, ctypes.c_size_t)
_GP = ctypes.POINTER(Geom)
SIGNATURES = {
    "lzb_version": (ctypes.c_char_p, []),
    "lzb_strerror": (ctypes.c_char_p, [_I]),
    "lzb_copy_bytes": (_I, [_P, _P, _U64, _P]),
    "lzb_field_range": (_I, [_P, _I, _U64, _P, _P]),
    "lzb_prequantize": (_I, [_P, _I, _U64, _D, _P, _P, _P]),
    "lzb_prequant_verify": (_I, [_D, _U64, _U64, _I, _P, _P]),
    "lzb_quantize_scratch_bytes": (_SZ, [_GP, _U64]),
    "lzb_quantize": (_I, [_P, _I, _GP, _D, _U32, _P, _I, _P, _P, _U64, _P, _P, _SZ, _P]),
    "lzb_quantize_ev": (_I, [_P, _I, _GP, _D, _U32, _P, _I, _P, _P, _U64, _P, _P, _SZ, _P, _P]),
    "lzb_histogram": (_I, [_P, _I, _U64, _U32, _P, _P, _P]),
    "lzb_codebook_scratch_bytes": (_SZ, [_U32]),
    "lzb_codebook": (_I, [_P, _U32, _P, _P, _P, _P, _SZ, _P]),
    "lzb_codebook_from_lengths": (_I, [_P, _U32, _P, _P, _P, _SZ, _P]),
    "lzb_huff_encode_scratch_bytes": (_SZ, [_U64]),
    "lzb_huff_encode": (_I, [_P, _I, _U64, _P, _P, _U32, _U32, _P, _U64, _P, _P, _SZ, _P]),
    "lzb_archive_finalize_huff": (_I, [_P, _U64, _P, _U64, _P, _U32, _P, _P, _P, _P, _P]),
    "lzb_huff_encode_at": (_I, [_P, _I, _U64, _P, _P, _U32, _U32, _U64, _P, _U64, _P, _P, _SZ, _P]),
    "lzb_huff_decode_scratch_bytes": (_SZ, [_U64, _U32, _U32]),
    "lzb_huff_decode": (_I, [_P, _U64, _U64, _P, _U32, _U32, _P, _I, _P, _P, _SZ, _P]),
    "lzb_huff_decode_robust": (_I, [_P, _U64, _U64, _P, _U32, _U32, _P, _I, _P, _P, _SZ, _P]),
    "lzb_huff_decode_at": (_I, [_P, _U64, _U64, _U64, _P, _U32, _U32, _P, _I, _P, _P, _SZ, _P]),
    "lzb_huff_range_scratch_bytes": (_SZ, [_U64, _U32, _U32]),
    "lzb_huff_range_maps": (_I, [_P, _U64, _U64, _U64, _P, _U32, _U32, _P, _P, _P, _SZ, _P]),
    "lzb_huff_range_decode": (_I, [_P, _U64, _U64, _U64, _P, _U32, _U32, _U32, _U32, _U64, _P, _I, _P, _P,
                                   _SZ, _P]),
    "lzb_rle_encode_scratch_bytes": (_SZ, [_U64]),
    "lzb_count_runs": (_I, [_P, _I, _U64, _P, _P]),
    "lzb_rle_encode": (_I, [_P, _I, _U64, _P, _P, _U64, _U64, _P, _P, _SZ, _P]),
    "lzb_rle_decode_scratch_bytes": (_SZ, [_U64]),
    "lzb_rle_decode": (_I, [_P, _P, _U64, _U32, _P, _I, _U64, _P, _P, _SZ, _P]),
    "lzb_reconstruct_scratch_bytes": (_SZ, [_GP, _U64]),
    "lzb_reconstruct": (_I, [_P, _I, _P, _U64, _GP, _D, _U32, _P, _I, _P, _P, _P, _SZ, _P]),
    "lzb_dequantize": (_I, [_P, _U64, _D, _P, _I, _P, _P]),
    "lzb_chunk_major": (_I, [_P, _P, _I, _GP, _I, _P]),
    "lzb_quality_scratch_bytes": (_SZ, [_U64]),
    "lzb_quality": (_I, [_P, _P, _I, _U64, _P, _P, _SZ, _P]),
}
# not in the C header but exported for the RLE sizing path
EXTRA = {"lzb_rle_encode_scratch_bytes_runs": (_SZ, [_U64, _U64])}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblzb.so and declare every entry point (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"liblzb.so not built ({path}); run `python -c 'import __graft_entry__ as g; g.build()'`"
            " -- there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, (res, args) in {**SIGNATURES, **EXTRA}.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2105_12912_b200 requires a CUDA (sm_100a) device; "
                           "there is no CPU fallback")
    return load_library()


def geom(dims, chunk) -> Geom:
    nx, ny, nz, ndim = dims
    cx, cy, cz = chunk
    return Geom(nx, ny, nz, cx, cy, cz, ndim, 0)


def check_rc(rc: int, what: str) -> None:
    if rc != LZB_OK:
        msg = load_library().lzb_strerror(rc).decode()
        raise CompressionError(f"{what}: liblzb returned {rc} ({msg})")


class Status:
    """A host view of one lzb_dstatus block read back from the device."""

    __slots__ = ("code", "detail", "u")

    def __init__(self, raw: np.ndarray | None = None, code: int = 0, detail: int = 0, u=None):
        if raw is not None:
            code = int(raw[:4].view(np.int32)[0])
            detail = int(raw[4:8].view(np.int32)[0])
            u = [int(v) for v in raw[8:56].view(np.uint64)]
        self.code, self.detail, self.u = code, detail, u

    def f64(self, i: int) -> float:
        return float(np.array([self.u[i]], np.uint64).view(np.float64)[0])


_STAGE = {}


def _pinned_stage(n: int):
    """Reusable pinned host buffer for the small host<->device transfers."""
    import torch

    b = _STAGE.get("buf")
    if b is None or b.numel() < n:
        b = torch.empty(max(int(n), 1 << 16), dtype=torch.uint8, pin_memory=True)
        _STAGE["buf"] = b
        _STAGE["off"] = 0
    return b


def small_h2d(dst, data: bytes) -> None:
    """Copy a few host bytes into a device tensor without the DMA queues: an SM
    copy kernel reads them from mapped pinned memory, so the write never waits
    behind a large transfer on a copy engine (a rotating region of the stage
    keeps earlier, still pending copies intact)."""
    import numpy as _np

    n = len(data)
    if n == 0:
        return
    b = _pinned_stage(8192 + n)
    off = max(_STAGE["off"], 4096)  # [0, 4096) belongs to read_status
    if off + n > b.numel():
        off = 4096
    b[off: off + n].numpy()[:] = _np.frombuffer(data, _np.uint8)
    _STAGE["off"] = (off + n + 255) & ~255
    check_rc(lib().lzb_copy_bytes(dst.data_ptr(), b.data_ptr() + off, n, stream_ptr()), "copy")


def read_status(block) -> list[Status]:
    """One device->host read of a (k x 64)-byte status tensor (synchronises).
    Done by an SM copy kernel into mapped pinned memory, not a copy engine, so
    it never waits behind a large transfer in flight on another stream."""
    import torch

    if not block.is_cuda:
        return [Status(r) for r in block.numpy().reshape(-1, STATUS_BYTES)]
    n = block.numel()
    if n > 4096:
        raise ValueError("status block larger than the read-back region")
    h = _pinned_stage(8192)
    check_rc(lib().lzb_copy_bytes(h.data_ptr(), block.data_ptr(), n, stream_ptr()), "copy")
    sync_current_stream()
    rec = np.frombuffer(h.numpy(), _STATUS_DT, n // STATUS_BYTES)
    return [Status(code=c, detail=d, u=u) for c, d, u in
            zip(rec["code"].tolist(), rec["detail"].tolist(), rec["u"].tolist())]


_STATUS_DT = np.dtype([("code", "<i4"), ("detail", "<i4"), ("u", "<u8", (6,)), ("pad", "V8")])


def raise_for(st: Status, stage: str, corrupt_msg: str | None = None) -> None:
    c = st.code
    if c == LZB_OK or c == LZB_E_CAPACITY:
        return
    if c == LZB_E_OVERFLOW:
        if stage == "reconstruct":
            raise QuantOverflowError("prefix-sum magnitude bound exceeded; use a larger error "
                                     "bound or smaller chunks")
        raise QuantOverflowError("prequantized magnitude exceeds the integer range; "
                                 "use a larger error bound")
    if c == LZB_E_ASSERT:
        raise AssertionError("prequantization error-bound invariant violated")
    if c == LZB_E_CORRUPT:
        raise CorruptArchiveError(corrupt_msg or f"{stage}: archive is corrupt")
    if c == LZB_E_DATA:
        if stage in ("reconstruct", "dequantize", "range"):
            raise DataError(f"non-finite value at element offset {st.u[2]}")
        raise DataError(f"{stage}: invalid data")
    raise CompressionError(f"{stage}: device status {c}")


def stream_ptr() -> int:
    """The current CUDA stream of the current device (raw cudaStream_t)."""
    import torch

    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


_SYNC = {}


def sync_current_stream() -> None:
    """Block until the current stream is idle (no torch.cuda.Stream object per call)."""
    import torch

    dev = torch._C._cuda_getDevice()
    raw = torch._C._cuda_getCurrentRawStream(dev)
    s = _SYNC.get((dev, raw))
    if s is None:
        s = _SYNC[(dev, raw)] = torch.cuda.ExternalStream(raw, device=dev) if raw \
            else torch.cuda.default_stream(dev)
    s.synchronize()


def ptr(t) -> int:
    return t.data_ptr() if t is not None else 0


def empty_bytes(n: int, device="cuda"):
    import torch

    return torch.empty(max(int(n), 1), dtype=torch.uint8, device=device)
