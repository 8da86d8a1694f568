"""Huffman bit streams (mirrors P/huffman.py): encode = K3, decode = K5, both on the GPU."""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .codebook import Codebook, _to_device, histogram
from .errors import CorruptArchiveError, DataError

_HEADER = struct.Struct("<QQ")


@dataclass(frozen=True)
class BitStream:
    """A packed MSB-first bit string with its exact bit and symbol counts (P/huffman.py:20-43)."""

    bit_len: int
    count: int
    data: np.ndarray  # uint8, ceil(bit_len / 8) bytes

    def to_bytes(self) -> bytes:
        return _HEADER.pack(self.bit_len, self.count) + self.data.tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "BitStream":
        if len(raw) < _HEADER.size:
            raise CorruptArchiveError("bit stream shorter than its header")
        bit_len, count = _HEADER.unpack_from(raw)
        nbytes = (bit_len + 7) // 8
        if len(raw) - _HEADER.size < nbytes:
            raise CorruptArchiveError("bit stream data truncated")
        data = np.frombuffer(raw, np.uint8, count=nbytes, offset=_HEADER.size).copy()
        return cls(bit_len, count, data)


def _sym_tensor(codes):
    import torch

    c = _to_device(codes, np.uint32)
    if c.dtype in (torch.int64, torch.uint64):
        c = c.to(torch.int32)
    return c


def encode(codes, book: Codebook) -> BitStream:
    """Concatenate code words MSB first (P/huffman.py:46-61) -- K3 on the GPU."""
    n = len(codes)
    if n == 0:
        return BitStream(0, 0, np.empty(0, np.uint8))
    c = _sym_tensor(codes)
    lens_h = book.lengths.astype(np.int64)
    cap = book.cap
    try:
        hist = histogram(c, cap)  # device histogram sizes the output: sum(c * len)
    except DataError:
        raise DataError("symbol without a code word in the stream") from None
    if (hist[lens_h == 0] > 0).any():
        raise DataError("symbol without a code word in the stream")
    L = N.lib()
    lens = _to_device(book.lengths, np.uint8)
    words = _to_device(book.codes.view(np.int64), np.int64)
    bits = int((hist * lens_h).sum())
    nbytes = (bits + 7) // 8
    out = N.empty_bytes(nbytes)
    st = N.empty_bytes(N.STATUS_BYTES)
    es = L.lzb_huff_encode_scratch_bytes(n)
    scr = N.empty_bytes(es)
    N.check_rc(L.lzb_huff_encode(c.data_ptr(), c.element_size(), n, lens.data_ptr(),
                                 words.data_ptr(), cap, book.max_len, out.data_ptr(), nbytes,
                                 st.data_ptr(),
                                 scr.data_ptr(), es, N.stream_ptr()), "huff_encode")
    (s,) = N.read_status(st)
    if s.code:
        raise DataError("symbol without a code word in the stream")
    return BitStream(s.u[0], n, out[:nbytes].cpu().numpy())


def decode(stream: BitStream, book: Codebook) -> np.ndarray:
    """Recover the symbol sequence (P/huffman.py:109-122) -- K5 on the GPU."""
    import torch

    if stream.count == 0:
        if stream.bit_len != 0:
            raise CorruptArchiveError("bit stream claims bits but no symbols")
        return np.empty(0, np.uint32)
    L = N.lib()
    data = _to_device(np.asarray(stream.data, np.uint8), np.uint8)
    lens = _to_device(book.lengths, np.uint8)
    maxlen = int(book.lengths.max())
    sb = 2 if book.cap <= 65536 else 4  # u16 symbols take the staged warp decoder
    out = torch.empty(stream.count, dtype=torch.int16 if sb == 2 else torch.int32, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    ds = L.lzb_huff_decode_scratch_bytes(stream.bit_len, maxlen, book.cap)
    scr = N.empty_bytes(ds)
    for fn in (L.lzb_huff_decode, L.lzb_huff_decode_robust):
        N.check_rc(fn(data.data_ptr(), stream.bit_len, stream.count, lens.data_ptr(),
                      book.cap, maxlen, out.data_ptr(), sb, st.data_ptr(),
                      scr.data_ptr(), ds, N.stream_ptr()), "huff_decode")
        (s,) = N.read_status(st)
        if s.code != N.LZB_E_RETRY:  # else: a stream the fast decoder cannot resolve
            break
    if s.code:
        raise CorruptArchiveError("bit stream does not decode to its declared symbols")
    if sb == 2:
        return out.cpu().numpy().view(np.uint16).astype(np.uint32)
    return out.cpu().numpy().view(np.uint32)
