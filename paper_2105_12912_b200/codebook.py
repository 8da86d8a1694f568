"""Histogram, canonical Huffman code book, entropy bounds (mirrors P/codebook.py).

``histogram`` and ``Codebook.from_counts`` / ``from_lengths`` run on the GPU
(lzb_histogram, K2 lzb_codebook, lzb_codebook_from_lengths).  The entropy and
redundancy-bound helpers are host arithmetic on a cap-sized histogram (the
reference's own float formulas, kept bit-identical; SURVEY 2 marks them
host-side).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CorruptArchiveError, DataError

MAX_CODE_LEN = 64


def _to_device(a, dtype):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to("cuda").contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype)).to("cuda")


def histogram(codes, cap: int) -> np.ndarray:
    """Symbol counts, int64 of length cap (P/codebook.py:23-27), on the GPU."""
    import torch

    L = N.lib()
    c = _to_device(codes, np.uint32)
    if c.dtype not in (torch.int32, torch.uint32, torch.int16, torch.uint16):
        c = c.to(torch.int32)
    sb = c.element_size()
    h = torch.empty(cap, dtype=torch.int64, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    N.check_rc(L.lzb_histogram(c.data_ptr(), sb, c.numel(), cap, h.data_ptr(), st.data_ptr(),
                               N.stream_ptr()), "histogram")
    (s,) = N.read_status(st)
    if s.code:
        mx = int(c.max().item())
        raise DataError(f"symbol {mx} out of range for cap {cap}")
    return h.cpu().numpy()


def entropy_bits(counts: np.ndarray) -> float:
    total = counts.sum()
    if total == 0:
        raise DataError("entropy of an empty histogram")
    p = counts[counts > 0] / total
    return float(-(p * np.log2(p)).sum()) + 0.0


def dominant_probability(counts: np.ndarray) -> float:
    total = counts.sum()
    if total == 0:
        raise DataError("empty histogram")
    return float(counts.max() / total)


def binary_entropy(p: float) -> float:
    if p <= 0.0 or p >= 1.0:
        return 0.0
    return float(-p * np.log2(p) - (1.0 - p) * np.log2(1.0 - p))


def redundancy_upper(p1: float) -> float:
    return p1 + 0.086


def redundancy_lower(p1: float) -> float:
    return 1.0 - binary_entropy(p1) if p1 > 0.4 else 0.0


@dataclass(frozen=True)
class EntropyReport:
    entropy: float
    p1: float
    r_minus: float
    r_plus: float
    b_lo: float
    b_hi: float
    b_exact: float | None = None


def entropy_report(counts: np.ndarray, book: "Codebook | None" = None) -> EntropyReport:
    """P/codebook.py:81-87."""
    h = entropy_bits(counts)
    p1 = dominant_probability(counts)
    r_minus, r_plus = redundancy_lower(p1), redundancy_upper(p1)
    b_exact = book.average_bits(counts) if book is not None else None
    return EntropyReport(h, p1, r_minus, r_plus, h + r_minus, h + r_plus, b_exact)


@dataclass(frozen=True)
class Codebook:
    """Canonical prefix code: per-symbol lengths (u8) and MSB-first code words (u64)."""

    lengths: np.ndarray
    codes: np.ndarray

    @property
    def cap(self) -> int:
        return len(self.lengths)

    @property
    def max_len(self) -> int:
        return int(self.lengths.max())

    def average_bits(self, counts: np.ndarray) -> float:
        total = counts.sum()
        if total == 0:
            raise DataError("empty histogram")
        return float((counts * self.lengths).sum() / total)

    def serialize_lengths(self) -> bytes:
        return self.lengths.tobytes()

    @classmethod
    def from_counts(cls, counts) -> "Codebook":
        """K2 on the GPU (two-queue Huffman == the reference's heap, P/codebook.py:143-190)."""
        import torch

        counts = np.asarray(counts, np.int64)
        cap = len(counts)
        if cap == 0 or not counts.any():
            raise DataError("cannot build a codebook from an empty histogram")
        L = N.lib()
        h = _to_device(counts, np.int64)
        lens = torch.empty(cap, dtype=torch.uint8, device="cuda")
        words = torch.empty(cap, dtype=torch.int64, device="cuda")
        st = N.empty_bytes(N.STATUS_BYTES)
        ss = L.lzb_codebook_scratch_bytes(cap)
        scr = N.empty_bytes(ss)
        N.check_rc(L.lzb_codebook(h.data_ptr(), cap, lens.data_ptr(), words.data_ptr(),
                                  st.data_ptr(), scr.data_ptr(), ss, N.stream_ptr()), "codebook")
        (s,) = N.read_status(st)
        if s.code:
            raise DataError("histogram too skewed: code length exceeds 64 bits")
        return cls(lens.cpu().numpy(), words.cpu().numpy().view(np.uint64))

    @classmethod
    def from_lengths(cls, raw) -> "Codebook":
        """Validated canonical code from serialized lengths (P/codebook.py:125-140)."""
        import torch

        lengths = np.frombuffer(raw, np.uint8).copy() if isinstance(raw, (bytes, bytearray)) \
            else np.asarray(raw, np.uint8)
        if lengths.max(initial=0) > MAX_CODE_LEN:
            raise CorruptArchiveError("codebook length exceeds 64 bits")
        if not lengths.any():
            raise CorruptArchiveError("codebook has no symbols")
        L = N.lib()
        cap = len(lengths)
        d = _to_device(lengths, np.uint8)
        words = torch.empty(cap, dtype=torch.int64, device="cuda")
        st = N.empty_bytes(N.STATUS_BYTES)
        N.check_rc(L.lzb_codebook_from_lengths(d.data_ptr(), cap, words.data_ptr(),
                                               st.data_ptr(), None, 0, N.stream_ptr()),
                   "codebook_from_lengths")
        (s,) = N.read_status(st)
        if s.code:
            if int((lengths > 0).sum()) == 1:
                raise CorruptArchiveError("single-symbol codebook must use length 1")
            raise CorruptArchiveError("codebook lengths violate Kraft equality")
        return cls(lengths, words.cpu().numpy().view(np.uint64))
