"""Run-length codec (mirrors P/rle.py): K4 encode and K7 decode on the GPU."""

from __future__ import annotations

import numpy as np

from . import _native as N
from .codebook import _to_device
from .errors import CorruptArchiveError, DataError

_MAX_RUN = 0xFFFFFFFF  # P/rle.py:14 (module attribute: tests may shrink it)


def run_length_encode(codes) -> tuple[np.ndarray, np.ndarray]:
    """(values, lengths), both u32; runs longer than _MAX_RUN split (P/rle.py:17-35)."""
    import torch

    n = len(codes)
    if n == 0:
        return np.empty(0, np.uint32), np.empty(0, np.uint32)
    L = N.lib()
    c = _to_device(codes, np.uint32)
    if c.dtype in (torch.int64, torch.uint64):
        c = c.to(torch.int32)
    cap_runs = n + n // _MAX_RUN + 1
    vals = torch.empty(cap_runs, dtype=torch.int32, device="cuda")
    lens = torch.empty(cap_runs, dtype=torch.int32, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    rs = L.lzb_rle_encode_scratch_bytes_runs(n, cap_runs)
    scr = N.empty_bytes(rs)
    N.check_rc(L.lzb_rle_encode(c.data_ptr(), c.element_size(), n, vals.data_ptr(),
                                lens.data_ptr(), cap_runs, _MAX_RUN, st.data_ptr(),
                                scr.data_ptr(), rs, N.stream_ptr()), "rle_encode")
    (s,) = N.read_status(st)
    if s.code:
        raise DataError("run-length encode failed")
    r = s.u[0]
    return (vals[:r].cpu().numpy().view(np.uint32).copy(),
            lens[:r].cpu().numpy().view(np.uint32).copy())


def run_length_decode(values, lengths) -> np.ndarray:
    """Expand (values, lengths) (P/rle.py:38-44)."""
    import torch

    values = np.asarray(values, np.uint32)
    lengths = np.asarray(lengths, np.uint32)
    if len(values) != len(lengths):
        raise CorruptArchiveError("run values and lengths differ in count")
    if len(lengths) and not lengths.all():
        raise CorruptArchiveError("zero-length run")
    n = int(lengths.astype(np.int64).sum())
    if n == 0:
        return np.empty(0, np.uint32)
    L = N.lib()
    v = _to_device(values, np.uint32)
    ln = _to_device(lengths, np.uint32)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    rs = L.lzb_rle_decode_scratch_bytes(len(values))
    scr = N.empty_bytes(rs)
    N.check_rc(L.lzb_rle_decode(v.data_ptr(), ln.data_ptr(), len(values), 0xFFFFFFFF,
                                out.data_ptr(), 4, n, st.data_ptr(), scr.data_ptr(), rs,
                                N.stream_ptr()), "rle_decode")
    (s,) = N.read_status(st)
    if s.code:
        raise CorruptArchiveError("run-length decode failed")
    return out.cpu().numpy().view(np.uint32).copy()


def average_bits_rle(lengths: np.ndarray, cap: int) -> float:
    """Cost of the run representation in bits per sample (P/rle.py:47-56)."""
    if len(lengths) == 0:
        raise DataError("no runs")
    value_bits = max(1, (cap - 1).bit_length())
    total = int(np.asarray(lengths).astype(np.int64).sum())
    return len(lengths) * (value_bits + 32) / total
