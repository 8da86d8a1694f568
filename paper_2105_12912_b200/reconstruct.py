"""Decoder back end (mirrors P/reconstruct.py) -- stage API over K6.

``reconstruct_grid`` gathers the grid-order codes into the chunk-major stream
and runs K6 lzb_reconstruct (fuse + partial sums + the int64 prequant output);
``dequantize`` runs lzb_dequantize.  The decompress path calls K6 directly on
the decoded stream.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .grid import SCALAR_DTYPES, ChunkSpec, Field
from .quantize import OutlierList, PrequantGrid, QuantConfig, QuantGrid, chunk_major


def _records(outliers: OutlierList) -> np.ndarray:
    rec = np.empty(len(outliers), [("i", "<u8"), ("d", "<i8")])
    rec["i"] = outliers.indices
    rec["d"] = outliers.deltas
    return rec.view(np.uint8)


def fuse_outliers(quant: QuantGrid, outliers: OutlierList, cfg: QuantConfig) -> np.ndarray:
    """q' = code - r, q'[idx] += delta (P/reconstruct.py:22-32), on the device."""
    import torch

    d = torch.from_numpy(np.ascontiguousarray(quant.codes, np.uint32).astype(np.int64)).to("cuda")
    d -= cfg.radius
    if len(outliers):
        idx = torch.from_numpy(np.asarray(outliers.indices, np.int64)).to("cuda")
        dl = torch.from_numpy(np.asarray(outliers.deltas, np.int64)).to("cuda")
        d.index_add_(0, idx, dl)
    return d.cpu().numpy()


def reconstruct_grid(quant: QuantGrid, outliers: OutlierList, cfg: QuantConfig, spec: ChunkSpec,
                     threads: int = 1) -> PrequantGrid:
    """Chunk-wise partial-sum reconstruction (P/reconstruct.py:60-76) -- K6."""
    import torch

    L = N.lib()
    dims = quant.dims
    n = dims.count
    stream = chunk_major(quant.codes, dims, spec, 0)
    codes = torch.from_numpy(stream.view(np.int32)).to("cuda")
    rec = torch.from_numpy(_records(outliers)).to("cuda") if len(outliers) else None
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    pre = torch.empty(n, dtype=torch.int64, device="cuda")
    g = N.geom(dims.as_tuple(), spec.as_tuple())
    rs = L.lzb_reconstruct_scratch_bytes(g, len(outliers))
    scr = N.empty_bytes(rs)
    st = N.empty_bytes(N.STATUS_BYTES)
    N.check_rc(L.lzb_reconstruct(codes.data_ptr(), 4, rec.data_ptr() if rec is not None else None,
                                 len(outliers), g, 0.5, cfg.cap, y.data_ptr(), 1, pre.data_ptr(),
                                 st.data_ptr(), scr.data_ptr(), rs, N.stream_ptr()),
               "reconstruct")
    (s,) = N.read_status(st)
    if s.code != N.LZB_E_DATA:  # y is scratch here (eb 0.5); only q matters
        N.raise_for(s, "reconstruct")
    return PrequantGrid(dims, pre.cpu().numpy())


def dequantize(prequant: PrequantGrid, cfg: QuantConfig, dtype) -> Field:
    """dtype(f64(q) * 2 eb_abs), finite check, range (P/reconstruct.py:79-88)."""
    import torch

    dt = SCALAR_DTYPES[dtype] if isinstance(dtype, str) else np.dtype(dtype)
    L = N.lib()
    q = torch.from_numpy(np.ascontiguousarray(prequant.codes, np.int64)).to("cuda")
    f64 = dt == np.float64
    y = torch.empty(q.numel(), dtype=torch.float64 if f64 else torch.float32, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    N.check_rc(L.lzb_dequantize(q.data_ptr(), q.numel(), cfg.eb_abs, y.data_ptr(), int(f64),
                                st.data_ptr(), N.stream_ptr()), "dequantize")
    (s,) = N.read_status(st)
    N.raise_for(s, "dequantize")
    return Field(prequant.dims, y.cpu().numpy(), s.f64(0), s.f64(1))
