"""Dual-quantization front end (mirrors P/quantize.py) -- stage API over K1.

``prequantize`` -> lzb_prequantize; ``construct_grid`` -> K1 lzb_quantize on
the int64 prequant grid (dtype 2) + a chunk-major -> grid scatter, giving the
reference's grid-order QuantGrid and the sorted OutlierList.  The compress
path itself never materialises either: K1 reads the floats and writes the
chunk-major stream directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DataError
from .grid import ChunkSpec, Dims, Field

_PREQUANT_LIMIT = 2 ** 59


@dataclass(frozen=True)
class QuantConfig:
    """P/quantize.py:25-40."""

    eb_abs: float
    cap: int = 1024

    def __post_init__(self) -> None:
        if self.cap < 4 or self.cap & (self.cap - 1):
            raise DataError(f"cap must be a power of two >= 4, got {self.cap}")
        if not (np.isfinite(self.eb_abs) and self.eb_abs > 0):
            raise DataError(f"eb_abs must be positive and finite, got {self.eb_abs}")

    @property
    def radius(self) -> int:
        return self.cap // 2


@dataclass(frozen=True)
class PrequantGrid:
    dims: Dims
    codes: np.ndarray  # flat int64

    def as_3d(self) -> np.ndarray:
        return self.codes.reshape(self.dims.shape3d)


@dataclass(frozen=True)
class QuantGrid:
    dims: Dims
    codes: np.ndarray  # flat uint32, grid order

    def as_3d(self) -> np.ndarray:
        return self.codes.reshape(self.dims.shape3d)


@dataclass(frozen=True)
class OutlierList:
    """P/quantize.py:69-87."""

    indices: np.ndarray
    deltas: np.ndarray

    def __post_init__(self) -> None:
        if len(self.indices) != len(self.deltas):
            raise DataError("outlier index/delta arrays differ in length")
        if len(self.indices) > 1 and not (np.diff(self.indices) > 0).all():
            raise DataError("outlier indices must be strictly increasing")

    def __len__(self) -> int:
        return len(self.indices)

    @classmethod
    def empty(cls) -> "OutlierList":
        return cls(np.empty(0, np.int64), np.empty(0, np.int64))


def prequantize_device(field: Field, cfg: QuantConfig):
    """round-half-away(f64(x) / (2 eb_abs)) on the GPU -> int64 CUDA tensor."""
    import torch

    from .pipeline import _as_device_values

    L = N.lib()
    x = _as_device_values(field)
    out = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    st = N.empty_bytes(N.STATUS_BYTES)
    N.check_rc(L.lzb_prequantize(x.data_ptr(), 0 if x.dtype == torch.float32 else 1, x.numel(),
                                 cfg.eb_abs, out.data_ptr(), st.data_ptr(), N.stream_ptr()),
               "prequantize")
    (s,) = N.read_status(st)
    N.raise_for(s, "prequantize")
    return out


def prequantize(field: Field, cfg: QuantConfig) -> PrequantGrid:
    """round-half-away(f64(x) / (2 eb_abs)) on the GPU (P/quantize.py:95-110)."""
    return PrequantGrid(field.dims, prequantize_device(field, cfg).cpu().numpy())


def quant_grid_device(pre, dims: Dims, cfg: QuantConfig, spec: ChunkSpec):
    """K1 over a device prequant grid -> (grid-order codes as an int32 CUDA tensor,
    cap-bin histogram as numpy int64).  Used by analyze (pairs gathered on device)."""
    import torch

    L = N.lib()
    n = dims.count
    codes = torch.empty(n, dtype=torch.int32, device=pre.device)
    hist = torch.empty(cfg.cap, dtype=torch.int64, device=pre.device)
    g = N.geom(dims.as_tuple(), spec.as_tuple())
    cap_out = n
    outl = torch.empty(2 * max(cap_out, 1), dtype=torch.int64, device=pre.device)
    qs = L.lzb_quantize_scratch_bytes(g, cap_out)
    scr = N.empty_bytes(qs, pre.device)
    st = N.empty_bytes(N.STATUS_BYTES, pre.device)
    N.check_rc(L.lzb_quantize(pre.data_ptr(), 2, g, 0.5, cfg.cap, codes.data_ptr(), 4,
                              hist.data_ptr(), outl.data_ptr(), cap_out, st.data_ptr(),
                              scr.data_ptr(), qs, N.stream_ptr()), "quantize")
    (s,) = N.read_status(st)
    N.raise_for(s, "quantize")
    grid = torch.empty_like(codes)
    N.check_rc(L.lzb_chunk_major(codes.data_ptr(), grid.data_ptr(), 4, g, 1, N.stream_ptr()),
               "chunk_major")
    return grid, hist.cpu().numpy()


def chunk_major(codes, dims: Dims, spec: ChunkSpec, direction: int) -> np.ndarray:
    """gather (0) / scatter (1) between grid order and the chunk-major stream (device)."""
    import torch

    L = N.lib()
    src = torch.from_numpy(np.ascontiguousarray(codes, np.uint32).view(np.int32)).to("cuda")
    dst = torch.empty_like(src)
    g = N.geom(dims.as_tuple(), spec.as_tuple())
    N.check_rc(L.lzb_chunk_major(src.data_ptr(), dst.data_ptr(), 4, g, direction,
                                 N.stream_ptr()), "chunk_major")
    return dst.cpu().numpy().view(np.uint32).copy()


def construct_grid(prequant: PrequantGrid, cfg: QuantConfig, spec: ChunkSpec,
                   threads: int = 1) -> tuple[QuantGrid, OutlierList]:
    """K1 over a prequant grid: grid-order codes + sorted outliers (P/quantize.py:161-193)."""
    import torch

    L = N.lib()
    dims = prequant.dims
    n = dims.count
    x = torch.from_numpy(np.ascontiguousarray(prequant.codes, np.int64)).to("cuda")
    codes = torch.empty(n, dtype=torch.int32, device="cuda")
    hist = torch.empty(cfg.cap, dtype=torch.int64, device="cuda")
    g = N.geom(dims.as_tuple(), spec.as_tuple())
    cap_out = n
    outl = torch.empty(2 * max(cap_out, 1), dtype=torch.int64, device="cuda")
    qs = L.lzb_quantize_scratch_bytes(g, cap_out)
    scr = N.empty_bytes(qs)
    st = N.empty_bytes(N.STATUS_BYTES)
    N.check_rc(L.lzb_quantize(x.data_ptr(), 2, g, 0.5, cfg.cap, codes.data_ptr(), 4,
                              hist.data_ptr(), outl.data_ptr(), cap_out, st.data_ptr(),
                              scr.data_ptr(), qs, N.stream_ptr()), "quantize")
    (s,) = N.read_status(st)
    N.raise_for(s, "quantize")
    k = s.u[0]
    stream = codes.cpu().numpy().view(np.uint32)
    grid = chunk_major(stream, dims, spec, 1)
    rec = outl[: 2 * k].cpu().numpy().reshape(-1, 2)
    return QuantGrid(dims, grid), OutlierList(rec[:, 0].copy(), rec[:, 1].copy())
