"""End-to-end compress / decompress and the archive format (mirrors P/pipeline.py).

The archive is the reference's, byte for byte: a 130-byte little-endian header
(``<8sHBB3I3IBdddIBQQ6Q``) and three 8-byte-aligned sections -- code book
(cap x u8 lengths), symbol stream (Huffman bit stream / RLE runs / RLE+VLE)
and outliers ({u64 index, i64 delta} sorted by index) -- P/pipeline.py:26-39,
184-221.

Every element-level stage runs on the GPU through liblzb.so (include/lzb.h):

  compress_device:   K1 lzb_quantize -> K2 lzb_codebook -> [host: section
                     table, workflow rule] -> K3 lzb_huff_encode or K4
                     lzb_rle_encode (+ histogram/K2/K3 on run values), all
                     written in place into one device archive tensor.
  decompress_device: [host: header + section validation] -> K5
                     lzb_huff_decode and/or K7 lzb_rle_decode -> K6
                     lzb_reconstruct -> device Field.

The host does only what the reference does on 130 header bytes: the section
table, validation, and the 1.09-bit workflow rule on two integers.  There is
no CPU fallback: without a CUDA device the compute entry points raise.
"""

from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CorruptArchiveError, DataError
from .grid import SCALAR_DTYPES, ChunkSpec, Dims, Field, dtype_name
from .smoothness import RLE_THRESHOLD_BITS, Workflow, estimate_bits

MAGIC = b"LZEBC\x00\x00\x01"
VERSION = 1
_HEADER = struct.Struct("<8sHBB3I3IBdddIBQQ6Q")  # P/pipeline.py:32
_SECTION_BASE = (_HEADER.size + 7) & ~7  # 136
_DTYPE_CODES = {"f32": 0, "f64": 1}
_DTYPE_NAMES = {0: "f32", 1: "f64"}
_EB_MODES = {"abs": 0, "rel": 1}
_OUTLIER_DT = np.dtype([("index", "<u8"), ("delta", "<i8")])
_WORKFLOW_ALIASES = {"auto": None, "huffman": Workflow.HUFFMAN, "huff": Workflow.HUFFMAN,
                     "rle": Workflow.RLE, "rlevle": Workflow.RLE_VLE}
_MAX_RUN = 0xFFFFFFFF  # P/rle.py:14



@dataclass(frozen=True)
class ArchiveHeader:
    """Decoded archive header (P/pipeline.py:50-73)."""

    dtype: str
    dims: Dims
    chunk: ChunkSpec
    eb_mode: str
    eb_value: float
    vmin: float
    vmax: float
    cap: int
    workflow: Workflow
    count: int
    outlier_count: int
    codebook: tuple[int, int]
    symbols: tuple[int, int]
    outliers: tuple[int, int]

    @property
    def eb_abs(self) -> float:
        if self.eb_mode == "abs":
            return self.eb_value
        return self.eb_value * (self.vmax - self.vmin)


@dataclass(frozen=True)
class QualityStats:
    """Size and distortion metrics (P/pipeline.py:76-89)."""

    compression_ratio: float
    max_abs_err: float
    rmse: float
    psnr: float

    def as_line(self) -> str:
        return (f"cr={self.compression_ratio:.6g} max_abs_err={self.max_abs_err:.6g} "
                f"rmse={self.rmse:.6g} psnr={self.psnr:.6g}")


def resolve_workflow(workflow) -> Workflow | None:
    """P/pipeline.py:92-99."""
    if workflow is None or isinstance(workflow, Workflow):
        return workflow
    try:
        return _WORKFLOW_ALIASES[workflow.lower()]
    except KeyError:
        raise DataError(f"unknown workflow {workflow!r}") from None


def _resolve_eb(mode: str, value: float, vmin: float, vmax: float) -> float:
    """P/pipeline.py:120-132."""
    if mode not in _EB_MODES:
        raise DataError(f"eb mode must be 'abs' or 'rel', got {mode!r}")
    if not (np.isfinite(value) and value > 0):
        raise DataError(f"error bound must be positive and finite, got {value}")
    if mode == "abs":
        return value
    if vmax <= vmin:
        raise DataError("relative error bound needs a nonzero value range; "
                        "use an absolute bound for constant fields")
    return value * (vmax - vmin)


def _check_cfg(eb_abs: float, cap: int) -> None:
    """QuantConfig validation (P/quantize.py:25-40)."""
    if cap < 4 or cap & (cap - 1):
        raise DataError(f"cap must be a power of two >= 4, got {cap}")
    if not (np.isfinite(eb_abs) and eb_abs > 0):
        raise DataError(f"eb_abs must be positive and finite, got {eb_abs}")


def _a8(v: int) -> int:
    return (v + 7) & ~7


def code_bytes_for(cap: int) -> int:
    return 2 if cap <= 65536 else 4


# ---------------------------------------------------------------------------
# device buffers
# ---------------------------------------------------------------------------
class _Pool:
    """Per-process cache of device work buffers, grown on demand (the torch
    caching allocator would also do; this keeps repeated calls allocation
    free and makes the buffer sizes explicit)."""

    def __init__(self):
        self.bufs = {}
        self.gen = 0  # bumped whenever a buffer is (re)allocated: invalidates cached launch plans

    def get(self, name: str, nbytes: int, device):
        import torch

        nbytes = max(int(nbytes), 1)
        t = self.bufs.get((name, str(device)))
        if t is None or t.numel() < nbytes:
            self.bufs[(name, str(device))] = None
            t = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self.bufs[(name, str(device))] = t
            self.gen += 1
        return t


_pool = _Pool()


def _dev(t):
    return t.data_ptr()


_NVTX = bool(os.environ.get("LZB_NVTX"))  # named ranges per stage for nsys / ncu --nvtx


class _Stage:
    """CUDA-event bracket around one stage when profiling (bench.py), and an
    NVTX range when LZB_NVTX is set; no-op otherwise."""

    __slots__ = ("prof", "name", "ev")

    def __init__(self, prof, name):
        self.prof, self.name, self.ev = prof, name, None

    def __enter__(self):
        if self.prof is not None or _NVTX:
            import torch

            if _NVTX:
                torch.cuda.nvtx.range_push(f"lzb.{self.name}")
            if self.prof is not None:
                self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                self.ev[0].record()
        return self

    def __exit__(self, *exc):
        if self.prof is not None and exc[0] is None:
            self.ev[1].record()
            self.prof.append((self.name, self.ev[0], self.ev[1]))
        if _NVTX:
            import torch

            torch.cuda.nvtx.range_pop()
        return False


@dataclass
class DeviceArchive:
    """An archive resident in device memory plus its decoded header."""

    data: object  # torch.uint8 CUDA tensor, exactly `nbytes` long view
    header: ArchiveHeader
    nbytes: int
    # Huffman stream facts known at compress time (bit length, symbols, max
    # code length): decompress_device(DeviceArchive) then needs no host reads
    stream: tuple | None = None

    def to_bytes(self) -> bytes:
        return self.data[: self.nbytes].cpu().numpy().tobytes()


def _as_device_values(field: Field):
    import torch

    if field.on_device:
        v = field.values
        if not v.is_contiguous():
            v = v.contiguous()
        return v.reshape(-1)
    host = np.ascontiguousarray(field.values).reshape(-1)
    return torch.from_numpy(host).to("cuda")


# Fields up to this many elements take the single-sync path: its archive
# buffer is sized for the worst case (32-bit code words), ~4 bytes/element.
_SINGLE_SYNC_MAX = 1 << 25


def compress_device(field: Field, eb: float, eb_mode: str = "rel", cap: int = 1024,
                    workflow=None, chunk: ChunkSpec | None = None, select_mode: str = "exact",
                    threads: int = 1, values=None, prof=None) -> DeviceArchive:
    """Compress to a device-resident archive (the timed region of bench.py).

    Same arguments and archive bytes as ``compress``; ``threads`` is accepted
    for API parity and ignored (the GPU is the thread pool).

    Small Huffman-candidate fields run K1 -> K2 -> K3 -> archive assembly as
    one launch sequence with a single status read at the end (no
    mid-pipeline read-back, so the GPU never idles on the host); when that
    read shows the field needs something else (RLE selection, a code word
    over 32 bits, outlier capacity) the staged path below re-runs it.
    """
    eb_abs = _resolve_eb(eb_mode, eb, field.vmin, field.vmax)
    _check_cfg(eb_abs, cap)
    chunk = chunk or ChunkSpec.default_for(field.dims.ndim)
    n = field.dims.count
    chosen = resolve_workflow(workflow)
    if (0 < n <= _SINGLE_SYNC_MAX and cap <= 4096 and code_bytes_for(cap) == 2 and select_mode == "exact"
            and chosen in (None, Workflow.HUFFMAN)):
        arc = _compress_single_sync(field, eb, eb_mode, eb_abs, cap, chosen, chunk, values, prof)
        if arc is not None:
            return arc
    return _compress_staged(field, eb, eb_mode, eb_abs, cap, workflow, chunk, select_mode, values, prof)


class _SSPlan:
    """Buffers and sizes of one single-sync compress shape, valid while the
    pool generation is unchanged (small fields: the Python setup is a
    measurable part of a call)."""

    __slots__ = ("gen", "g", "codes", "hist", "lengths", "cwords", "st", "cb_scr", "cap_out", "outl", "qs",
                 "q_scr", "sym_off", "worst", "big", "es", "e_scr")


_SS_PLANS: dict = {}


def _ss_plan(dims: Dims, chunk: ChunkSpec, cap: int, dev) -> _SSPlan:
    sdev = str(dev)
    key = (dims.as_tuple(), chunk.as_tuple(), cap, sdev, _pool.bufs.get(("outcap", sdev), 0))
    pl = _SS_PLANS.get(key)
    if pl is not None and pl.gen == _pool.gen:
        return pl
    L = N.lib()
    n = dims.count
    pl = _SSPlan()
    pl.g = N.geom(dims.as_tuple(), chunk.as_tuple())
    pl.codes = _pool.get("codes", n * 2, dev)
    pl.hist = _pool.get("hist", cap * 8, dev)
    pl.lengths = _pool.get("lengths", cap, dev)
    pl.cwords = _pool.get("cwords", cap * 8, dev)
    pl.st = _pool.get("status", 8 * N.STATUS_BYTES, dev)
    pl.cb_scr = _pool.get("cb_scratch", L.lzb_codebook_scratch_bytes(cap), dev)
    pl.cap_out = int(_pool.bufs.get(("outcap", sdev), 0) or min(n, n // 128 + 4096))
    pl.outl = _pool.get("outliers", pl.cap_out * 16, dev)
    pl.qs = L.lzb_quantize_scratch_bytes(pl.g, pl.cap_out)
    pl.q_scr = _pool.get("q_scratch", pl.qs, dev)
    pl.sym_off = _a8(_SECTION_BASE + cap)
    pl.worst = pl.sym_off + 16 + 4 * n + 8 + 16 * pl.cap_out  # code words <= 32 bits on this path
    pl.big = _pool.get("arc_stage", pl.worst, dev)
    pl.es = L.lzb_huff_encode_scratch_bytes(n)
    pl.e_scr = _pool.get("e_scratch", pl.es, dev)
    pl.gen = _pool.gen
    _SS_PLANS[key] = pl
    return pl


_SIDE: dict = {}


def _side_stream(dev):
    """(second stream, histogram-final event, code-book-done event) per device:
    K2 runs beside K1's outlier compaction / ordering launches."""
    import torch

    key = str(dev)
    v = _SIDE.get(key)
    if v is None:
        side = torch.cuda.Stream(device=dev)
        ev_hist, ev_book = torch.cuda.Event(), torch.cuda.Event()
        ev_hist.record()  # create the handles (torch events are created lazily)
        ev_book.record()
        v = _SIDE[key] = (side, ev_hist, ev_book)
    return v


def _compress_single_sync(field: Field, eb, eb_mode, eb_abs, cap, chosen, chunk, values, prof):
    """K1, K2, K3 and lzb_archive_finalize_huff back to back; one read-back.
    Returns None when the staged path must run instead."""
    dims = field.dims
    n = dims.count
    dt = dtype_name(field.values)
    x = values if values is not None else _as_device_values(field)
    dev = x.device
    L = N.lib()
    sp = N.stream_ptr()
    pl = _ss_plan(dims, chunk, cap, dev)
    g, codes, hist, lengths, cwords, st = pl.g, pl.codes, pl.hist, pl.lengths, pl.cwords, pl.st
    stp = _dev(st)
    cb_scr, cap_out, outl, qs, q_scr = pl.cb_scr, pl.cap_out, pl.outl, pl.qs, pl.q_scr
    sym_off, worst, big, es, e_scr = pl.sym_off, pl.worst, pl.big, pl.es, pl.e_scr
    if prof is None:  # K2 on a second stream as soon as the histogram is final
        import torch

        side, ev_hist, ev_book = _side_stream(dev)
        N.check_rc(L.lzb_quantize_ev(_dev(x), _DTYPE_CODES[dt], g, eb_abs, cap, _dev(codes), 2, _dev(hist),
                                     _dev(outl), cap_out, stp, _dev(q_scr), qs, sp, ev_hist.cuda_event),
                   "quantize")
        side.wait_event(ev_hist)
        N.check_rc(L.lzb_codebook(_dev(hist), cap, _dev(lengths), _dev(cwords), stp + N.STATUS_BYTES,
                                  _dev(cb_scr), cb_scr.numel(), side.cuda_stream), "codebook")
        ev_book.record(side)
        torch.cuda.current_stream(dev).wait_event(ev_book)
    else:  # stage timing: one stream
        with _Stage(prof, "K1_quantize"):
            N.check_rc(L.lzb_quantize(_dev(x), _DTYPE_CODES[dt], g, eb_abs, cap, _dev(codes), 2, _dev(hist),
                                      _dev(outl), cap_out, stp, _dev(q_scr), qs, sp), "quantize")
        with _Stage(prof, "K2_codebook"):
            N.check_rc(L.lzb_codebook(_dev(hist), cap, _dev(lengths), _dev(cwords), stp + N.STATUS_BYTES,
                                      _dev(cb_scr), cb_scr.numel(), sp), "codebook")
    with _Stage(prof, "K3_huff_encode"):
        N.check_rc(L.lzb_huff_encode(_dev(codes), 2, n, _dev(lengths), _dev(cwords), cap, N.LZB_MAXLEN_DEVICE,
                                     _dev(big) + sym_off + 16, worst - sym_off - 16, stp + 2 * N.STATUS_BYTES,
                                     _dev(e_scr), es, sp), "huff_encode")
    hdr = _HEADER.pack(MAGIC, VERSION, _DTYPE_CODES[dt], dims.ndim, dims.nx, dims.ny, dims.nz,
                       chunk.cx, chunk.cy, chunk.cz, _EB_MODES[eb_mode], eb, field.vmin, field.vmax, cap,
                       int(Workflow.HUFFMAN), n, 0, _SECTION_BASE, cap, sym_off, 0, 0, 0)
    with _Stage(prof, "assemble"):
        N.check_rc(L.lzb_archive_finalize_huff(_dev(big), worst, hdr, sym_off, _dev(lengths), cap, stp,
                                               stp + N.STATUS_BYTES, _dev(outl), stp + 6 * N.STATUS_BYTES, sp),
                   "finalize")
    sq, sb, se, _, _, _, sf, _ = N.read_status(st[: 8 * N.STATUS_BYTES])  # the one sync
    if sq.code == N.LZB_E_CAPACITY:
        _pool.bufs[("outcap", str(dev))] = sq.u[0] + 1024
        return None
    N.raise_for(sq, "quantize")
    N.raise_for(sb, "codebook")
    if chosen is None and float(np.float64(sb.u[0]) / np.float64(sb.u[1])) <= RLE_THRESHOLD_BITS:
        return None  # P/codebook.py:110-115 + P/smoothness.py:111-136 select RLE+VLE
    if se.code == N.LZB_E_RETRY or sf.code == N.LZB_E_CAPACITY:
        return None  # a code word over 32 bits
    N.raise_for(se, "encode")
    N.raise_for(sf, "finalize")
    bits, n_out, total = sb.u[0], sq.u[0], sf.u[0]
    arc = _new_archive(total, dev)
    arc.copy_(big[:total])
    header = ArchiveHeader(dt, dims, chunk, eb_mode, eb, field.vmin, field.vmax, cap, Workflow.HUFFMAN, n,
                           n_out, (_SECTION_BASE, cap), (sym_off, 16 + (bits + 7) // 8),
                           (sf.u[1], 16 * n_out))
    return DeviceArchive(arc, header, total, (bits, n, int(sb.u[2])))


def _compress_staged(field: Field, eb, eb_mode, eb_abs, cap, workflow, chunk, select_mode, values, prof):
    """K1 + K2, one read-back, then the workflow's encoder sized from it."""
    dims = field.dims
    n = dims.count
    dt = dtype_name(field.values)
    x = values if values is not None else _as_device_values(field)
    dev = x.device
    L = N.lib()
    sp = N.stream_ptr()
    cb = code_bytes_for(cap)
    g = N.geom(dims.as_tuple(), chunk.as_tuple())

    codes = _pool.get("codes", n * cb, dev)
    hist = _pool.get("hist", cap * 8, dev)
    lengths = _pool.get("lengths", cap, dev)
    cwords = _pool.get("cwords", cap * 8, dev)
    st = _pool.get("status", 8 * N.STATUS_BYTES, dev)
    stp = _dev(st)
    cb_scr = _pool.get("cb_scratch", L.lzb_codebook_scratch_bytes(cap), dev)

    cap_out = int(_pool.bufs.get(("outcap", str(dev)), 0) or min(n, n // 128 + 4096))
    while True:
        outl = _pool.get("outliers", cap_out * 16, dev)
        qs = L.lzb_quantize_scratch_bytes(g, cap_out)
        q_scr = _pool.get("q_scratch", qs, dev)
        with _Stage(prof, "K1_quantize"):
            N.check_rc(L.lzb_quantize(_dev(x), _DTYPE_CODES[dt], g, eb_abs, cap, _dev(codes), cb,
                                      _dev(hist), _dev(outl), cap_out, stp, _dev(q_scr), qs, sp),
                       "quantize")
        with _Stage(prof, "K2_codebook"):
            N.check_rc(L.lzb_codebook(_dev(hist), cap, _dev(lengths), _dev(cwords),
                                      stp + N.STATUS_BYTES, _dev(cb_scr), cb_scr.numel(), sp),
                       "codebook")
        sq, sb = N.read_status(st[: 2 * N.STATUS_BYTES])  # sync 1
        if sq.code == N.LZB_E_CAPACITY:
            cap_out = sq.u[0] + 1024
            _pool.bufs[("outcap", str(dev))] = cap_out
            continue
        N.raise_for(sq, "quantize")
        break
    n_out = sq.u[0]

    chosen = resolve_workflow(workflow)
    if chosen is None:
        if select_mode == "exact":
            if sb.code:
                N.raise_for(sb, "codebook")
            b = float(np.float64(sb.u[0]) / np.float64(sb.u[1]))  # P/codebook.py:110-115
        elif select_mode == "estimate":
            counts = hist[: cap * 8].cpu().numpy().view(np.int64)
            b = estimate_bits(counts)
        else:
            raise DataError(f"unknown selection mode {select_mode!r}")
        chosen = Workflow.RLE_VLE if b <= RLE_THRESHOLD_BITS else Workflow.HUFFMAN

    pads = []  # byte ranges to zero (alignment padding)
    if chosen is Workflow.HUFFMAN:
        if sb.code:
            N.raise_for(sb, "codebook")
        bits = sb.u[0]
        nbytes = (bits + 7) // 8
        cb_len, sym_len = cap, 16 + nbytes
        cb_off = _SECTION_BASE
        sym_off = _a8(cb_off + cb_len)
        out_off = _a8(sym_off + sym_len)
        total = out_off + 16 * n_out
        arc = _new_archive(total, dev)
        pads += [(cb_off + cb_len, sym_off), (sym_off + sym_len, out_off)]
        arc[cb_off: cb_off + cap].copy_(lengths[:cap])
        _h2d(arc, sym_off, struct.pack("<QQ", bits, n))
        es = L.lzb_huff_encode_scratch_bytes(n)
        e_scr = _pool.get("e_scratch", es, dev)
        with _Stage(prof, "K3_huff_encode"):
            N.check_rc(L.lzb_huff_encode(_dev(codes), cb, n, _dev(lengths), _dev(cwords), cap,
                                         sb.u[2], _dev(arc) + sym_off + 16, nbytes,
                                         stp + 2 * N.STATUS_BYTES, _dev(e_scr), es, sp),
                       "huff_encode")
        check_slots = [2]
    else:
        N.check_rc(L.lzb_count_runs(_dev(codes), cb, n, stp + 3 * N.STATUS_BYTES, sp), "count_runs")
        (sc,) = N.read_status(st[3 * N.STATUS_BYTES: 4 * N.STATUS_BYTES])
        N.raise_for(sc, "count_runs")
        runs = sc.u[0]
        extra = n // _MAX_RUN + 1 if n > _MAX_RUN else 0
        cap_runs = runs + extra
        vals = _pool.get("rle_vals", cap_runs * 4, dev)
        lens = _pool.get("rle_lens", cap_runs * 4, dev)
        rs = L.lzb_rle_encode_scratch_bytes_runs(n, cap_runs)
        r_scr = _pool.get("r_scratch", rs, dev)
        N.check_rc(L.lzb_rle_encode(_dev(codes), cb, n, _dev(vals), _dev(lens), cap_runs, _MAX_RUN,
                                    stp + 3 * N.STATUS_BYTES, _dev(r_scr), rs, sp), "rle_encode")
        if extra:
            (sr,) = N.read_status(st[3 * N.STATUS_BYTES: 4 * N.STATUS_BYTES])
            N.raise_for(sr, "rle_encode")
            R = sr.u[0]
        else:
            R = runs
        if chosen is Workflow.RLE:
            cb_len, sym_len = 0, 8 + 8 * R
            cb_off = _SECTION_BASE
            sym_off = _a8(cb_off)
            out_off = _a8(sym_off + sym_len)
            total = out_off + 16 * n_out
            arc = _new_archive(total, dev)
            pads += [(sym_off + sym_len, out_off)]
            _h2d(arc, sym_off, struct.pack("<Q", R))
            arc[sym_off + 8: sym_off + 8 + 4 * R].copy_(vals[: 4 * R])
            arc[sym_off + 8 + 4 * R: sym_off + 8 + 8 * R].copy_(lens[: 4 * R])
            check_slots = [3]
        else:
            vh = _pool.get("vhist", cap * 8, dev)
            N.check_rc(L.lzb_histogram(_dev(vals), 4, R, cap, _dev(vh), stp + 4 * N.STATUS_BYTES,
                                       sp), "histogram")
            N.check_rc(L.lzb_codebook(_dev(vh), cap, _dev(lengths), _dev(cwords),
                                      stp + 5 * N.STATUS_BYTES, _dev(cb_scr), cb_scr.numel(), sp),
                       "codebook")
            sr, sh, sv = N.read_status(st[3 * N.STATUS_BYTES: 6 * N.STATUS_BYTES])  # sync 2
            N.raise_for(sr, "rle_encode")
            N.raise_for(sh, "histogram")
            N.raise_for(sv, "codebook")
            bits = sv.u[0]
            nbytes = (bits + 7) // 8
            sub = 16 + nbytes
            cb_len, sym_len = cap, 8 + sub + 4 * R
            cb_off = _SECTION_BASE
            sym_off = _a8(cb_off + cb_len)
            out_off = _a8(sym_off + sym_len)
            total = out_off + 16 * n_out
            arc = _new_archive(total, dev)
            pads += [(cb_off + cb_len, sym_off), (sym_off + sym_len, out_off)]
            arc[cb_off: cb_off + cap].copy_(lengths[:cap])
            _h2d(arc, sym_off, struct.pack("<QQQ", R, bits, R))
            es = L.lzb_huff_encode_scratch_bytes(R)
            e_scr = _pool.get("e_scratch", es, dev)
            N.check_rc(L.lzb_huff_encode(_dev(vals), 4, R, _dev(lengths), _dev(cwords), cap,
                                         sv.u[2], _dev(arc) + sym_off + 24, nbytes,
                                         stp + 2 * N.STATUS_BYTES, _dev(e_scr), es, sp),
                       "huff_encode")
            lo = sym_off + 8 + sub
            arc[lo: lo + 4 * R].copy_(lens[: 4 * R])
            check_slots = [2]

    hdr_bytes = _HEADER.pack(
        MAGIC, VERSION, _DTYPE_CODES[dt], dims.ndim, dims.nx, dims.ny, dims.nz,
        chunk.cx, chunk.cy, chunk.cz, _EB_MODES[eb_mode], eb, field.vmin, field.vmax, cap,
        int(chosen), n, n_out, cb_off, cb_len, sym_off, sym_len, out_off, 16 * n_out)
    _h2d(arc, 0, hdr_bytes + bytes(_SECTION_BASE - len(hdr_bytes)))
    for a, b in pads:
        if b > a:
            arc[a:b].zero_()
    with _Stage(prof, "assemble"):
        if n_out:
            arc[out_off: out_off + 16 * n_out].copy_(outl[: 16 * n_out])
    final = N.read_status(st[: 8 * N.STATUS_BYTES])  # sync: encode status
    for k in check_slots:
        N.raise_for(final[k], "encode")
    header = ArchiveHeader(dt, dims, chunk, eb_mode, eb, field.vmin, field.vmax, cap, chosen, n,
                           n_out, (cb_off, cb_len), (sym_off, sym_len), (out_off, 16 * n_out))
    stream = (bits, n, int(sb.u[2])) if chosen is Workflow.HUFFMAN else None
    return DeviceArchive(arc[:total], header, total, stream)


def _new_archive(total: int, dev):
    """Fresh tensor per archive (the caching allocator recycles the memory), so a
    returned DeviceArchive is never overwritten by a later call."""
    import torch

    return torch.empty(total, dtype=torch.uint8, device=dev)


def _h2d(arc, off: int, data: bytes) -> None:
    N.small_h2d(arc[off: off + len(data)], data)


def compress(field: Field, eb: float, eb_mode: str = "rel", cap: int = 1024, workflow=None,
             chunk: ChunkSpec | None = None, select_mode: str = "exact", threads: int = 1) -> bytes:
    """Compress a field into archive bytes (P/pipeline.py:135-221)."""
    return compress_device(field, eb, eb_mode, cap, workflow, chunk, select_mode,
                           threads).to_bytes()


def parse_header(raw, total: int | None = None) -> ArchiveHeader:
    """Validate and decode an archive header + section table (P/pipeline.py:224-272).

    ``raw`` is ``bytes`` or a device uint8 tensor (only 130 bytes are read back);
    ``total`` overrides the archive length when ``raw`` is only a prefix.
    """
    if not isinstance(raw, (bytes, bytearray, memoryview)):
        total = raw.numel() if total is None else total
        raw = raw[: min(raw.numel(), _HEADER.size)].cpu().numpy().tobytes()
    elif total is None:
        total = len(raw)
    if len(raw) < _HEADER.size:
        raise CorruptArchiveError("archive shorter than its header")
    (magic, version, dtype_code, ndim, nx, ny, nz, cx, cy, cz, eb_code, eb_value, vmin, vmax,
     cap, wf_code, count, outlier_count, cb_off, cb_len, sym_off, sym_len, out_off,
     out_len) = _HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise CorruptArchiveError("bad magic")
    if version != VERSION:
        raise CorruptArchiveError(f"unsupported version {version}")
    if dtype_code not in _DTYPE_NAMES:
        raise CorruptArchiveError(f"unknown dtype code {dtype_code}")
    try:
        workflow = Workflow(wf_code)
        dims = Dims(nx, ny, nz, ndim=ndim)
        chunk = ChunkSpec(cx, cy, cz)
    except (ValueError, DataError) as exc:
        raise CorruptArchiveError(f"invalid header field: {exc}") from exc
    if count != dims.count:
        raise CorruptArchiveError("element count disagrees with dims")
    if cap < 4 or cap & (cap - 1):
        raise CorruptArchiveError(f"invalid cap {cap}")
    eb_mode = "abs" if eb_code == 0 else "rel" if eb_code == 1 else None
    if eb_mode is None:
        raise CorruptArchiveError(f"unknown eb mode {eb_code}")
    if not (np.isfinite(eb_value) and eb_value > 0):
        raise CorruptArchiveError("invalid error bound")
    if eb_mode == "rel" and not vmax > vmin:
        raise CorruptArchiveError("relative bound with degenerate value range")
    prev_end = _SECTION_BASE
    for off, length in ((cb_off, cb_len), (sym_off, sym_len), (out_off, out_len)):
        if off % 8 or off < prev_end or off + length > total:
            raise CorruptArchiveError("section table out of bounds or overlapping")
        prev_end = off + length
    if cb_len != (0 if workflow is Workflow.RLE else cap):
        raise CorruptArchiveError("codebook section size mismatch")
    if out_len != outlier_count * _OUTLIER_DT.itemsize:
        raise CorruptArchiveError("outlier section size mismatch")
    return ArchiveHeader(_DTYPE_NAMES[dtype_code], dims, chunk, eb_mode, eb_value, vmin, vmax,
                         cap, workflow, count, outlier_count, (cb_off, cb_len),
                         (sym_off, sym_len), (out_off, out_len))


def _validate_lengths_host(cb: np.ndarray) -> int:
    """Header-level code book checks before the device decode (P/codebook.py:125-140).
    Returns the max code length (the K5 launch geometry needs it)."""
    mx = int(cb.max()) if cb.size else 0
    if mx > 64:
        raise CorruptArchiveError("codebook length exceeds 64 bits")
    if mx == 0:
        raise CorruptArchiveError("codebook has no symbols")
    return mx


def decompress_device(arc, raw_host: bytes | None = None, prof=None, out=None):
    """Decode a device archive tensor; returns (values CUDA tensor, header, vmin, vmax).

    ``raw_host`` (optional) is the same archive on the host, used for the
    small header-level reads; without it ~100 bytes + the code book are read
    back from the device.  ``arc`` may also be the DeviceArchive returned by
    compress_device: its header and Huffman stream facts are already on the
    host, so nothing is read back before the decode.
    """
    import torch

    known = None
    if isinstance(arc, DeviceArchive):  # header (and stream facts) already on the host
        hdr, known, arc = arc.header, arc.stream, arc.data[: arc.nbytes]
    else:
        hdr = parse_header(raw_host if raw_host is not None else arc, total=arc.numel())

    def host_bytes(a: int, b: int) -> bytes:
        if raw_host is not None and b <= len(raw_host):
            return bytes(raw_host[a:b])
        return arc[a:b].cpu().numpy().tobytes()

    dims, chunk, cap = hdr.dims, hdr.chunk, hdr.cap
    n = hdr.count
    cb = code_bytes_for(cap)
    L = N.lib()
    sp = N.stream_ptr()
    dev = arc.device
    st = _pool.get("dstatus", 4 * N.STATUS_BYTES, dev)
    stp = _dev(st)
    st.zero_()
    base = _dev(arc)
    sym_off, sym_len = hdr.symbols
    huff = None  # (bits ptr, bit_len, count, maxlen) of the Huffman stream, if any
    vals_rle = None
    if hdr.workflow is Workflow.HUFFMAN:
        if known is not None:  # written by compress_device: no host round trip
            bit_len, count, maxlen = known
        else:
            cbytes = np.frombuffer(host_bytes(hdr.codebook[0], sum(hdr.codebook)), np.uint8)
            maxlen = _validate_lengths_host(cbytes)
            head = host_bytes(sym_off, sym_off + min(16, sym_len))
            if len(head) < 16:
                raise CorruptArchiveError("bit stream shorter than its header")
            bit_len, count = struct.unpack_from("<QQ", head)
        if sym_len - 16 < (bit_len + 7) // 8:
            raise CorruptArchiveError("bit stream data truncated")
        if count != n:
            raise CorruptArchiveError("decoded stream length does not match the grid")
        huff = (base + sym_off + 16, bit_len, count, maxlen)
    else:
        if sym_len < 8:
            raise CorruptArchiveError("run section shorter than its count")
        (R,) = struct.unpack_from("<Q", host_bytes(sym_off, sym_off + 8))
        if hdr.workflow is Workflow.RLE:
            if sym_len != 8 + 8 * R:
                raise CorruptArchiveError("run section size mismatch")
            vptr, lptr = base + sym_off + 8, base + sym_off + 8 + 4 * R
        else:
            head = host_bytes(sym_off + 8, sym_off + 8 + min(16, sym_len - 8))
            if len(head) < 16:
                raise CorruptArchiveError("bit stream shorter than its header")
            bit_len, count = struct.unpack_from("<QQ", head)
            nbytes = (bit_len + 7) // 8
            if sym_len - 8 - 16 < nbytes:
                raise CorruptArchiveError("bit stream data truncated")
            sub = 16 + nbytes
            if count != R or sym_len != 8 + sub + 4 * R:
                raise CorruptArchiveError("run section size mismatch")
            cbytes = np.frombuffer(host_bytes(hdr.codebook[0], sum(hdr.codebook)), np.uint8)
            maxlen = _validate_lengths_host(cbytes)
            vals = _pool.get("dvals", 4 * max(R, 1), dev)
            vals_rle = (base + sym_off + 24, bit_len, R, maxlen, vals)
            vptr, lptr = _dev(vals), base + sym_off + 8 + sub
    out_off, out_len = hdr.outliers
    dtn = torch.float32 if hdr.dtype == "f32" else torch.float64
    y = out if out is not None else torch.empty(n, dtype=dtn, device=dev)
    g = N.geom(dims.as_tuple(), chunk.as_tuple())



    def run(robust: bool) -> None:
        """Launch the decode + reconstruct kernels (no host sync)."""
        dec = L.lzb_huff_decode_robust if robust else L.lzb_huff_decode
        codes = _pool.get("dcodes", n * cb, dev)
        if huff is not None:
            bptr, bit_len, count, maxlen = huff
            ds = L.lzb_huff_decode_scratch_bytes(bit_len, maxlen, cap)
            d_scr = _pool.get("d_scratch", ds, dev)
            with _Stage(prof, "K5_huff_decode"):
                N.check_rc(dec(bptr, bit_len, count, base + hdr.codebook[0], cap, maxlen, _dev(codes), cb,
                               stp, _dev(d_scr), ds, sp), "huff_decode")
        else:
            if vals_rle is not None:
                vb, bit_len, R_, maxlen, vals = vals_rle
                ds = L.lzb_huff_decode_scratch_bytes(bit_len, maxlen, cap)
                d_scr = _pool.get("d_scratch", ds, dev)
                N.check_rc(dec(vb, bit_len, R_, base + hdr.codebook[0], cap, maxlen, _dev(vals), 4,
                               stp, _dev(d_scr), ds, sp), "huff_decode")
            rs = L.lzb_rle_decode_scratch_bytes(R)
            r_scr = _pool.get("rd_scratch", rs, dev)
            N.check_rc(L.lzb_rle_decode(vptr, lptr, R, cap, _dev(codes), cb, n,
                                        stp + N.STATUS_BYTES, _dev(r_scr), rs, sp), "rle_decode")
        rcs = L.lzb_reconstruct_scratch_bytes(g, hdr.outlier_count)
        rc_scr = _pool.get("rc_scratch", rcs, dev)
        with _Stage(prof, "K6_reconstruct"):
            N.check_rc(L.lzb_reconstruct(_dev(codes), cb, base + out_off, hdr.outlier_count, g,
                                         hdr.eb_abs, cap, y.data_ptr(), _DTYPE_CODES[hdr.dtype], None,
                                         stp + 2 * N.STATUS_BYTES, _dev(rc_scr), rcs, sp),
                       "reconstruct")

    run(False)
    sd, sr, sk = N.read_status(st[: 3 * N.STATUS_BYTES])  # the one sync
    if sd.code == N.LZB_E_RETRY:  # a stream the fast decoder cannot resolve (rare)
        run(True)
        sd, sr, sk = N.read_status(st[: 3 * N.STATUS_BYTES])
    N.raise_for(sd, "decode", "bit stream does not decode to its declared symbols")
    N.raise_for(sr, "rle_decode", "run section does not decode to the grid")
    if sk.code == N.LZB_E_CORRUPT:
        raise CorruptArchiveError("invalid outlier list")
    N.raise_for(sk, "reconstruct")
    return y, hdr, sk.f64(0), sk.f64(1)


def decompress(raw, threads: int = 1) -> Field:
    """Decode an archive back into a Field (P/pipeline.py:318-326).

    ``raw`` may be bytes (values come back as numpy, like the reference) or a
    CUDA uint8 tensor (values stay on the device)."""
    import torch

    if isinstance(raw, (bytes, bytearray, memoryview)):
        raw = bytes(raw)
        parse_header(raw)  # header errors before any device work
        arc = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to("cuda")
        y, hdr, vmin, vmax = decompress_device(arc, raw)
        return Field(hdr.dims, y.cpu().numpy(), vmin, vmax)
    y, hdr, vmin, vmax = decompress_device(raw)
    return Field(hdr.dims, y, vmin, vmax)


def stats(original: Field, reconstructed: Field, archive_bytes: int) -> QualityStats:
    """Distortion and size metrics (P/pipeline.py:329-345), reduced on the GPU."""
    import torch

    if original.dims != reconstructed.dims:
        raise DataError("fields have different dims")
    if archive_bytes <= 0:
        raise DataError("archive size must be positive")
    a = _as_device_values(original)
    b = _as_device_values(reconstructed)
    if a.dtype != b.dtype:
        a = a.to(torch.float64)
        b = b.to(torch.float64)
    L = N.lib()
    st = _pool.get("qstatus", N.STATUS_BYTES, a.device)
    qs = L.lzb_quality_scratch_bytes(a.numel())
    scr = _pool.get("q_scr", qs, a.device)
    N.check_rc(L.lzb_quality(a.data_ptr(), b.data_ptr(), 0 if a.dtype == torch.float32 else 1,
                             a.numel(), _dev(st), _dev(scr), qs, N.stream_ptr()), "quality")
    (s,) = N.read_status(st)
    max_err = s.f64(0)
    rmse = float(math.sqrt(s.f64(1) / a.numel()))
    rng = original.value_range
    if rmse == 0.0:
        psnr = math.inf
    elif rng == 0.0:
        psnr = -math.inf
    else:
        psnr = 20.0 * math.log10(rng / rmse)
    return QualityStats(original.nbytes / archive_bytes, max_err, rmse, psnr)


def gather_chunk_major(quant, spec: ChunkSpec) -> np.ndarray:
    """Grid-order codes -> chunk-major stream (P/pipeline.py:102-105), on device."""
    from .quantize import chunk_major

    return chunk_major(quant.codes, quant.dims, spec, 0)


def scatter_chunk_major(stream, dims: Dims, spec: ChunkSpec):
    """Inverse of gather_chunk_major (P/pipeline.py:108-117), on device."""
    from .quantize import QuantGrid, chunk_major

    if len(stream) != dims.count:
        raise CorruptArchiveError("symbol stream length does not match the grid")
    return QuantGrid(dims, chunk_major(stream, dims, spec, 1))


_SCALAR = SCALAR_DTYPES
