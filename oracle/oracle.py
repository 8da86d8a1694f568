"""CPU oracle for the lzebc compress/decompress path.  TEST INFRASTRUCTURE ONLY.

This module is the parity checker (and the timed CPU baseline) for the B200
product in ``paper_2105_12912_b200``.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
it.  The product never imports, links or calls anything under ``oracle/``.

It restates the reference package (``/root/reference/pkg/src/lzebc``, cited
below as ``P/<file>:<line>``) in two layers:

* ``lzb_oracle.c`` (plain C, loaded with ctypes): the element loops --
  prequantization, the per-chunk Lorenzo delta loop, bit packing, bit-serial
  canonical decoding, run-length coding and the per-chunk prefix-sum
  reconstruction.
* this file: the host logic -- error-bound resolution, the heap Huffman
  code-length build, canonical code assignment, workflow selection and the
  130-byte archive header / section table.

Parity pin: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by the reference itself (``oracle/gen_golden.py`` ->
``tests/golden/``), and, when ``/root/reference`` is mounted, against the live
reference on fresh random inputs.
"""

from __future__ import annotations

import ctypes
import heapq
import math
import os
import struct

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblzb_oracle.so")

# Status codes of lzb_oracle.c
_OK, _E_DATA, _E_OVERFLOW, _E_CORRUPT, _E_ASSERT = 0, 2, 3, 4, 6


class OracleError(Exception):
    """Base: the oracle's exceptions mirror P/errors.py:4-17 by name."""


class DataError(OracleError):
    pass


class QuantOverflowError(DataError):
    pass


class CorruptArchiveError(OracleError):
    pass


def build() -> str:
    """Compile lzb_oracle.c (make -C oracle); returns the library path."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.orc_prequantize.argtypes = [P, I, I64, D, P, I]
        L.orc_prequantize.restype = I
        L.orc_construct_stream.argtypes = [P, I64, I64, I64, I, I64, I64, I64, I64, P, P, P, I64, I]
        L.orc_construct_stream.restype = I64
        L.orc_gather_chunk_major.argtypes = [P, I64, I64, I64, I64, I64, I64, P]
        L.orc_scatter_chunk_major.argtypes = [P, I64, I64, I64, I64, I64, I64, P]
        L.orc_histogram.argtypes = [P, I64, I64, P]
        L.orc_histogram.restype = I
        L.orc_huff_encode.argtypes = [P, I64, P, P, I64, P, I64]
        L.orc_huff_encode.restype = I64
        L.orc_huff_decode.argtypes = [P, I64, I64, P, P, P, P, P]
        L.orc_huff_decode.restype = I64
        L.orc_rle_encode.argtypes = [P, I64, ctypes.c_uint64, P, P, I64]
        L.orc_rle_encode.restype = I64
        L.orc_rle_decode.argtypes = [P, P, I64, P, I64]
        L.orc_rle_decode.restype = I
        L.orc_reconstruct_stream.argtypes = [P, I64, I64, I64, I, I64, I64, I64, I64, P, P, I64,
                                             P, D, I, P, I]
        L.orc_reconstruct_stream.restype = I
        L.orc_finite_minmax.argtypes = [P, I, I64, P, P]
        L.orc_finite_minmax.restype = I64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# geometry (P/grid.py:24, 116-132)
# --------------------------------------------------------------------------
DEFAULT_CHUNK = {1: (256, 1, 1), 2: (16, 16, 1), 3: (8, 8, 8)}
MAX_CODE_LEN = 64  # P/codebook.py:20
RLE_THRESHOLD_BITS = 1.09  # P/smoothness.py:26
MAX_RUN = 0xFFFFFFFF  # P/rle.py:14
HUFFMAN, RLE, RLE_VLE = 0, 1, 2  # P/smoothness.py:32-37


def check_finite_minmax(values: np.ndarray) -> tuple[float, float]:
    """Field.from_array / ingest range + finiteness (P/grid.py:155-202)."""
    v = np.ascontiguousarray(values)
    lo, hi = ctypes.c_double(), ctypes.c_double()
    bad = lib().orc_finite_minmax(_p(v), int(v.dtype == np.float64), v.size,
                                  ctypes.byref(lo), ctypes.byref(hi))
    if bad >= 0:
        raise DataError(f"non-finite value at element offset {bad}")
    return float(lo.value), float(hi.value)


# --------------------------------------------------------------------------
# quantization (P/quantize.py:90-213)
# --------------------------------------------------------------------------
def prequantize(values: np.ndarray, eb_abs: float, threads: int = 1) -> np.ndarray:
    """round-half-away(f64(x) / (2 eb_abs)) as int64 (P/quantize.py:95-110)."""
    v = np.ascontiguousarray(values)
    out = np.empty(v.size, np.int64)
    st = lib().orc_prequantize(_p(v), int(v.dtype == np.float64), v.size, float(eb_abs),
                               _p(out), threads)
    if st == _E_OVERFLOW:
        raise QuantOverflowError("prequantized magnitude exceeds the integer range; "
                                 "use a larger error bound")
    if st == _E_ASSERT:
        raise AssertionError("prequantization error-bound invariant violated")
    return out


def construct_stream(pre: np.ndarray, dims, chunk, radius: int, threads: int = 1):
    """construct_grid + gather_chunk_major (P/quantize.py:161-193,
    P/pipeline.py:102-105): chunk-major u32 codes and sorted outliers."""
    nx, ny, nz, ndim = dims
    cx, cy, cz = chunk
    n = nx * ny * nz
    stream = np.empty(n, np.uint32)
    cap_out = max(1024, n // 64)
    while True:
        oi = np.empty(cap_out, np.int64)
        od = np.empty(cap_out, np.int64)
        k = lib().orc_construct_stream(_p(pre), nx, ny, nz, ndim, cx, cy, cz, radius,
                                       _p(stream), _p(oi), _p(od), cap_out, threads)
        if k == -1:
            cap_out = n
            continue
        if k < 0:
            raise MemoryError("oracle outlier buffer")
        return stream, oi[:k].copy(), od[:k].copy()


def gather_chunk_major(grid_codes: np.ndarray, dims, chunk) -> np.ndarray:
    nx, ny, nz, _ = dims
    g = np.ascontiguousarray(grid_codes, np.uint32)
    out = np.empty(g.size, np.uint32)
    lib().orc_gather_chunk_major(_p(g), nx, ny, nz, *chunk, _p(out))
    return out


def scatter_chunk_major(stream: np.ndarray, dims, chunk) -> np.ndarray:
    nx, ny, nz, _ = dims
    s = np.ascontiguousarray(stream, np.uint32)
    out = np.empty(s.size, np.uint32)
    lib().orc_scatter_chunk_major(_p(s), nx, ny, nz, *chunk, _p(out))
    return out


def histogram(sym: np.ndarray, cap: int) -> np.ndarray:
    """bincount with a range check (P/codebook.py:23-27)."""
    s = np.ascontiguousarray(sym, np.uint32)
    h = np.empty(cap, np.int64)
    if lib().orc_histogram(_p(s), s.size, cap, _p(h)) != _OK:
        raise DataError(f"symbol {int(s.max())} out of range for cap {cap}")
    return h


# --------------------------------------------------------------------------
# codebook (P/codebook.py:110-190)
# --------------------------------------------------------------------------
def huffman_lengths(counts: np.ndarray) -> np.ndarray:
    """Code lengths of the deterministic heap Huffman tree (P/codebook.py:143-176).

    Queue keys are (frequency, tie) with tie = symbol for leaves and
    cap + k for the k-th internal node; both keys are unique, so the pop
    order -- and hence the tree -- is fully determined.  Depths are computed
    top-down over the internal nodes in reverse creation order.
    """
    cap = len(counts)
    syms = [s for s in range(cap) if counts[s] > 0]
    lengths = np.zeros(cap, np.uint8)
    if not syms:
        raise DataError("cannot build a codebook from an empty histogram")
    if len(syms) == 1:
        lengths[syms[0]] = 1
        return lengths
    n = len(syms)
    pq = [(int(counts[s]), s, i) for i, s in enumerate(syms)]
    heapq.heapify(pq)
    children = []  # internal node k -> (left id, right id)
    while len(pq) > 1:
        fa, _, a = heapq.heappop(pq)
        fb, _, b = heapq.heappop(pq)
        k = len(children)
        children.append((a, b))
        heapq.heappush(pq, (fa + fb, cap + k, n + k))
    depth = [0] * (n + len(children))
    for k in range(len(children) - 1, -1, -1):
        d = depth[n + k] + 1
        a, b = children[k]
        depth[a] = d
        depth[b] = d
    for i, s in enumerate(syms):
        if depth[i] > MAX_CODE_LEN:
            raise DataError("histogram too skewed: code length exceeds 64 bits")
        lengths[s] = depth[i]
    return lengths


def canonical_codes(lengths: np.ndarray) -> np.ndarray:
    """Canonical code words by ascending (length, symbol) (P/codebook.py:179-190)."""
    codes = np.zeros(len(lengths), np.uint64)
    code = 0
    prev = None
    for length in range(1, MAX_CODE_LEN + 1):
        for s in np.flatnonzero(lengths == length):
            if prev is not None:
                code = (code + 1) << (length - prev)
            prev = length
            codes[s] = code
    return codes


def validate_lengths(lengths: np.ndarray) -> None:
    """Codebook.from_lengths checks (P/codebook.py:125-140)."""
    if len(lengths) and int(lengths.max()) > MAX_CODE_LEN:
        raise CorruptArchiveError("codebook length exceeds 64 bits")
    used = [int(v) for v in lengths if v]
    if not used:
        raise CorruptArchiveError("codebook has no symbols")
    if len(used) == 1:
        if used[0] != 1:
            raise CorruptArchiveError("single-symbol codebook must use length 1")
    elif sum(1 << (MAX_CODE_LEN - v) for v in used) != 1 << MAX_CODE_LEN:
        raise CorruptArchiveError("codebook lengths violate Kraft equality")


def average_bits(counts: np.ndarray, lengths: np.ndarray) -> float:
    """Exact <b> = float(sum(c*len) / total) in numpy semantics (P/codebook.py:110-115)."""
    total = counts.sum()
    if total == 0:
        raise DataError("empty histogram")
    return float((counts * lengths).sum() / total)


# --------------------------------------------------------------------------
# entropy and selection (P/codebook.py:30-87, P/smoothness.py:111-136)
# --------------------------------------------------------------------------
def entropy_bits(counts: np.ndarray) -> float:
    total = counts.sum()
    p = counts[counts > 0] / total
    return float(-(p * np.log2(p)).sum()) + 0.0


def _binary_entropy(p: float) -> float:
    if p <= 0.0 or p >= 1.0:
        return 0.0
    return float(-p * np.log2(p) - (1.0 - p) * np.log2(1.0 - p))


def select_workflow(counts: np.ndarray, mode: str = "exact") -> tuple[int, float]:
    """1.09-bit rule: <b> <= 1.09 -> RLE_VLE else HUFFMAN."""
    if mode == "exact":
        b = average_bits(counts, huffman_lengths(counts))
    elif mode == "estimate":
        h = entropy_bits(counts)
        p1 = float(counts.max() / counts.sum())
        r_lo = 1.0 - _binary_entropy(p1) if p1 > 0.4 else 0.0
        r_hi = p1 + 0.086
        b = ((h + r_lo) + (h + r_hi)) / 2.0
    else:
        raise DataError(f"unknown selection mode {mode!r}")
    return (RLE_VLE if b <= RLE_THRESHOLD_BITS else HUFFMAN), b


# --------------------------------------------------------------------------
# Huffman bit stream (P/huffman.py:20-122)
# --------------------------------------------------------------------------
def huff_encode(sym: np.ndarray, lengths: np.ndarray, codes: np.ndarray) -> tuple[int, int, bytes]:
    s = np.ascontiguousarray(sym, np.uint32)
    lens = lengths.astype(np.int64)
    if s.size == 0:
        return 0, 0, b""
    bits = int(lens[s].sum())
    out = np.zeros((bits + 7) // 8, np.uint8)
    L8 = np.ascontiguousarray(lengths, np.uint8)
    C64 = np.ascontiguousarray(codes, np.uint64)
    got = lib().orc_huff_encode(_p(s), s.size, _p(L8), _p(C64), len(lengths), _p(out), out.size)
    if got == -1:
        raise DataError("symbol without a code word in the stream")
    assert got == bits
    return bits, s.size, out.tobytes()


def bitstream_bytes(bit_len: int, count: int, data: bytes) -> bytes:
    """BitStream.to_bytes: <QQ header + data (P/huffman.py:28-29)."""
    return struct.pack("<QQ", bit_len, count) + data


def parse_bitstream(raw: bytes) -> tuple[int, int, bytes]:
    """BitStream.from_bytes (P/huffman.py:31-43)."""
    if len(raw) < 16:
        raise CorruptArchiveError("bit stream shorter than its header")
    bit_len, count = struct.unpack_from("<QQ", raw)
    nbytes = (bit_len + 7) // 8
    if len(raw) - 16 < nbytes:
        raise CorruptArchiveError("bit stream data truncated")
    return bit_len, count, bytes(raw[16:16 + nbytes])


def huff_decode(bit_len: int, count: int, data: bytes, lengths: np.ndarray) -> np.ndarray:
    """Canonical bit-serial decode (P/huffman.py:64-122)."""
    out = np.empty(count, np.uint32)
    if count == 0:
        if bit_len != 0:
            raise CorruptArchiveError("bit stream claims bits but no symbols")
        return out
    codes = canonical_codes(lengths)
    first = np.zeros(MAX_CODE_LEN + 2, np.uint64)
    cnt = np.zeros(MAX_CODE_LEN + 2, np.uint64)
    off = np.zeros(MAX_CODE_LEN + 2, np.int64)
    order = []
    for length in range(1, MAX_CODE_LEN + 1):
        members = list(np.flatnonzero(lengths == length))
        if members:
            first[length] = codes[members[0]]
            cnt[length] = len(members)
            off[length] = len(order)
            order.extend(members)
    syms = np.array(order if order else [0], np.uint32)
    buf = np.frombuffer(data, np.uint8) if data else np.zeros(1, np.uint8)
    buf = np.ascontiguousarray(buf)
    got = lib().orc_huff_decode(_p(buf), bit_len, count, _p(first), _p(cnt), _p(off), _p(syms),
                                _p(out))
    if got != count:
        raise CorruptArchiveError("bit stream does not decode to its declared symbols")
    return out


# --------------------------------------------------------------------------
# run-length codec (P/rle.py:17-44)
# --------------------------------------------------------------------------
def rle_encode(sym: np.ndarray, max_run: int = MAX_RUN) -> tuple[np.ndarray, np.ndarray]:
    s = np.ascontiguousarray(sym, np.uint32)
    cap_runs = s.size + s.size // max(1, max_run) + 1
    v = np.empty(cap_runs, np.uint32)
    ln = np.empty(cap_runs, np.uint32)
    r = lib().orc_rle_encode(_p(s), s.size, max_run, _p(v), _p(ln), cap_runs)
    assert r >= 0
    return v[:r].copy(), ln[:r].copy()


def rle_decode(values: np.ndarray, lengths: np.ndarray, n: int) -> np.ndarray:
    if len(values) != len(lengths):
        raise CorruptArchiveError("run values and lengths differ in count")
    v = np.ascontiguousarray(values, np.uint32)
    ln = np.ascontiguousarray(lengths, np.uint32)
    if ln.size and not ln.all():
        raise CorruptArchiveError("zero-length run")
    out = np.empty(n, np.uint32)
    st = lib().orc_rle_decode(_p(v), _p(ln), v.size, _p(out), n)
    if st != 0:
        raise CorruptArchiveError("decoded stream length does not match the grid")
    return out


# --------------------------------------------------------------------------
# reconstruction (P/reconstruct.py:22-88)
# --------------------------------------------------------------------------
def reconstruct(stream: np.ndarray, dims, chunk, radius: int, out_idx: np.ndarray,
                out_delta: np.ndarray, eb_abs: float, dtype: str, threads: int = 1,
                want_pre: bool = False):
    nx, ny, nz, ndim = dims
    n = nx * ny * nz
    s = np.ascontiguousarray(stream, np.uint32)
    oi = np.ascontiguousarray(out_idx, np.int64)
    od = np.ascontiguousarray(out_delta, np.int64)
    vals = np.empty(n, np.float64 if dtype == "f64" else np.float32)
    pre = np.empty(n, np.int64) if want_pre else None
    st = lib().orc_reconstruct_stream(_p(s), nx, ny, nz, ndim, *chunk, radius, _p(oi), _p(od),
                                      oi.size, _p(pre) if want_pre else None, float(eb_abs),
                                      int(dtype == "f64"), _p(vals), threads)
    if st == _E_OVERFLOW:
        raise QuantOverflowError("prefix-sum magnitude bound exceeded; use a larger error bound "
                                 "or smaller chunks")
    return (vals, pre) if want_pre else vals


# --------------------------------------------------------------------------
# archive (P/pipeline.py:26-326, layout SURVEY Appendix A)
# --------------------------------------------------------------------------
MAGIC = b"LZEBC\x00\x00\x01"
VERSION = 1
HEADER = struct.Struct("<8sHBB3I3IBdddIBQQ6Q")  # 130 bytes
SECTION_BASE = (HEADER.size + 7) & ~7  # 136
_WF = {"auto": None, "huffman": HUFFMAN, "huff": HUFFMAN, "rle": RLE, "rlevle": RLE_VLE}


def resolve_eb(mode: str, value: float, vmin: float, vmax: float) -> float:
    """P/pipeline.py:120-132."""
    if mode not in ("abs", "rel"):
        raise DataError(f"eb mode must be 'abs' or 'rel', got {mode!r}")
    if not (np.isfinite(value) and value > 0):
        raise DataError(f"error bound must be positive and finite, got {value}")
    if mode == "abs":
        return value
    if vmax <= vmin:
        raise DataError("relative error bound needs a nonzero value range; "
                        "use an absolute bound for constant fields")
    return value * (vmax - vmin)


def compress(values: np.ndarray, dims, vmin: float, vmax: float, eb: float, eb_mode: str = "rel",
             cap: int = 1024, workflow=None, chunk=None, select_mode: str = "exact",
             threads: int = 1) -> bytes:
    """Archive bytes for a flat field (P/pipeline.py:135-221).

    dims = (nx, ny, nz, ndim); chunk = (cx, cy, cz) or None for the default.
    """
    nx, ny, nz, ndim = dims
    eb_abs = resolve_eb(eb_mode, eb, vmin, vmax)
    if cap < 4 or cap & (cap - 1):
        raise DataError(f"cap must be a power of two >= 4, got {cap}")
    if not (np.isfinite(eb_abs) and eb_abs > 0):
        raise DataError(f"eb_abs must be positive and finite, got {eb_abs}")
    chunk = tuple(chunk) if chunk else DEFAULT_CHUNK[ndim]
    radius = cap // 2
    pre = prequantize(values, eb_abs, threads)
    stream, oidx, odelta = construct_stream(pre, dims, chunk, radius, threads)
    if workflow is None or isinstance(workflow, int):
        chosen = workflow
    else:
        if workflow.lower() not in _WF:
            raise DataError(f"unknown workflow {workflow!r}")
        chosen = _WF[workflow.lower()]
    if chosen is None:
        chosen, _ = select_workflow(histogram(stream, cap), select_mode)
    if chosen == HUFFMAN:
        lens = huffman_lengths(histogram(stream, cap))
        cb = lens.tobytes()
        sym = bitstream_bytes(*huff_encode(stream, lens, canonical_codes(lens)))
    else:
        rv, rl = rle_encode(stream)
        if chosen == RLE:
            cb = b""
            sym = (struct.pack("<Q", len(rv)) + rv.astype("<u4").tobytes()
                   + rl.astype("<u4").tobytes())
        else:
            lens = huffman_lengths(histogram(rv, cap))
            cb = lens.tobytes()
            sym = (struct.pack("<Q", len(rv))
                   + bitstream_bytes(*huff_encode(rv, lens, canonical_codes(lens)))
                   + rl.astype("<u4").tobytes())
    rec = np.empty(len(oidx), [("i", "<u8"), ("d", "<i8")])
    rec["i"] = oidx
    rec["d"] = odelta
    outb = rec.tobytes()
    sections = [cb, sym, outb]
    offs = []
    pos = SECTION_BASE
    for sec in sections:
        offs.append(pos)
        pos = (pos + len(sec) + 7) & ~7
    hdr = HEADER.pack(MAGIC, VERSION, 1 if values.dtype == np.float64 else 0, ndim, nx, ny, nz,
                      *chunk, 1 if eb_mode == "rel" else 0, eb, vmin, vmax, cap, chosen,
                      nx * ny * nz, len(oidx), offs[0], len(cb), offs[1], len(sym), offs[2],
                      len(outb))
    blob = bytearray(offs[2] + len(outb))
    blob[:len(hdr)] = hdr
    for off, sec in zip(offs, sections):
        blob[off:off + len(sec)] = sec
    return bytes(blob)


def parse_header(raw: bytes) -> dict:
    """Header + section-table validation (P/pipeline.py:224-272)."""
    if len(raw) < HEADER.size:
        raise CorruptArchiveError("archive shorter than its header")
    (magic, version, dt, ndim, nx, ny, nz, cx, cy, cz, ebm, eb, vmin, vmax, cap, wf, count,
     n_out, cbo, cbl, syo, syl, ouo, oul) = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise CorruptArchiveError("bad magic")
    if version != VERSION:
        raise CorruptArchiveError(f"unsupported version {version}")
    if dt not in (0, 1):
        raise CorruptArchiveError(f"unknown dtype code {dt}")
    if wf not in (0, 1, 2):
        raise CorruptArchiveError("invalid header field: workflow")
    if ndim not in (1, 2, 3) or (ndim == 1 and (ny != 1 or nz != 1)) or (ndim == 2 and nz != 1):
        raise CorruptArchiveError("invalid header field: dims")
    if min(nx, ny, nz) < 1 or min(cx, cy, cz) < 1:
        raise CorruptArchiveError("invalid header field: extents")
    if count != nx * ny * nz:
        raise CorruptArchiveError("element count disagrees with dims")
    if cap < 4 or cap & (cap - 1):
        raise CorruptArchiveError(f"invalid cap {cap}")
    if ebm not in (0, 1):
        raise CorruptArchiveError(f"unknown eb mode {ebm}")
    if not (np.isfinite(eb) and eb > 0):
        raise CorruptArchiveError("invalid error bound")
    if ebm == 1 and not vmax > vmin:
        raise CorruptArchiveError("relative bound with degenerate value range")
    prev = SECTION_BASE
    for off, ln in ((cbo, cbl), (syo, syl), (ouo, oul)):
        if off % 8 or off < prev or off + ln > len(raw):
            raise CorruptArchiveError("section table out of bounds or overlapping")
        prev = off + ln
    if cbl != (0 if wf == RLE else cap):
        raise CorruptArchiveError("codebook section size mismatch")
    if oul != n_out * 16:
        raise CorruptArchiveError("outlier section size mismatch")
    eb_abs = eb if ebm == 0 else eb * (vmax - vmin)
    return dict(dtype="f64" if dt else "f32", dims=(nx, ny, nz, ndim), chunk=(cx, cy, cz),
                eb_mode="rel" if ebm else "abs", eb=eb, eb_abs=eb_abs, vmin=vmin, vmax=vmax,
                cap=cap, workflow=wf, count=count, n_out=n_out, codebook=(cbo, cbl),
                symbols=(syo, syl), outliers=(ouo, oul))


def decode_symbols(raw: bytes, h: dict) -> np.ndarray:
    """P/pipeline.py:275-303."""
    off, ln = h["symbols"]
    sec = raw[off:off + ln]
    cb = np.frombuffer(raw[h["codebook"][0]:sum(h["codebook"])], np.uint8).copy()
    if h["workflow"] == HUFFMAN:
        validate_lengths(cb)
        stream = huff_decode(*parse_bitstream(sec), cb)
    else:
        if len(sec) < 8:
            raise CorruptArchiveError("run section shorter than its count")
        (runs,) = struct.unpack_from("<Q", sec)
        if h["workflow"] == RLE:
            if len(sec) != 8 + 8 * runs:
                raise CorruptArchiveError("run section size mismatch")
            rv = np.frombuffer(sec, "<u4", runs, 8).copy()
            rl = np.frombuffer(sec, "<u4", runs, 8 + 4 * runs).copy()
        else:
            bl, cnt, data = parse_bitstream(sec[8:])
            sub = 16 + (bl + 7) // 8
            if cnt != runs or len(sec) != 8 + sub + 4 * runs:
                raise CorruptArchiveError("run section size mismatch")
            validate_lengths(cb)
            rv = huff_decode(bl, cnt, data, cb)
            rl = np.frombuffer(sec, "<u4", runs, 8 + sub).copy()
        if len(rv) != len(rl):
            raise CorruptArchiveError("run values and lengths differ in count")
        if rl.size and not rl.all():
            raise CorruptArchiveError("zero-length run")
        if int(rl.astype(np.int64).sum()) != h["count"]:
            raise CorruptArchiveError("decoded stream length does not match the grid")
        stream = rle_decode(rv, rl, h["count"])
    if len(stream) != h["count"]:
        raise CorruptArchiveError("decoded stream length does not match the grid")
    if len(stream) and int(stream.max()) >= h["cap"]:
        raise CorruptArchiveError("decoded symbol out of range")
    return stream


def decode_outliers(raw: bytes, h: dict) -> tuple[np.ndarray, np.ndarray]:
    """P/pipeline.py:306-315."""
    rec = np.frombuffer(raw, [("i", "<u8"), ("d", "<i8")], h["n_out"], h["outliers"][0])
    idx = rec["i"].astype(np.int64)
    if len(idx) and int(rec["i"].max()) >= h["count"]:
        raise CorruptArchiveError("outlier index out of range")
    if len(idx) > 1 and not (np.diff(idx) > 0).all():
        raise CorruptArchiveError("invalid outlier list: outlier indices must be strictly "
                                  "increasing")
    return idx, rec["d"].astype(np.int64)


def decompress(raw: bytes, threads: int = 1, want_pre: bool = False):
    """P/pipeline.py:318-326.  Returns (values, dims, vmin, vmax) [+ prequant]."""
    h = parse_header(raw)
    stream = decode_symbols(raw, h)
    oidx, odelta = decode_outliers(raw, h)
    res = reconstruct(stream, h["dims"], h["chunk"], h["cap"] // 2, oidx, odelta, h["eb_abs"],
                      h["dtype"], threads, want_pre)
    vals = res[0] if want_pre else res
    lo, hi = check_finite_minmax(vals)
    if want_pre:
        return vals, h["dims"], lo, hi, res[1]
    return vals, h["dims"], lo, hi


def stats(orig: np.ndarray, recon: np.ndarray, vrange: float, archive_bytes: int):
    """QualityStats (P/pipeline.py:329-345): (cr, max_abs_err, rmse, psnr)."""
    diff = orig.astype(np.float64) - recon.astype(np.float64)
    max_err = float(np.abs(diff).max())
    rmse = float(math.sqrt(np.mean(diff * diff)))
    if rmse == 0.0:
        psnr = math.inf
    elif vrange == 0.0:
        psnr = -math.inf
    else:
        psnr = 20.0 * math.log10(vrange / rmse)
    return orig.nbytes / archive_bytes, max_err, rmse, psnr
