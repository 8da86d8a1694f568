"""Slab-parallel compression across GPUs.

The field is cut along its slowest axis into slabs of whole chunk layers
(z for 3D, y for 2D, x for 1D).  Chunks never read across a chunk boundary
(P/quantize.py:136-141), so every slab quantises independently, and each
slab is simultaneously a contiguous range of the row-major grid, of the
chunk-major symbol stream and of the globally sorted outlier list.  The only
exchanges are

  1. all-reduce (sum) of the cap-bin int64 histogram -> every rank builds the
     identical canonical code book (K2) and takes the identical 1.09-bit
     workflow decision;
  2. all-gather of the per-rank (bits, outliers) -> each rank knows the bit
     offset B_k of its slab inside the dense Huffman stream and the record
     offset O_k of its outliers;

after which rank k encodes its slab at bit phase B_k mod 8 (lzb_huff_encode_at)
into its own byte slice.  Neighbouring slices share at most one boundary
byte, which the assembly OR-merges; the result is byte-identical to the
single-GPU archive (and to the reference's).

When the 1.09-bit rule selects RLE+VLE, each rank run-length encodes its
slab (K4), the ranks all-gather each slab's boundary runs (first / last
value, total length, split count) and every rank applies the same stitching
plan (``plan_rle_stitch``): a maximal run that crosses slab boundaries --
possibly through whole single-run slabs -- is emitted once, by the rank
where it starts, re-split at the u32 limit exactly as the single-device
encoder splits it.  The run-value histogram of the stitched runs is
all-reduced for the VLE code book, the ranks' value bits and run counts are
all-gathered for offsets, and each rank encodes its values at its bit phase;
the archive is again byte-identical to the single-device one.

Decompression comes in two forms.  ``decompress_sharded`` inverts
``compress_sharded`` with no collective (each rank still holds its own
slice).  ``decompress_archive_sharded`` decodes ONE stored archive,
replicated on every rank, whose slab layout is unknown: rank k takes an
equal, 4096-bit-aligned range of the dense stream, builds that range's
transfer map F_k(phase) = (symbols, exit phase) with the self-synchronising
decoder (lzb_huff_range_maps), the maps are all-gathered (maxlen words per
rank) and chained from phase 0 on every rank, each rank decodes its range
from its resolved entry phase (lzb_huff_range_decode), an all-to-all moves
the symbols to their slab's owner, and each rank reconstructs its slab with
the outlier records of its index range.

The per-rank compute is behind ``SlabOps`` (device kernels in production,
``DeviceSlabOps``); tests drive the same collective/offset/assembly logic
with CPU stand-ins over a gloo process group.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import DataError
from .grid import ChunkSpec, Dims

_HEADER = struct.Struct("<8sHBB3I3IBdddIBQQ6Q")
_SECTION_BASE = (_HEADER.size + 7) & ~7
MAGIC = b"LZEBC\x00\x00\x01"
_WF_CODE = {"HUFFMAN": 0, "RLE": 1, "RLE_VLE": 2}


def _a8(x: int) -> int:
    return (x + 7) & ~7


def archive_layout(meta: dict) -> dict:
    """Section offsets of the archive a sharded compress produces, the same
    as the single-device writer's (P/pipeline.py:158-221):

      HUFFMAN  [cap code lengths] [bit_len][count][bits]
      RLE      (no code book)     [runs][u32 values x runs][u32 lengths x runs]
      RLE_VLE  [cap code lengths] [runs][bit_len][count = runs][value bits][u32 lengths x runs]
    """
    wf = meta.get("workflow", "HUFFMAN")
    cap, runs = meta["cap"], meta.get("n_runs", 0)
    nbytes = 0 if wf == "RLE" else (meta["total_bits"] + 7) // 8
    cb_len = 0 if wf == "RLE" else cap
    cb_off = _SECTION_BASE
    sym_off = _a8(cb_off + cb_len)
    prefix = {"HUFFMAN": 16, "RLE": 8, "RLE_VLE": 24}[wf]
    data_off = sym_off + prefix
    if wf == "RLE":
        sym_len, vals_off, lens_off = 8 + 8 * runs, data_off, data_off + 4 * runs
    else:
        sym_len = prefix + nbytes + (4 * runs if wf == "RLE_VLE" else 0)
        vals_off, lens_off = None, data_off + nbytes
    out_off = _a8(sym_off + sym_len)
    return dict(wf=wf, cb_off=cb_off, cb_len=cb_len, sym_off=sym_off, sym_len=sym_len,
                data_off=data_off, vals_off=vals_off, lens_off=lens_off, nbytes=nbytes,
                out_off=out_off, total=out_off + 16 * meta["total_out"], runs=runs)


def archive_prefix(meta: dict, lay: dict) -> bytes:
    """The symbol section's fixed fields (written once, by rank 0)."""
    if lay["wf"] == "HUFFMAN":
        return struct.pack("<QQ", meta["total_bits"], meta["dims"].count)
    if lay["wf"] == "RLE":
        return struct.pack("<Q", lay["runs"])
    return struct.pack("<QQQ", lay["runs"], meta["total_bits"], lay["runs"])


def archive_header(meta: dict, lay: dict) -> bytes:
    dims, chunk = meta["dims"], meta["chunk"]
    return _HEADER.pack(MAGIC, 1, meta["dtype_code"], dims.ndim, dims.nx, dims.ny, dims.nz,
                        chunk.cx, chunk.cy, chunk.cz, 1 if meta["eb_mode"] == "rel" else 0,
                        meta["eb"], meta["vmin"], meta["vmax"], meta["cap"], _WF_CODE[lay["wf"]],
                        dims.count, meta["total_out"], lay["cb_off"], lay["cb_len"],
                        lay["sym_off"], lay["sym_len"], lay["out_off"], 16 * meta["total_out"])


def slab_bounds(dims: Dims, chunk: ChunkSpec, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) along the slowest axis for `rank`, in whole chunk layers; the
    layers are spread as evenly as possible (earlier ranks get the extra)."""
    if dims.ndim == 3:
        n, c = dims.nz, chunk.cz
    elif dims.ndim == 2:
        n, c = dims.ny, chunk.cy
    else:
        n, c = dims.nx, chunk.cx
    layers = (n + c - 1) // c
    q, r = divmod(layers, world)
    l0 = rank * q + min(rank, r)
    l1 = l0 + q + (1 if rank < r else 0)
    return min(n, l0 * c), min(n, l1 * c)


def slab_dims(dims: Dims, lo: int, hi: int) -> Dims:
    if dims.ndim == 3:
        return Dims(dims.nx, dims.ny, hi - lo, ndim=3)
    if dims.ndim == 2:
        return Dims(dims.nx, hi - lo, ndim=2)
    return Dims(hi - lo, ndim=1)


def slab_index_offset(dims: Dims, lo: int) -> int:
    """Global row-major index of the slab's first element."""
    if dims.ndim == 3:
        return lo * dims.nx * dims.ny
    if dims.ndim == 2:
        return lo * dims.nx
    return lo


@dataclass
class SlabResult:
    """What a rank holds after sharded compression (the timed end state)."""

    rank: int
    byte_start: int       # offset of `bits` inside the symbol stream's data bytes
    bits: object          # uint8 slice (phase-shifted, boundary bytes partial)
    records: object       # this slab's outlier records, global indices (16 B each)
    record_start: int     # record offset inside the outlier section
    meta: dict            # header fields shared by all ranks
    phase: int = 0        # bit phase of the slab's first bit inside bits[0]
    nbits: int = 0        # the slab's bits in the dense stream
    n_out: int = 0        # the slab's outlier records
    rle: dict | None = None  # RLE+VLE: emitted run lengths, run offset, the slab's own runs


class SlabOps:
    """Per-rank compute used by compress_sharded (device kernels or stand-ins)."""

    def quantize(self, values, sdims: Dims, chunk: ChunkSpec, eb_abs: float, cap: int):
        """-> (codes handle, hist int64[cap] (same device as codes), n_out, records handle)."""
        raise NotImplementedError

    def codebook(self, hist, cap: int):
        """-> (lengths handle, code words handle, maxlen int, total_bits int)."""
        raise NotImplementedError

    def local_bits(self, hist, lengths) -> int:
        raise NotImplementedError

    def encode_at(self, codes, n: int, lengths, words, cap: int, maxlen: int, phase: int,
                  bits: int, sym_bytes: int | None = None):
        """-> uint8 slice of ceil((phase + bits) / 8) bytes."""
        raise NotImplementedError

    def offset_records(self, records, n_out: int, offset: int):
        """Global indices: add `offset` to every record's index."""
        raise NotImplementedError

    def to_tensor(self, x):
        """Object -> torch tensor on the collective's device (for all_reduce)."""
        raise NotImplementedError

    # -- RLE+VLE compress --
    def rle_local(self, codes, n: int, max_run: int):
        """Runs of the slab's symbols -> (values, lengths, R, boundary) where
        boundary = (R, head value, head total, head entries, tail value, tail
        total, tail entries); a maximal run split at max_run spans several
        consecutive entries of one value."""
        raise NotImplementedError

    def rle_emit(self, values, lengths, a: int, b: int, group, max_run: int):
        """Entries [a, b) followed by the re-split run `group` = (value,
        total) (or nothing) -> (values u32, lengths u32, count)."""
        raise NotImplementedError

    def value_hist(self, values, n: int, cap: int):
        """int64[cap] histogram of n run values (same device as values)."""
        raise NotImplementedError

    def rle_decode_local(self, values, lengths, runs: int, n: int, cap: int):
        """The slab's symbols from its own (unstitched) runs."""
        raise NotImplementedError

    # -- decompress side (decompress_sharded) --
    def decode_at(self, bits, phase: int, nbits: int, count: int, lengths, cap: int, maxlen: int):
        """Symbols of a slab slice whose first bit is bit `phase` of bits[0]."""
        raise NotImplementedError

    def local_records(self, records, n_out: int, offset: int):
        """Slab-local copy of global-index records (subtract `offset`)."""
        raise NotImplementedError

    def reconstruct(self, codes, sdims: Dims, chunk: ChunkSpec, eb_abs: float, cap: int, records,
                    n_out: int, dtype_code: int):
        """Slab values (fuse outliers, partial sums, dequantise)."""
        raise NotImplementedError


    # -- single-archive decompress (decompress_archive_sharded) --
    def stream_info(self, arc, hdr) -> tuple[int, int, int]:
        """(bit_len, symbol count, max code length) of a Huffman archive."""
        raise NotImplementedError

    def range_maps(self, arc, hdr, bit_len: int, lo: int, hi: int, maxlen: int):
        """int64[maxlen] transfer map of stream bits [lo, hi): (symbols << 8) | exit."""
        raise NotImplementedError

    def range_decode(self, arc, hdr, bit_len: int, lo: int, hi: int, maxlen: int, entry: int,
                     exit_phase: int, count: int):
        """The `count` symbols (code_bytes each) decoded from bit lo + entry."""
        raise NotImplementedError

    def exchange(self, codes, send_bytes: list[int], recv_bytes: list[int], group):
        """all-to-all of byte ranges (rank order on both sides)."""
        raise NotImplementedError

    def slab_records(self, arc, hdr, idx_lo: int, idx_hi: int):
        """(slab-local records, count) of the outliers with lo <= index < hi."""
        raise NotImplementedError

    def rle_slab_codes(self, arc, hdr, s_lo: int, s_hi: int):
        """Symbols [s_lo, s_hi) of a run-length archive (RLE / RLE+VLE): the
        run section is validated whole, only the overlapping runs expanded."""
        raise NotImplementedError


EXIT_END = 0xFE
EXIT_INVALID = 0xFF
RANGE_ALIGN = 4096  # LZB_DEC_RANGE_ALIGN


def stream_ranges(bit_len: int, world: int) -> list[tuple[int, int]]:
    """Equal, RANGE_ALIGN-aligned bit ranges of the dense stream, rank order."""
    t = (bit_len + RANGE_ALIGN - 1) // RANGE_ALIGN
    q, r = divmod(t, world)
    out = []
    for k in range(world):
        t0 = k * q + min(k, r)
        t1 = t0 + q + (1 if k < r else 0)
        out.append((min(bit_len, t0 * RANGE_ALIGN), min(bit_len, t1 * RANGE_ALIGN)))
    return out


def chain_ranges(maps: list, ranges: list[tuple[int, int]], count: int):
    """Chain the ranks' transfer maps from phase 0 (the stream start).

    Returns per rank (entry phase, exit phase, first symbol, symbols).  A
    chain that hits an invalid code word, ends early, or does not end exactly
    at the stream end with `count` symbols is a corrupt archive."""
    from .errors import CorruptArchiveError

    e, o = 0, 0
    out = []
    for k, (lo, hi) in enumerate(ranges):
        if hi <= lo:
            out.append((e, e, o, 0))
            continue
        if e == EXIT_END or e == EXIT_INVALID or e >= len(maps[k]):
            raise CorruptArchiveError("bit stream does not decode to its declared symbols")
        v = int(maps[k][e])
        n, x = v >> 8, v & 0xFF
        out.append((e, x, o, n))
        e, o = x, o + n
    if e != EXIT_END or o != count:
        raise CorruptArchiveError("bit stream does not decode to its declared symbols")
    return out


def _overlap(a0: int, a1: int, b0: int, b1: int) -> int:
    return max(0, min(a1, b1) - max(a0, b0))


def decompress_archive_sharded(ops: SlabOps, arc, group=None, raw_host: bytes | None = None):
    """Rank-local part of decompressing ONE archive held by every rank.

    Returns (this rank's slab values or None, (lo, hi) along the slowest
    axis, header).  Collectives: one all-gather of maxlen int64 per rank and
    one all-to-all of symbols (each rank sends to the one or two slab owners
    its stream range overlaps)."""
    import torch
    import torch.distributed as dist

    from .pipeline import Workflow, code_bytes_for, parse_header

    hdr = parse_header(raw_host if raw_host is not None else arc)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dims, chunk, cap = hdr.dims, hdr.chunk, hdr.cap
    lo, hi = slab_bounds(dims, chunk, rank, world)
    sd = slab_dims(dims, lo, hi) if hi > lo else None
    if hdr.workflow is not Workflow.HUFFMAN:
        # the run section is small and read by every rank; each rank expands
        # only the runs that overlap its slab's symbols (no exchange)
        if sd is None:
            return None, (lo, hi), hdr
        a, b = slab_index_offset(dims, lo), slab_index_offset(dims, hi)
        codes = ops.rle_slab_codes(arc, hdr, a, b)
        recs, n_out = ops.slab_records(arc, hdr, a, b)
        y = ops.reconstruct(codes, sd, chunk, hdr.eb_abs, cap, recs, n_out,
                            0 if hdr.dtype == "f32" else 1)
        return y, (lo, hi), hdr
    bit_len, count, maxlen = ops.stream_info(arc, hdr)
    ranges = stream_ranges(bit_len, world)
    r_lo, r_hi = ranges[rank]
    if r_hi > r_lo:
        fmap = ops.range_maps(arc, hdr, bit_len, r_lo, r_hi, maxlen)
    else:
        fmap = ops.to_tensor(np.arange(maxlen, dtype=np.int64))  # empty range: identity
    fmap = fmap.to(torch.int64).reshape(-1)
    allm = [torch.zeros_like(fmap) for _ in range(world)]
    dist.all_gather(allm, fmap, group=group)
    chain = chain_ranges([m.cpu().numpy() for m in allm], ranges, count)
    entry, exit_phase, first, n_sym = chain[rank]
    cb = code_bytes_for(cap)
    mine = ops.range_decode(arc, hdr, bit_len, r_lo, r_hi, maxlen, entry, exit_phase, n_sym)         if n_sym else None
    # symbol ranges of the slabs (a slab's first chunk-major symbol is its
    # first row-major element: slabs are whole chunk layers)
    starts = [slab_index_offset(dims, slab_bounds(dims, chunk, j, world)[0]) for j in range(world)]
    starts.append(dims.count)
    send = [cb * _overlap(first, first + n_sym, starts[j], starts[j + 1]) for j in range(world)]
    recv = [cb * _overlap(c[2], c[2] + c[3], starts[rank], starts[rank + 1]) for c in chain]
    codes = ops.exchange(mine, send, recv, group)
    if sd is None:
        return None, (lo, hi), hdr
    recs, n_out = ops.slab_records(arc, hdr, starts[rank], starts[rank + 1])
    y = ops.reconstruct(codes, sd, chunk, hdr.eb_abs, cap, recs, n_out,
                        0 if hdr.dtype == "f32" else 1)
    return y, (lo, hi), hdr


def plan_rle_stitch(infos: list, max_run: int):
    """Stitching plan of the slabs' local runs (identical on every rank).

    infos[k] = (R, head value, head total, head entries, tail value, tail
    total, tail entries) of rank k's local runs (R = 0: empty slab).  Returns
    (keep, group, emitted): rank k keeps its local entries [keep[k][0],
    keep[k][1]) and then emits group[k] = (value, total) re-split at max_run
    (the maximal run that starts with its tail and may continue through the
    following slabs), or nothing; emitted[k] is its entry count."""
    world = len(infos)
    keep = [(0, 0)] * world
    group = [None] * world
    cur = None  # open run crossing a boundary: [value, total, owner rank]
    for k, (R, hv, ht, hc, tv, tt, tc) in enumerate(infos):
        if R == 0:
            continue
        uniform = hc == R  # the whole slab is one maximal run
        a = 0
        if cur is not None and cur[0] == hv:
            cur[1] += ht
            a = hc
            if uniform:
                keep[k] = (R, R)
                continue
        elif cur is not None:
            group[cur[2]] = (cur[0], cur[1])
            cur = None
        if cur is None and uniform:
            cur = [hv, ht, k]
            keep[k] = (0, 0)
            continue
        if cur is not None:
            group[cur[2]] = (cur[0], cur[1])
        cur = [tv, tt, k]
        keep[k] = (a, R - tc)
    if cur is not None:
        group[cur[2]] = (cur[0], cur[1])
    emitted = [(b - a) + (0 if g is None else -(-g[1] // max_run)) for (a, b), g in zip(keep, group)]
    return keep, group, emitted


def split_run(total: int, max_run: int) -> list[int]:
    """P/rle.py:17-35: a run longer than max_run becomes max_run-long runs and a remainder."""
    q, r = divmod(total, max_run)
    return [max_run] * q + ([r] if r else [])


def _boundary(hv, hl, tv, tl, r: int) -> tuple:
    """Boundary tuple of a slab's runs from its first / last entries (a
    split maximal run = consecutive entries of one value)."""
    if r == 0:
        return (0, 0, 0, 0, 0, 0, 0)
    hc = 1
    while hc < len(hv) and hv[hc] == hv[0]:
        hc += 1
    tc = 1
    while tc < len(tv) and tv[len(tv) - 1 - tc] == tv[-1]:
        tc += 1
    if hc == len(hv) and len(hv) < r or tc == len(tv) and len(tv) < r:
        raise NotImplementedError("a boundary run split into more than 64 entries")
    return (r, int(hv[0]), int(hl[:hc].astype(np.int64).sum()), hc,
            int(tv[-1]), int(tl[len(tl) - tc:].astype(np.int64).sum()), tc)


def _compress_sharded_rle(ops, codes, n_local, n_out, recs, dims, lo, cap, meta, rank, world, group,
                          device, max_run, vle: bool = True):
    import torch
    import torch.distributed as dist

    if n_local:
        vals, lens, r_k, info = ops.rle_local(codes, n_local, max_run)
    else:
        vals, lens, r_k, info = None, None, 0, (0, 0, 0, 0, 0, 0, 0)
    mine = torch.tensor(list(info), dtype=torch.int64, device=device)
    allv = [torch.zeros(7, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    infos = [tuple(int(x) for x in v) for v in allv]
    keep, grp, emitted = plan_rle_stitch(infos, max_run)
    a, b = keep[rank]
    e_k = emitted[rank]
    ev, el = (ops.rle_emit(vals, lens, a, b, grp[rank], max_run) if e_k else (None, None))
    if n_out:
        recs = ops.offset_records(recs, n_out, slab_index_offset(dims, lo))
    if not vle:  # RLE alone: the stitched runs are the symbol section; only record offsets remain
        mv = torch.tensor([n_out], dtype=torch.int64, device=device)
        allo = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
        dist.all_gather(allo, mv, group=group)
        outs = [int(v[0]) for v in allo]
        meta.update(workflow="RLE", total_bits=0, total_out=sum(outs), lengths=None, maxlen=0,
                    n_runs=sum(emitted))
        rle = dict(lens=el, vals=ev, run_start=sum(emitted[:rank]), n_runs=e_k, local=(vals, lens, r_k))
        return SlabResult(rank, 0, None, recs, sum(outs[:rank]), meta, n_out=n_out, rle=rle)
    # run-value histogram of the stitched runs -> the VLE code book
    vh = ops.value_hist(ev, e_k, cap) if e_k else None
    h = ops.to_tensor(vh) if vh is not None else torch.zeros(cap, dtype=torch.int64, device=device)
    h = h.to(torch.int64).clone()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    lengths, words, maxlen, total_vbits = ops.codebook(h, cap)
    my_bits = ops.local_bits(vh, lengths) if vh is not None else 0
    mv = torch.tensor([my_bits, n_out], dtype=torch.int64, device=device)
    allb = [torch.zeros(2, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(allb, mv, group=group)
    allb = [(int(v[0]), int(v[1])) for v in allb]
    B_k = sum(v[0] for v in allb[:rank])
    O_k = sum(v[1] for v in allb[:rank])
    assert sum(v[0] for v in allb) == total_vbits
    phase = B_k % 8
    bits = ops.encode_at(ev, e_k, lengths, words, cap, maxlen, phase, my_bits, sym_bytes=4) \
        if e_k else None
    meta.update(workflow="RLE_VLE", total_bits=total_vbits, total_out=sum(v[1] for v in allb),
                lengths=lengths, maxlen=maxlen, n_runs=sum(emitted))
    rle = dict(lens=el, run_start=sum(emitted[:rank]), n_runs=e_k, local=(vals, lens, r_k))
    return SlabResult(rank, B_k // 8, bits, recs, O_k, meta, phase=phase, nbits=my_bits,
                      n_out=n_out, rle=rle)


def compress_sharded(ops: SlabOps, values, dims: Dims, vmin: float, vmax: float, eb: float,
                     eb_mode: str, cap: int, chunk: ChunkSpec, dtype_code: int, group=None,
                     device=None, max_run: int = 0xFFFFFFFF, workflow=None,
                     select_mode: str = "exact") -> SlabResult:
    """Rank-local part of the sharded compress (every rank calls this with its slab).

    ``workflow`` (None = select, or "huff" / "rle" / "rlevle" / a Workflow)
    and ``select_mode`` ("exact": the code book's bits per symbol;
    "estimate": the entropy-bracket midpoint) mean what they mean for
    ``compress`` (P/pipeline.py:135-182, P/smoothness.py:111-136); the
    decision is taken from the all-reduced histogram, so every rank takes
    the same one."""
    import torch
    import torch.distributed as dist

    from .pipeline import _check_cfg, _resolve_eb, resolve_workflow
    from .smoothness import RLE_THRESHOLD_BITS, Workflow, estimate_bits

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    eb_abs = _resolve_eb(eb_mode, eb, vmin, vmax)
    _check_cfg(eb_abs, cap)
    if device is None:  # an empty slab still joins the collectives on the ops' device
        device = getattr(ops, "device", None)
    lo, hi = slab_bounds(dims, chunk, rank, world)
    sd = slab_dims(dims, lo, hi) if hi > lo else None
    if sd is not None:
        codes, hist, n_out, recs = ops.quantize(values, sd, chunk, eb_abs, cap)
        n_local = sd.count
    else:
        codes, hist, n_out, recs, n_local = None, None, 0, None, 0
    # (1) all-reduce of the histogram
    h = ops.to_tensor(hist) if hist is not None else torch.zeros(cap, dtype=torch.int64,
                                                                 device=device)
    h = h.to(torch.int64).clone()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    chosen = resolve_workflow(workflow)
    if select_mode not in ("exact", "estimate"):
        raise DataError(f"unknown selection mode {select_mode!r}")
    book = None
    if chosen is None:
        if select_mode == "exact":
            book = ops.codebook(h, cap)
            b = float(np.float64(book[3]) / np.float64(dims.count))  # P/codebook.py:110-115
        else:
            b = estimate_bits(h.cpu().numpy())
        chosen = Workflow.RLE_VLE if b <= RLE_THRESHOLD_BITS else Workflow.HUFFMAN
    meta = dict(dims=dims, chunk=chunk, cap=cap, eb=eb, eb_mode=eb_mode, vmin=vmin, vmax=vmax,
                dtype_code=dtype_code, workflow="HUFFMAN")
    if chosen is not Workflow.HUFFMAN:
        return _compress_sharded_rle(ops, codes, n_local, n_out, recs, dims, lo, cap, meta, rank,
                                     world, group, h.device, max_run,
                                     vle=chosen is Workflow.RLE_VLE)
    lengths, words, maxlen, total_bits = book if book is not None else ops.codebook(h, cap)
    # (2) all-gather of (bits, outliers)
    my_bits = ops.local_bits(hist, lengths) if hist is not None else 0
    mine = torch.tensor([my_bits, n_out], dtype=torch.int64, device=h.device)
    allv = [torch.zeros(2, dtype=torch.int64, device=h.device) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    allv = [(int(v[0]), int(v[1])) for v in allv]
    B_k = sum(v[0] for v in allv[:rank])
    O_k = sum(v[1] for v in allv[:rank])
    total_out = sum(v[1] for v in allv)
    assert sum(v[0] for v in allv) == total_bits
    # (3) encode at the slab's bit phase; outliers to global indices
    phase = B_k % 8
    bits = ops.encode_at(codes, n_local, lengths, words, cap, maxlen, phase, my_bits) \
        if n_local else None
    if n_out:
        recs = ops.offset_records(recs, n_out, slab_index_offset(dims, lo))
    meta.update(total_bits=total_bits, total_out=total_out, lengths=lengths, maxlen=maxlen)
    return SlabResult(rank, B_k // 8, bits, recs, O_k, meta, phase=phase, nbits=my_bits, n_out=n_out)


def decompress_sharded(ops: SlabOps, res: SlabResult, group=None):
    """Rank-local inverse of compress_sharded: the rank decodes its own slice of
    the dense stream (its first bit at res.phase, res.nbits long -- exactly the
    bits lzb_huff_encode_at wrote) and reconstructs its slab from it and its
    outlier records.  No collective: the slab boundaries are chunk-layer
    boundaries, so a slab's symbols, chunks and records are all its own.
    Returns the slab's values (None for an empty slab)."""
    import torch.distributed as dist

    from .pipeline import _resolve_eb

    m = res.meta
    dims, chunk, cap = m["dims"], m["chunk"], m["cap"]
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = slab_bounds(dims, chunk, rank, world)
    if hi <= lo:
        return None
    sd = slab_dims(dims, lo, hi)
    eb_abs = _resolve_eb(m["eb_mode"], m["eb"], m["vmin"], m["vmax"])
    if res.rle is not None:  # the slab's own runs (before stitching) decode exactly its symbols
        vals, lens, r_k = res.rle["local"]
        codes = ops.rle_decode_local(vals, lens, r_k, sd.count, cap)
    else:
        codes = ops.decode_at(res.bits, res.phase, res.nbits, sd.count, m["lengths"], cap,
                              m["maxlen"])
    recs = ops.local_records(res.records, res.n_out, slab_index_offset(dims, lo)) if res.n_out \
        else None
    return ops.reconstruct(codes, sd, chunk, eb_abs, cap, recs, res.n_out, m["dtype_code"])


def assemble(results: list[SlabResult], lengths_bytes: bytes) -> bytes:
    """Archive bytes from every rank's slice (rank order).  Byte-identical to
    the single-device archive: the dense stream is the OR of the phase-shifted
    slices (they overlap in at most one byte); runs and records go to their
    ranks' offsets."""
    m = results[0].meta
    lay = archive_layout(m)
    blob = np.zeros(lay["total"], np.uint8)
    hdr = archive_header(m, lay)
    blob[: len(hdr)] = np.frombuffer(hdr, np.uint8)
    if lay["cb_len"]:
        blob[lay["cb_off"]: lay["cb_off"] + m["cap"]] = np.frombuffer(lengths_bytes, np.uint8)[: m["cap"]]
    pre = archive_prefix(m, lay)
    blob[lay["sym_off"]: lay["sym_off"] + len(pre)] = np.frombuffer(pre, np.uint8)
    data = blob[lay["data_off"]: lay["data_off"] + lay["nbytes"]]
    for r in results:
        if r.bits is not None:
            sl = np.asarray(r.bits, np.uint8)
            end = min(lay["nbytes"], r.byte_start + len(sl))
            data[r.byte_start:end] |= sl[: end - r.byte_start]
        if r.records is not None and len(r.records):
            rb = np.asarray(r.records, np.uint8)
            o = lay["out_off"] + 16 * r.record_start
            blob[o: o + len(rb)] = rb
        if r.rle is not None and r.rle["n_runs"]:
            k, a = r.rle["n_runs"], 4 * r.rle["run_start"]
            blob[lay["lens_off"] + a: lay["lens_off"] + a + 4 * k] = _host_bytes(r.rle["lens"])[: 4 * k]
            if lay["vals_off"] is not None:
                blob[lay["vals_off"] + a: lay["vals_off"] + a + 4 * k] = _host_bytes(r.rle["vals"])[: 4 * k]
    return blob.tobytes()


def allgather_archive(res: SlabResult, group=None, device=None, lengths=None):
    """The whole archive, byte-identical to the single-device one, on EVERY
    rank, built from the ranks' slices with one all-gather (NCCL on GPUs).
    Each rank contributes [bits slice | records | run lengths | run values];
    the receivers OR the bit slices (neighbours share at most one byte) and
    place the rest at their offsets.  This is how a sharded compress hands
    a stored archive to ``decompress_archive_sharded`` without any rank
    compressing the full field.  ``device``: where the returned archive
    lives (default: where the backend exchanges -- this GPU for NCCL, host
    memory for gloo); ``lengths``: the code lengths if res.meta has none."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    m = res.meta
    lay = archive_layout(m)
    out_device = device
    # the collective runs where the backend moves data (NCCL: this GPU; gloo: host)
    device = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")

    def u8(x, nbytes):
        if x is None or nbytes == 0:
            return torch.empty(0, dtype=torch.uint8, device=device)
        if isinstance(x, (bytes, bytearray)):
            x = np.frombuffer(x, np.uint8)
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        return t.reshape(-1).view(torch.uint8)[:nbytes].to(device)

    k = res.rle["n_runs"] if res.rle is not None else 0
    nb = 0 if res.bits is None else (res.bits.numel() if isinstance(res.bits, torch.Tensor)
                                     else np.asarray(res.bits).nbytes)
    parts = [u8(res.bits, nb), u8(res.records, 16 * res.n_out),
             u8(res.rle["lens"] if k else None, 4 * k),
             u8(res.rle.get("vals") if k and lay["vals_off"] is not None else None,
                4 * k if lay["vals_off"] is not None else 0)]
    sizes = [p.numel() for p in parts]
    info = torch.tensor(sizes + [res.byte_start, res.record_start,
                                 res.rle["run_start"] if k else 0], dtype=torch.int64, device=device)
    infos = [torch.zeros_like(info) for _ in range(world)]
    dist.all_gather(infos, info, group=group)
    infos = [[int(v) for v in t.cpu()] for t in infos]
    width = max(max(sum(t[:4]) for t in infos), 1)
    mine = torch.zeros(width, dtype=torch.uint8, device=device)
    if sum(sizes):
        torch.cat(parts, out=mine[: sum(sizes)])
    pieces = [torch.empty(width, dtype=torch.uint8, device=device) for _ in range(world)]
    dist.all_gather(pieces, mine, group=group)

    arc = torch.zeros(lay["total"], dtype=torch.uint8, device=device)
    fixed = bytearray(archive_header(m, lay))
    arc[: len(fixed)] = torch.frombuffer(fixed, dtype=torch.uint8).to(device)
    if lay["cb_len"]:
        lens = lengths if lengths is not None else m["lengths"]
        arc[lay["cb_off"]: lay["cb_off"] + m["cap"]] = u8(lens, m["cap"])
    pre = bytearray(archive_prefix(m, lay))
    arc[lay["sym_off"]: lay["sym_off"] + len(pre)] = torch.frombuffer(pre, dtype=torch.uint8).to(device)
    for (n_bits, n_rec, n_len, n_val, bstart, rstart, runstart), pc in zip(infos, pieces):
        o = 0
        if n_bits:  # a slice may run one byte past the stream's end (its phase padding)
            w = min(n_bits, lay["nbytes"] - bstart)
            if w > 0:
                arc[lay["data_off"] + bstart: lay["data_off"] + bstart + w].bitwise_or_(pc[:w])
            o += n_bits
        if n_rec:
            arc[lay["out_off"] + 16 * rstart: lay["out_off"] + 16 * rstart + n_rec] = pc[o: o + n_rec]
            o += n_rec
        if n_len:
            arc[lay["lens_off"] + 4 * runstart: lay["lens_off"] + 4 * runstart + n_len] = pc[o: o + n_len]
            o += n_len
        if n_val:
            arc[lay["vals_off"] + 4 * runstart: lay["vals_off"] + 4 * runstart + n_val] = pc[o: o + n_val]
    return arc if out_device is None else arc.to(out_device)


def gather_results(res: SlabResult, group=None) -> list[SlabResult] | None:
    """Gather every rank's slice to rank 0 (outside the timed region)."""
    import torch.distributed as dist

    rle = None
    if res.rle is not None:
        rle = {k: (None if res.rle.get(k) is None else _host_bytes(res.rle[k])) for k in ("lens", "vals")}
        rle.update(run_start=res.rle["run_start"], n_runs=res.rle["n_runs"])
    host = SlabResult(res.rank, res.byte_start,
                      None if res.bits is None else _host_bytes(res.bits),
                      None if res.records is None else _host_bytes(res.records),
                      res.record_start, {k: v for k, v in res.meta.items() if k != "lengths"},
                      rle=rle)
    out = [None] * dist.get_world_size(group) if dist.get_rank(group) == 0 else None
    dist.gather_object(host, out, dst=0, group=group)
    return out


def _host_bytes(x) -> np.ndarray:
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy().view(np.uint8).reshape(-1)
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x).view(np.uint8).reshape(-1)


# ---------------------------------------------------------------------------
# production ops: the liblzb.so kernels
# ---------------------------------------------------------------------------
class DeviceSlabOps(SlabOps):
    def __init__(self, device):
        self.device = device

    def quantize(self, values, sdims, chunk, eb_abs, cap):
        import torch

        from . import _native as N
        from .pipeline import code_bytes_for

        L = N.lib()
        n = sdims.count
        cb = code_bytes_for(cap)
        codes = torch.empty(n * cb, dtype=torch.uint8, device=self.device)
        hist = torch.empty(cap, dtype=torch.int64, device=self.device)
        g = N.geom(sdims.as_tuple(), chunk.as_tuple())
        cap_out = min(n, n // 128 + 4096)
        dt = 0 if values.dtype == torch.float32 else 1
        while True:
            recs = torch.empty(max(cap_out, 1) * 16, dtype=torch.uint8, device=self.device)
            qs = L.lzb_quantize_scratch_bytes(g, cap_out)
            scr = N.empty_bytes(qs, self.device)
            st = N.empty_bytes(N.STATUS_BYTES, self.device)
            N.check_rc(L.lzb_quantize(values.data_ptr(), dt, g, eb_abs, cap, codes.data_ptr(), cb,
                                      hist.data_ptr(), recs.data_ptr(), cap_out, st.data_ptr(),
                                      scr.data_ptr(), qs, N.stream_ptr()), "quantize")
            (s,) = N.read_status(st)
            if s.code == N.LZB_E_CAPACITY:
                cap_out = s.u[0] + 1024
                continue
            N.raise_for(s, "quantize")
            return codes, hist, s.u[0], recs[: 16 * s.u[0]]

    def codebook(self, hist, cap):
        import torch

        from . import _native as N

        L = N.lib()
        lens = torch.empty(cap, dtype=torch.uint8, device=self.device)
        words = torch.empty(cap, dtype=torch.int64, device=self.device)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        ss = L.lzb_codebook_scratch_bytes(cap)
        scr = N.empty_bytes(ss, self.device)
        N.check_rc(L.lzb_codebook(hist.data_ptr(), cap, lens.data_ptr(), words.data_ptr(),
                                  st.data_ptr(), scr.data_ptr(), ss, N.stream_ptr()), "codebook")
        (s,) = N.read_status(st)
        if s.code:
            raise DataError("histogram too skewed: code length exceeds 64 bits")
        return lens, words, s.u[2], s.u[0]

    def local_bits(self, hist, lengths):
        import torch

        return int((hist.to(torch.int64) * lengths.to(torch.int64)).sum().item())

    def encode_at(self, codes, n, lengths, words, cap, maxlen, phase, bits, sym_bytes=None):
        from . import _native as N
        from .pipeline import code_bytes_for

        L = N.lib()
        sb = sym_bytes or code_bytes_for(cap)
        nbytes = (phase + bits + 7) // 8
        out = N.empty_bytes(nbytes + 4, self.device)
        out[: nbytes].zero_()
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        es = L.lzb_huff_encode_scratch_bytes(n)
        scr = N.empty_bytes(es, self.device)
        N.check_rc(L.lzb_huff_encode_at(codes.data_ptr(), sb, n,
                                        lengths.data_ptr(), words.data_ptr(), cap, maxlen, phase,
                                        out.data_ptr(), nbytes, st.data_ptr(), scr.data_ptr(), es,
                                        N.stream_ptr()), "huff_encode_at")
        return out[:nbytes]

    def rle_local(self, codes, n, max_run):
        import torch

        from . import _native as N

        L = N.lib()
        cb = codes.numel() // n  # code bytes (the quantize output is n * code_bytes)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        N.check_rc(L.lzb_count_runs(codes.data_ptr(), cb, n, st.data_ptr(), N.stream_ptr()), "count_runs")
        (sc,) = N.read_status(st)
        N.raise_for(sc, "count_runs")
        cap_runs = sc.u[0] + (n // max_run + 1 if n > max_run else 0)
        vals = torch.empty(max(cap_runs, 1), dtype=torch.int32, device=self.device)
        lens = torch.empty(max(cap_runs, 1), dtype=torch.int32, device=self.device)
        rs = L.lzb_rle_encode_scratch_bytes_runs(n, cap_runs)
        scr = N.empty_bytes(rs, self.device)
        N.check_rc(L.lzb_rle_encode(codes.data_ptr(), cb, n, vals.data_ptr(), lens.data_ptr(), cap_runs,
                                    max_run, st.data_ptr(), scr.data_ptr(), rs, N.stream_ptr()),
                   "rle_encode")
        (sr,) = N.read_status(st)
        N.raise_for(sr, "rle_encode")
        r = sr.u[0]
        vals, lens = vals[:r], lens[:r]
        k = min(r, 64)
        hv_ = vals[:k].cpu().numpy().view(np.uint32)
        hl_ = lens[:k].cpu().numpy().view(np.uint32)
        tv_ = vals[r - k:].cpu().numpy().view(np.uint32)
        tl_ = lens[r - k:].cpu().numpy().view(np.uint32)
        return vals, lens, r, _boundary(hv_, hl_, tv_, tl_, r)

    def rle_emit(self, values, lengths, a, b, group, max_run):
        import torch

        parts_v, parts_l = [values[a:b]], [lengths[a:b]]
        if group is not None:
            sp = split_run(group[1], max_run)
            parts_v.append(torch.full((len(sp),), group[0], dtype=torch.int32, device=self.device))
            parts_l.append(torch.tensor(np.array(sp, np.uint32).view(np.int32), device=self.device))
        return torch.cat(parts_v).contiguous(), torch.cat(parts_l).contiguous()

    def value_hist(self, values, n, cap):
        import torch

        from . import _native as N

        L = N.lib()
        h = torch.empty(cap, dtype=torch.int64, device=self.device)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        N.check_rc(L.lzb_histogram(values.data_ptr(), 4, n, cap, h.data_ptr(), st.data_ptr(),
                                   N.stream_ptr()), "histogram")
        (s,) = N.read_status(st)
        N.raise_for(s, "histogram")
        return h

    def rle_decode_local(self, values, lengths, runs, n, cap):
        import torch

        from . import _native as N
        from .pipeline import code_bytes_for

        L = N.lib()
        cb = code_bytes_for(cap)
        sym = torch.empty(n * cb, dtype=torch.uint8, device=self.device)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        rs = L.lzb_rle_decode_scratch_bytes(runs)
        scr = N.empty_bytes(rs, self.device)
        N.check_rc(L.lzb_rle_decode(values.data_ptr(), lengths.data_ptr(), runs, cap, sym.data_ptr(), cb,
                                    n, st.data_ptr(), scr.data_ptr(), rs, N.stream_ptr()), "rle_decode")
        self._decode_status = st
        return sym

    def offset_records(self, records, n_out, offset):
        import torch

        r = records.view(torch.int64).view(-1, 2)
        r[:, 0] += offset
        return records

    def to_tensor(self, x):
        import torch

        return torch.as_tensor(x, device=self.device)

    def decode_at(self, bits, phase, nbits, count, lengths, cap, maxlen):
        import torch

        from . import _native as N
        from .pipeline import code_bytes_for

        L = N.lib()
        cb = code_bytes_for(cap)
        sym = torch.empty(count * cb, dtype=torch.uint8, device=self.device)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        ds = L.lzb_huff_decode_scratch_bytes(nbits, maxlen, cap)
        scr = N.empty_bytes(ds, self.device)
        N.check_rc(L.lzb_huff_decode_at(bits.data_ptr(), phase, nbits, count, lengths.data_ptr(), cap,
                                        maxlen, sym.data_ptr(), cb, st.data_ptr(), scr.data_ptr(), ds,
                                        N.stream_ptr()), "huff_decode_at")
        self._decode_status = st  # read with the reconstruct status (one sync)
        return sym

    def local_records(self, records, n_out, offset):
        import torch

        r = records.view(torch.int64).view(-1, 2).clone()
        r[:, 0] -= offset
        return r.view(torch.uint8).view(-1)

    def reconstruct(self, codes, sdims, chunk, eb_abs, cap, records, n_out, dtype_code):
        import torch

        from . import _native as N
        from .errors import CorruptArchiveError
        from .pipeline import code_bytes_for

        L = N.lib()
        y = torch.empty(sdims.count, dtype=torch.float32 if dtype_code == 0 else torch.float64,
                        device=self.device)
        g = N.geom(sdims.as_tuple(), chunk.as_tuple())
        rs = L.lzb_reconstruct_scratch_bytes(g, n_out)
        scr = N.empty_bytes(rs, self.device)
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        N.check_rc(L.lzb_reconstruct(codes.data_ptr(), code_bytes_for(cap),
                                     records.data_ptr() if records is not None else None, n_out, g,
                                     eb_abs, cap, y.data_ptr(), dtype_code, None, st.data_ptr(),
                                     scr.data_ptr(), rs, N.stream_ptr()), "reconstruct")
        if getattr(self, "_decode_status", None) is not None:
            (sd,) = N.read_status(self._decode_status)
            N.raise_for(sd, "decode", "bit stream does not decode to its declared symbols")
        (sk,) = N.read_status(st)
        if sk.code == N.LZB_E_CORRUPT:
            raise CorruptArchiveError("invalid outlier list")
        N.raise_for(sk, "reconstruct")
        return y

    # -- single-archive decompress --
    def _host(self, arc, a: int, b: int) -> bytes:
        return arc[a:b].cpu().numpy().tobytes()

    def stream_info(self, arc, hdr):
        from .errors import CorruptArchiveError
        from .pipeline import _validate_lengths_host

        sym_off, sym_len = hdr.symbols
        if sym_len < 16:
            raise CorruptArchiveError("bit stream shorter than its header")
        bit_len, count = struct.unpack("<QQ", self._host(arc, sym_off, sym_off + 16))
        if sym_len - 16 < (bit_len + 7) // 8:
            raise CorruptArchiveError("bit stream data truncated")
        if count != hdr.count:
            raise CorruptArchiveError("decoded stream length does not match the grid")
        cb = np.frombuffer(self._host(arc, hdr.codebook[0], sum(hdr.codebook)), np.uint8)
        return bit_len, count, _validate_lengths_host(cb)

    def _range_scratch(self, lo, hi, maxlen, cap):
        from . import _native as N

        key = (lo, hi, maxlen, cap)
        if getattr(self, "_rkey", None) != key:
            L = N.lib()
            self._rbytes = L.lzb_huff_range_scratch_bytes(hi - lo, maxlen, cap)
            self._rscr = N.empty_bytes(self._rbytes, self.device)
            self._rst = N.empty_bytes(N.STATUS_BYTES, self.device)
            self._rkey = key
        return self._rscr, self._rbytes, self._rst

    def range_maps(self, arc, hdr, bit_len, lo, hi, maxlen):
        import torch

        from . import _native as N

        L = N.lib()
        scr, nb, st = self._range_scratch(lo, hi, maxlen, hdr.cap)
        fmap = torch.empty(maxlen, dtype=torch.int64, device=self.device)
        base = arc.data_ptr()
        N.check_rc(L.lzb_huff_range_maps(base + hdr.symbols[0] + 16, bit_len, lo, hi,
                                         base + hdr.codebook[0], hdr.cap, maxlen, fmap.data_ptr(),
                                         st.data_ptr(), scr.data_ptr(), nb, N.stream_ptr()),
                   "huff_range_maps")
        (s,) = N.read_status(st)
        N.raise_for(s, "decode", "bit stream does not decode to its declared symbols")
        return fmap

    def range_decode(self, arc, hdr, bit_len, lo, hi, maxlen, entry, exit_phase, count):
        import torch

        from . import _native as N
        from .pipeline import code_bytes_for

        L = N.lib()
        cb = code_bytes_for(hdr.cap)
        scr, nb, st = self._range_scratch(lo, hi, maxlen, hdr.cap)
        sym = torch.empty(count * cb, dtype=torch.uint8, device=self.device)
        base = arc.data_ptr()
        N.check_rc(L.lzb_huff_range_decode(base + hdr.symbols[0] + 16, bit_len, lo, hi,
                                           base + hdr.codebook[0], hdr.cap, maxlen, entry,
                                           exit_phase if exit_phase < 0xFE else 0, count,
                                           sym.data_ptr(), cb, st.data_ptr(), scr.data_ptr(), nb,
                                           N.stream_ptr()), "huff_range_decode")
        self._decode_status = st
        return sym

    def exchange(self, codes, send_bytes, recv_bytes, group):
        import torch
        import torch.distributed as dist

        inp = codes if codes is not None else torch.empty(0, dtype=torch.uint8, device=self.device)
        out = torch.empty(sum(recv_bytes), dtype=torch.uint8, device=self.device)
        if dist.get_backend(group) == "gloo":  # CPU transport (tests, same-device runs)
            o = torch.empty(sum(recv_bytes), dtype=torch.uint8)
            dist.all_to_all_single(o, inp.cpu(), recv_bytes, send_bytes, group=group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, recv_bytes, send_bytes, group=group)
        return out

    def slab_records(self, arc, hdr, idx_lo, idx_hi):
        import torch

        n = hdr.outlier_count
        if n == 0:
            return None, 0
        off = hdr.outliers[0]
        r = arc[off: off + 16 * n].view(torch.int64).view(-1, 2)
        # P/pipeline.py:306-315: indices strictly increasing and < count, else the
        # archive is corrupt -- checked on every rank, so all ranks fail alike
        idx = r[:, 0]
        bad = (idx[0] < 0) | (idx[-1] >= hdr.count)
        if n > 1:
            bad = bad | (idx[1:] <= idx[:-1]).any()
        if bool(bad):
            from .errors import CorruptArchiveError

            raise CorruptArchiveError("invalid outlier list")
        b = torch.searchsorted(r[:, 0].contiguous(),
                               torch.tensor([idx_lo, idx_hi], dtype=torch.int64, device=arc.device))
        a, z = (int(v) for v in b.cpu())
        if z <= a:
            return None, 0
        return self.local_records(r[a:z].reshape(-1).view(torch.uint8), z - a, idx_lo), z - a

    def rle_slab_codes(self, arc, hdr, s_lo, s_hi):
        import torch

        from . import _native as N
        from .errors import CorruptArchiveError
        from .pipeline import Workflow, _validate_lengths_host

        L = N.lib()
        cap, n = hdr.cap, hdr.count
        sym_off, sym_len = hdr.symbols
        if sym_len < 8:
            raise CorruptArchiveError("run section shorter than its count")
        (R,) = struct.unpack("<Q", self._host(arc, sym_off, sym_off + 8))
        base = arc.data_ptr()
        st = N.empty_bytes(N.STATUS_BYTES, self.device)
        if hdr.workflow is Workflow.RLE:
            if sym_len != 8 + 8 * R:
                raise CorruptArchiveError("run section size mismatch")
            vals = arc[sym_off + 8: sym_off + 8 + 4 * R].view(torch.int32)
            lo_len = sym_off + 8 + 4 * R
        else:
            if sym_len < 24:
                raise CorruptArchiveError("bit stream shorter than its header")
            bit_len, count = struct.unpack("<QQ", self._host(arc, sym_off + 8, sym_off + 24))
            nbytes = (bit_len + 7) // 8
            if sym_len - 24 < nbytes:
                raise CorruptArchiveError("bit stream data truncated")
            if count != R or sym_len != 8 + 16 + nbytes + 4 * R:
                raise CorruptArchiveError("run section size mismatch")
            cb = np.frombuffer(self._host(arc, hdr.codebook[0], sum(hdr.codebook)), np.uint8)
            maxlen = _validate_lengths_host(cb)
            vals = torch.empty(max(R, 1), dtype=torch.int32, device=self.device)
            ds = L.lzb_huff_decode_scratch_bytes(bit_len, maxlen, cap)
            scr = N.empty_bytes(ds, self.device)
            N.check_rc(L.lzb_huff_decode(base + sym_off + 24, bit_len, R, base + hdr.codebook[0], cap,
                                         maxlen, vals.data_ptr(), 4, st.data_ptr(), scr.data_ptr(), ds,
                                         N.stream_ptr()), "huff_decode")
            (sd,) = N.read_status(st)
            N.raise_for(sd, "decode", "bit stream does not decode to its declared symbols")
            lo_len = sym_off + 24 + nbytes
        if R == 0:
            raise CorruptArchiveError("run section does not decode to the grid")
        lens = arc[lo_len: lo_len + 4 * R].clone().view(torch.int32)  # unaligned in RLE+VLE
        l64 = lens.to(torch.int64) & 0xFFFFFFFF
        cum = torch.cumsum(l64, 0)
        bad = torch.stack([(l64 == 0).any().to(torch.int64), cum[-1]]).cpu()
        if int(bad[0]) or int(bad[1]) != n:  # P/rle.py:38-44
            raise CorruptArchiveError("run section does not decode to the grid")
        q = torch.tensor([s_lo, s_hi - 1], dtype=torch.int64, device=self.device)
        ra, rb = (int(v) for v in torch.searchsorted(cum, q, right=True).cpu())
        sub_v = vals[ra: rb + 1].contiguous()
        sub_l = lens[ra: rb + 1].clone()
        edges = torch.stack([cum[ra] - l64[ra], cum[rb]]).cpu()
        first_start, last_end = int(edges[0]), int(edges[1])
        def as_i32(v: int) -> int:  # u32 run length in the int32 tensor's bit pattern
            return int(np.uint32(v).view(np.int32))

        cum_ra = int(edges[0]) + int(l64[ra])
        if ra == rb:
            sub_l[0] = as_i32(s_hi - s_lo)
        else:
            sub_l[0] = as_i32(cum_ra - s_lo)
            sub_l[-1] = as_i32(int(l64[rb]) - (last_end - s_hi))
        return self.rle_decode_local(sub_v, sub_l, rb - ra + 1, s_hi - s_lo, cap)
