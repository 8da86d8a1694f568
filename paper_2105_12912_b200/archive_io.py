"""Archive files: device archive <-> file through pinned host staging, and
the parallel per-rank write of a sharded archive (the
on-disk format is the reference's, P/pipeline.py:26-39, 184-221).

* ``save(arc, path)`` / ``load(path)``: the archive moves in 64 MB pieces
  through two pinned host buffers, so the device<->host copy of one piece
  overlaps the file write / read of the other.
* ``write_sharded(res, path, lengths)``: every rank of a sharded compress
  (``distributed.compress_sharded``) writes its own byte ranges of the
  archive file with ``pwrite`` -- its slice of the dense bit stream, its
  outlier records, its run lengths (RLE+VLE) -- and rank 0 the header,
  the code book and the section prefixes.  Slices of neighbouring ranks
  share at most a boundary byte; one all-gather of each rank's first and
  last byte lets the lowest sharing rank write their OR.  The file is
  byte-identical to the single-device archive.
"""

from __future__ import annotations

import os

import numpy as np

from .distributed import archive_header, archive_layout, archive_prefix

_PIECE = 64 << 20


def _host_u8(x) -> np.ndarray:
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy().view(np.uint8).reshape(-1)
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x).view(np.uint8).reshape(-1)


def _pwrite_all(fd: int, data, off: int) -> None:
    """os.pwrite until every byte is written (one call moves at most ~2 GiB on
    Linux, and may move less)."""
    mv = memoryview(data).cast("B")
    done = 0
    while done < len(mv):
        k = os.pwrite(fd, mv[done: done + _PWRITE_MAX], off + done)
        if k <= 0:
            raise OSError(f"pwrite wrote {k} bytes at offset {off + done}")
        done += k


_PWRITE_MAX = 1 << 30


def save(arc, path: str) -> int:
    """Write an archive (DeviceArchive, CUDA/CPU uint8 tensor or bytes) to
    `path`; returns the byte count."""
    import torch

    data = getattr(arc, "data", arc)
    n = getattr(arc, "nbytes", None)
    if isinstance(data, (bytes, bytearray, memoryview)):
        with open(path, "wb") as fh:
            fh.write(data)
        return len(data)
    n = data.numel() if n is None else n
    fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        if not data.is_cuda:
            _pwrite_all(fd, data[:n].numpy(), 0)
            return n
        bufs = [torch.empty(min(_PIECE, max(n, 1)), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        events = [None, None]
        pending = None  # (buf index, file offset, length) copied but not yet written
        for k, off in enumerate(range(0, n, _PIECE)):
            ln = min(_PIECE, n - off)
            b = k & 1
            if events[b] is not None:
                events[b].synchronize()
            bufs[b][:ln].copy_(data[off: off + ln], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            events[b] = ev
            if pending is not None:  # write the previous piece while this one copies
                pb, poff, pln = pending
                events[pb].synchronize()
                _pwrite_all(fd, bufs[pb][:pln].numpy(), poff)
            pending = (b, off, ln)
        if pending is not None:
            pb, poff, pln = pending
            events[pb].synchronize()
            _pwrite_all(fd, bufs[pb][:pln].numpy(), poff)
        return n
    finally:
        os.close(fd)


def load(path: str, device="cuda"):
    """Read an archive file into a device uint8 tensor (pinned, overlapped)."""
    import torch

    n = os.path.getsize(path)
    out = torch.empty(n, dtype=torch.uint8, device=device)
    bufs = [torch.empty(min(_PIECE, max(n, 1)), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    events = [None, None]
    with open(path, "rb", buffering=0) as fh:
        for k, off in enumerate(range(0, n, _PIECE)):
            ln = min(_PIECE, n - off)
            b = k & 1
            if events[b] is not None:
                events[b].synchronize()  # the buffer's previous upload is done
            got = fh.readinto(memoryview(bufs[b].numpy())[:ln])
            if got != ln:
                raise OSError(f"{path}: short read")
            out[off: off + ln].copy_(bufs[b][:ln], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            events[b] = ev
    torch.cuda.synchronize()
    return out


def write_sharded(res, path: str, lengths_bytes: bytes | None = None, group=None) -> int:
    """Every rank writes its parts of the archive file; returns its size.
    `lengths_bytes` (the cap code lengths) is only needed on rank 0 and
    defaults to res.meta["lengths"]."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    m = res.meta
    lay = archive_layout(m)
    sl = _host_u8(res.bits) if res.bits is not None else np.zeros(0, np.uint8)
    first = res.byte_start
    last = res.byte_start + len(sl) - 1
    # NCCL groups have no CPU transport: the exchange tensors live where the
    # backend can move them
    tdev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor([len(sl), first, last, int(sl[0]) if len(sl) else 0,
                         int(sl[-1]) if len(sl) else 0], dtype=torch.int64, device=tdev)
    allv = [torch.zeros(5, dtype=torch.int64, device=tdev) for _ in range(world)]
    dist.all_gather(allv, mine, group=group)
    info = [tuple(int(x) for x in v.cpu()) for v in allv]
    # boundary bytes: OR of every rank's contribution, written by the lowest contributor
    merged: dict[int, list] = {}
    for k, (ln, f, l, fv, lv) in enumerate(info):
        if not ln:
            continue
        for idx, val in ((f, fv), (l, lv)) if l != f else ((f, fv),):
            e = merged.setdefault(idx, [0, k])
            e[0] |= val
            e[1] = min(e[1], k)
    if rank == 0:
        fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        os.ftruncate(fd, lay["total"])  # zero padding between sections
        _pwrite_all(fd, archive_header(m, lay), 0)
        if lay["cb_len"]:
            lens = lengths_bytes if lengths_bytes is not None else _host_u8(m["lengths"]).tobytes()
            _pwrite_all(fd, bytes(lens[: m["cap"]]), lay["cb_off"])
        _pwrite_all(fd, archive_prefix(m, lay), lay["sym_off"])
        os.close(fd)
    dist.barrier(group=group)
    fd = os.open(path, os.O_WRONLY)
    try:
        if len(sl):
            lo, hi = 0, len(sl)
            if first in merged:
                val, owner = merged[first]
                if owner == rank:
                    _pwrite_all(fd, bytes([val]), lay["data_off"] + first)
                lo = 1
            if last in merged and hi > lo:
                val, owner = merged[last]
                if owner == rank:
                    _pwrite_all(fd, bytes([val]), lay["data_off"] + last)
                hi -= 1
            if hi > lo:
                _pwrite_all(fd, sl[lo:hi], lay["data_off"] + first + lo)
        if res.records is not None and res.n_out:
            _pwrite_all(fd, _host_u8(res.records)[: 16 * res.n_out],
                        lay["out_off"] + 16 * res.record_start)
        if res.rle is not None and res.rle["n_runs"]:
            k, a = res.rle["n_runs"], 4 * res.rle["run_start"]
            _pwrite_all(fd, _host_u8(res.rle["lens"])[: 4 * k], lay["lens_off"] + a)
            if lay["vals_off"] is not None:
                _pwrite_all(fd, _host_u8(res.rle["vals"])[: 4 * k], lay["vals_off"] + a)
    finally:
        os.close(fd)
    dist.barrier(group=group)
    return lay["total"]
