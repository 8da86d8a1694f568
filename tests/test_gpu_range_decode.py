"""GPU: bit-range decode (lzb_huff_range_maps / lzb_huff_range_decode), the
per-rank step of decompressing ONE archive on several GPUs.

The ranks are simulated in one process: every range's transfer map is built
through the C-ABI, the maps are chained on the host exactly as
decompress_archive_sharded does after its all-gather, and the ranges'
symbols, concatenated in rank order, must equal the stream.  A 2-rank gloo
run of decompress_archive_sharded on one device covers the collectives."""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _streams():
    rng = np.random.default_rng(2105)
    g = np.array([int(1e6 * 0.5 ** abs(i - 32)) + 1 for i in range(64)], np.int64)
    yield "peaked", rng.choice(64, size=200_000, p=g / g.sum()).astype(np.uint32), 64
    yield "uniform", rng.integers(0, 1024, size=150_000).astype(np.uint32), 1024
    # geometric tail: code lengths into the 30s (long-code paths)
    p = 0.55 ** np.arange(40)
    yield "long", rng.choice(40, size=300_000, p=p / p.sum()).astype(np.uint32), 64
    yield "tiny", np.array([3, 1, 2, 3, 3], np.uint32), 4
    yield "big", rng.choice(64, size=3_000_000, p=g / g.sum()).astype(np.uint32), 64
    yield "wide", rng.integers(0, 70_000, size=100_000).astype(np.uint32), 131072


def _range_decode_all(bs, book, cap, world):
    import torch

    from paper_2105_12912_b200 import _native as N
    from paper_2105_12912_b200 import distributed as D

    L = N.lib()
    cb = 2 if cap <= 65536 else 4
    maxlen = int(book.lengths.max())
    data = np.concatenate([np.asarray(bs.data, np.uint8), np.zeros(16, np.uint8)])
    d = torch.from_numpy(data).cuda()
    lens = torch.from_numpy(book.lengths.astype(np.uint8)).cuda()
    ranges = D.stream_ranges(bs.bit_len, world)
    st = N.empty_bytes(N.STATUS_BYTES)
    maps, scr = [], []
    for lo, hi in ranges:
        if hi <= lo:
            maps.append(None)
            scr.append(None)
            continue
        nb = L.lzb_huff_range_scratch_bytes(hi - lo, maxlen, cap)
        s = N.empty_bytes(nb)
        f = torch.empty(maxlen, dtype=torch.int64, device="cuda")
        N.check_rc(L.lzb_huff_range_maps(d.data_ptr(), bs.bit_len, lo, hi, lens.data_ptr(), cap,
                                         maxlen, f.data_ptr(), st.data_ptr(), s.data_ptr(), nb,
                                         N.stream_ptr()), "range_maps")
        (sm,) = N.read_status(st)
        assert sm.code == 0
        maps.append(f.cpu().numpy())
        scr.append((s, nb))
    chain = D.chain_ranges(maps, ranges, bs.count)
    out = []
    for (lo, hi), (e, x, first, n), sc in zip(ranges, chain, scr):
        if n == 0:
            continue
        sym = torch.empty(n, dtype=torch.int16 if cb == 2 else torch.int32, device="cuda")
        N.check_rc(L.lzb_huff_range_decode(d.data_ptr(), bs.bit_len, lo, hi, lens.data_ptr(), cap,
                                           maxlen, e, x if x < 0xFE else 0, n, sym.data_ptr(), cb,
                                           st.data_ptr(), sc[0].data_ptr(), sc[1], N.stream_ptr()),
                   "range_decode")
        (sd,) = N.read_status(st)
        assert sd.code == 0, (lo, hi)
        v = sym.cpu().numpy()
        out.append(v.view(np.uint16).astype(np.uint32) if cb == 2 else v.view(np.uint32))
    return np.concatenate(out) if out else np.empty(0, np.uint32), chain


@pytest.mark.parametrize("name,stream,cap", list(_streams()), ids=[s[0] for s in _streams()])
def test_range_decode_concatenates_to_stream(cuda, name, stream, cap):
    import paper_2105_12912_b200 as lzb

    book = lzb.Codebook.from_counts(np.bincount(stream, minlength=cap))
    bs = lzb.encode(stream, book)
    for world in (1, 2, 3, 5, 8):
        got, chain = _range_decode_all(bs, book, cap, world)
        assert np.array_equal(got, stream), (name, world)
        assert sum(c[3] for c in chain) == len(stream)


def test_range_maps_rejects_bad_ranges(cuda):
    import torch

    from paper_2105_12912_b200 import _native as N

    L = N.lib()
    d = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    lens = torch.tensor([1, 1, 0, 0], dtype=torch.uint8, device="cuda")
    f = torch.empty(1, dtype=torch.int64, device="cuda")
    st = N.empty_bytes(N.STATUS_BYTES)
    s = N.empty_bytes(1 << 20)
    for lo, hi in ((100, 8192), (0, 5000), (8192, 8192), (0, 40000)):
        rc = L.lzb_huff_range_maps(d.data_ptr(), 30000, lo, hi, lens.data_ptr(), 4, 1, f.data_ptr(),
                                   st.data_ptr(), s.data_ptr(), 1 << 20, N.stream_ptr())
        assert rc == N.LZB_E_ARG, (lo, hi)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, arc_bytes, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import distributed as D

        arc = torch.frombuffer(bytearray(arc_bytes), dtype=torch.uint8).cuda()
        y, (lo, hi), hdr = D.decompress_archive_sharded(D.DeviceSlabOps("cuda"), arc)
        q.put((rank, lo, hi, None if y is None else y.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("workflow", [None, "rle", "rlevle"])
def test_sharded_decompress_of_one_archive_same_device(cuda, workflow):
    import torch.multiprocessing as mp

    from helpers import smooth

    shape = (48, 40, 64)
    vals = smooth(shape).reshape(-1).astype(np.float32)
    if workflow is not None:
        vals = np.round(vals / 8).astype(np.float32)  # long runs
    arc = O.compress(vals, (64, 40, 48, 3), float(vals.min()), float(vals.max()),
                     1e-4 if workflow is None else 1e-2, workflow=workflow)
    assert O.parse_header(arc)["workflow"] == {None: 0, "rle": 1, "rlevle": 2}[workflow]
    ref = O.decompress(arc)[0].reshape(shape)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, arc, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=300) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lo, hi, y in got:
        assert np.array_equal(y, ref[lo:hi].reshape(-1)), rank


def test_range_decode_agrees_with_whole_stream_decode_on_damaged_streams(cuda):
    """Flipped bits, a shortened bit length and a wrong symbol count: the
    chained ranges either fail (CorruptArchiveError / a non-zero status)
    exactly when the whole-stream decoder fails, or return its symbols."""
    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200.errors import CorruptArchiveError
    from paper_2105_12912_b200.huffman import BitStream

    rng = np.random.default_rng(99)
    g = np.array([int(1e6 * 0.6 ** abs(i - 20)) + 1 for i in range(40)], np.int64)
    stream = rng.choice(40, size=120_000, p=g / g.sum()).astype(np.uint32)
    book = lzb.Codebook.from_counts(np.bincount(stream, minlength=64))
    bs = lzb.encode(stream, book)
    cases = []
    for _ in range(6):
        d = np.asarray(bs.data, np.uint8).copy()
        k = int(rng.integers(0, bs.bit_len))
        d[k // 8] ^= np.uint8(0x80 >> (k % 8))
        cases.append(BitStream(bs.bit_len, bs.count, d))
    cases.append(BitStream(bs.bit_len - 3, bs.count, np.asarray(bs.data, np.uint8)))
    cases.append(BitStream(bs.bit_len, bs.count + 1, np.asarray(bs.data, np.uint8)))
    cases.append(BitStream(bs.bit_len, bs.count - 1, np.asarray(bs.data, np.uint8)))
    for i, c in enumerate(cases):
        try:
            want = lzb.decode(c, book)
        except CorruptArchiveError:
            want = None
        for world in (2, 5):
            try:
                got, _ = _range_decode_all(c, book, 64, world)
            except (CorruptArchiveError, AssertionError):
                got = None
            if want is None:
                assert got is None, (i, world)
            else:
                assert got is not None and np.array_equal(got, want), (i, world)
