"""CPU, world_size 2 over gloo: the sharded-compress host logic (slab
bounds, histogram all-reduce, code book, bit/outlier all-gather, bit-phase
slices, OR-merge assembly) reproduces the single-device archive byte for
byte.  The per-rank compute is a CPU stand-in built on the oracle (test
infrastructure); production uses DeviceSlabOps (the CUDA kernels)."""

import os
import socket
import struct

import numpy as np
import pytest

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleSlabOps:
    """CPU stand-in for DeviceSlabOps (tests only)."""

    def quantize(self, values, sdims, chunk, eb_abs, cap):
        pre = O.prequantize(np.asarray(values), eb_abs)
        stream, oi, od = O.construct_stream(pre, sdims.as_tuple(), chunk.as_tuple(), cap // 2)
        rec = np.empty(len(oi), [("i", "<u8"), ("d", "<i8")])
        rec["i"] = oi
        rec["d"] = od
        return stream, O.histogram(stream, cap), len(oi), rec.view(np.uint8)

    def codebook(self, hist, cap):
        h = hist.numpy() if hasattr(hist, "numpy") else np.asarray(hist)
        lens = O.huffman_lengths(h)
        return lens, O.canonical_codes(lens), int(lens.max()), int((h * lens).sum())

    def local_bits(self, hist, lengths):
        return int((np.asarray(hist) * lengths.astype(np.int64)).sum())

    def encode_at(self, codes, n, lengths, words, cap, maxlen, phase, bits, sym_bytes=None):
        b, _, data = O.huff_encode(codes, lengths, words)
        assert b == bits
        arr = np.unpackbits(np.frombuffer(data, np.uint8))[:bits]
        arr = np.concatenate([np.zeros(phase, np.uint8), arr])
        return np.packbits(arr)

    def rle_local(self, codes, n, max_run):
        from paper_2105_12912_b200 import distributed as D

        v, ln = O.rle_encode(np.asarray(codes), max_run)
        return v, ln, len(v), D._boundary(v[:64], ln[:64], v[-64:], ln[-64:], len(v))

    def rle_emit(self, values, lengths, a, b, group, max_run):
        from paper_2105_12912_b200 import distributed as D

        v, ln = list(values[a:b]), list(lengths[a:b])
        if group is not None:
            sp = D.split_run(group[1], max_run)
            v += [group[0]] * len(sp)
            ln += sp
        return np.array(v, np.uint32), np.array(ln, np.uint32)

    def value_hist(self, values, n, cap):
        return O.histogram(np.asarray(values, np.uint32), cap)

    def rle_decode_local(self, values, lengths, runs, n, cap):
        return O.rle_decode(values, lengths, n)

    def offset_records(self, records, n_out, offset):
        r = records.view([("i", "<u8"), ("d", "<i8")]).copy()
        r["i"] += offset
        return r.view(np.uint8)

    def to_tensor(self, x):
        import torch

        return torch.from_numpy(np.asarray(x, np.int64))

    def decode_at(self, bits, phase, nbits, count, lengths, cap, maxlen):
        arr = np.unpackbits(np.asarray(bits, np.uint8))[phase: phase + nbits]
        return O.huff_decode(nbits, count, np.packbits(arr).tobytes(), np.asarray(lengths, np.uint8))

    def local_records(self, records, n_out, offset):
        r = np.asarray(records, np.uint8).view([("i", "<u8"), ("d", "<i8")]).copy()
        r["i"] -= offset
        return r

    def reconstruct(self, codes, sdims, chunk, eb_abs, cap, records, n_out, dtype_code):
        oi = records["i"].astype(np.int64) if records is not None else np.empty(0, np.int64)
        od = records["d"] if records is not None else np.empty(0, np.int64)
        return O.reconstruct(codes, sdims.as_tuple(), chunk.as_tuple(), cap // 2, oi, od, eb_abs,
                             "f32" if dtype_code == 0 else "f64")


    # -- single-archive decompress: the true code-word boundaries come from a
    # whole-stream oracle decode; a range walk decodes bit-serially from its
    # entry until it lands on one of them (self-synchronisation), then follows
    # the true path.
    def stream_info(self, arc, hdr):
        off = hdr.symbols[0]
        bit_len, count = struct.unpack_from("<QQ", arc, off)
        lens = np.frombuffer(arc, np.uint8, hdr.codebook[1], hdr.codebook[0])
        data = arc[off + 16: off + 16 + (bit_len + 7) // 8]
        self._syms = O.huff_decode(bit_len, count, data, lens)
        self._bits = np.unpackbits(np.frombuffer(data, np.uint8))
        self._bounds = np.concatenate([[0], np.cumsum(lens[self._syms].astype(np.int64))])
        codes = O.canonical_codes(lens)
        self._book = {(int(n), int(codes[i])) for i, n in enumerate(lens) if n}
        self._cap = hdr.cap
        return bit_len, count, int(lens.max())

    def _walk(self, pos, hi, bit_len):
        n = 0
        while pos < hi:
            j = int(np.searchsorted(self._bounds, pos))
            if self._bounds[j] == pos:  # synced
                k = int(np.searchsorted(self._bounds, hi))
                return n + k - j, int(self._bounds[k])
            code, ln = 0, 0
            while (ln, code) not in self._book:
                if pos + ln >= bit_len or ln >= 64:
                    return None
                code = (code << 1) | int(self._bits[pos + ln])
                ln += 1
            pos += ln
            n += 1
        return n, pos

    def range_maps(self, arc, hdr, bit_len, lo, hi, maxlen):
        import torch

        f = np.zeros(maxlen, np.int64)
        for ph in range(maxlen):
            w = self._walk(lo + ph, hi, bit_len)
            if w is None:
                f[ph] = 0xFF
            elif hi == bit_len:
                f[ph] = (w[0] << 8) | (0xFE if w[1] == bit_len else 0xFF)
            else:
                f[ph] = (w[0] << 8) | (w[1] - hi)
        return torch.from_numpy(f)

    def range_decode(self, arc, hdr, bit_len, lo, hi, maxlen, entry, exit_phase, count):
        j = int(np.searchsorted(self._bounds, lo + entry))
        assert self._bounds[j] == lo + entry
        assert self._bounds[j + count] == (bit_len if exit_phase == 0xFE else hi + exit_phase)
        return self._syms[j: j + count].astype(np.uint16 if self._cap <= 65536 else np.uint32)

    def exchange(self, codes, send_bytes, recv_bytes, group):
        import torch
        import torch.distributed as dist

        dt = np.uint16 if self._cap <= 65536 else np.uint32
        inp = torch.from_numpy(np.ascontiguousarray(codes).view(np.uint8).copy()) \
            if codes is not None else torch.empty(0, dtype=torch.uint8)
        out = torch.empty(sum(recv_bytes), dtype=torch.uint8)
        dist.all_to_all_single(out, inp, recv_bytes, send_bytes, group=group)
        return out.numpy().view(dt)

    def slab_records(self, arc, hdr, idx_lo, idx_hi):
        r = np.frombuffer(arc, [("i", "<u8"), ("d", "<i8")], hdr.outlier_count, hdr.outliers[0])
        sel = r[(r["i"] >= idx_lo) & (r["i"] < idx_hi)]
        if not len(sel):
            return None, 0
        return self.local_records(sel.view(np.uint8), len(sel), idx_lo), len(sel)

    def rle_slab_codes(self, arc, hdr, s_lo, s_hi):
        return O.decode_symbols(arc, O.parse_header(arc))[s_lo:s_hi]


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import ChunkSpec, Dims
        from paper_2105_12912_b200 import distributed as D

        vals, shape, eb, path = case
        dims = Dims.of(*shape[::-1])
        chunk = ChunkSpec.default_for(dims.ndim)
        lo, hi = D.slab_bounds(dims, chunk, rank, world)
        full = vals.reshape(shape)
        slab = full[lo:hi].reshape(-1) if dims.ndim > 1 else full[lo:hi]
        res = D.compress_sharded(OracleSlabOps(), slab, dims, float(vals.min()),
                                 float(vals.max()), eb, "rel", 1024, chunk, 0)
        from paper_2105_12912_b200 import archive_io

        archive_io.write_sharded(res, path)  # parallel pwrite of every rank's parts
        # slab-local decompress of the rank's own slice == that slab of the
        # single-device decompress
        y = D.decompress_sharded(OracleSlabOps(), res)
        ref = O.decompress(O.compress(vals, dims.as_tuple(), float(vals.min()), float(vals.max()),
                                      eb))[0].reshape(shape)
        want = ref[lo:hi].reshape(-1) if dims.ndim > 1 else ref[lo:hi]
        if hi > lo:
            assert y is not None and np.array_equal(y, want), rank
        else:
            assert y is None  # more ranks than chunk layers: an empty slab
        ref_arc = O.compress(vals, dims.as_tuple(), float(vals.min()), float(vals.max()), eb)
        assert D.allgather_archive(res).numpy().tobytes() == ref_arc, rank
        res.meta.pop("lengths")
        got = D.gather_results(res)
        if rank == 0:
            lens = OracleSlabOps().codebook(
                O.histogram(O.construct_stream(O.prequantize(vals, eb * float(vals.max() - vals.min())),
                                               dims.as_tuple(), chunk.as_tuple(), 512)[0], 1024),
                1024)[0]
            q.put(D.assemble(got, lens.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,world", [(s, w) for s in [(40, 30, 36), (300, 257), (70001,)]
                                          for w in (2, 3)] + [((40, 30, 36), 8), ((300, 257), 4)])
def test_sharded_archive_is_byte_identical(shape, world, tmp_path):
    import torch.multiprocessing as mp

    from helpers import smooth

    vals = smooth(shape).reshape(-1)
    eb = 1e-4
    ref = O.compress(vals, tuple(list(shape[::-1]) + [1] * (3 - len(shape))) + (len(shape),),
                     float(vals.min()), float(vals.max()), eb)
    assert O.parse_header(ref)["workflow"] == O.HUFFMAN
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "sharded.lzb")
    procs = [ctx.Process(target=_worker, args=(r, world, port, (vals, shape, eb, path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == ref
    with open(path, "rb") as fh:
        assert fh.read() == ref  # the ranks' parallel file write


def _archive_worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import distributed as D

        arc, shape = case
        y, (lo, hi), hdr = D.decompress_archive_sharded(OracleSlabOps(), arc, raw_host=arc)
        ref = O.decompress(arc)[0].reshape(shape)
        want = ref[lo:hi].reshape(-1) if len(shape) > 1 else ref[lo:hi]
        if hi > lo:
            assert y is not None and np.array_equal(np.asarray(y), want), rank
        else:
            assert y is None
        q.put((rank, lo, hi))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,workflow,world",
                         [(s, wf, w) for s, wf in [((40, 30, 36), None), ((300, 257), None),
                                                  ((70,), None), ((64, 64), "rle")]
                          for w in (2, 3)] + [((40, 30, 36), None, 8)])
def test_sharded_decompress_of_one_archive(shape, workflow, world):
    """Every rank holds the same archive; the ranks' slabs of the bit-range
    decode (transfer maps all-gathered and chained, symbols all-to-all'd to
    the slab owners) equal the single-process decompress."""
    import torch.multiprocessing as mp

    from helpers import smooth

    vals = smooth(shape).reshape(-1)
    if workflow == "rle":
        vals = np.round(vals * 2).astype(np.float32)  # long runs of equal codes
    dims = tuple(list(shape[::-1]) + [1] * (3 - len(shape))) + (len(shape),)
    arc = O.compress(vals, dims, float(vals.min()), float(vals.max()), 1e-4 if workflow is None
                     else 1e-2, workflow=workflow)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_archive_worker, args=(r, world, port, (arc, shape), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][1] == 0 and all(a[2] == b[1] for a, b in zip(got, got[1:]))


def test_stream_ranges_and_chain():
    from paper_2105_12912_b200 import distributed as D
    from paper_2105_12912_b200.errors import CorruptArchiveError

    for bit_len in (1, 4095, 4096, 4097, 10 * 4096 + 5):
        for world in (1, 2, 3, 8):
            r = D.stream_ranges(bit_len, world)
            assert r[0][0] == 0 and r[-1][1] == bit_len
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all(lo % 4096 == 0 for lo, hi in r if hi > lo)
    # two ranges: [0,4096) maps phase 0 -> 3 symbols exit 2; [4096,..) phase 2 -> END
    ranges = [(0, 4096), (4096, 5000), (5000, 5000)]
    m0 = np.array([(3 << 8) | 2, 0xFF, 0xFF], np.int64)
    m1 = np.array([0xFF, 0xFF, (4 << 8) | 0xFE], np.int64)
    assert D.chain_ranges([m0, m1, None], ranges, 7) == [(0, 2, 0, 3), (2, 0xFE, 3, 4),
                                                         (0xFE, 0xFE, 7, 0)]
    with pytest.raises(CorruptArchiveError):
        D.chain_ranges([m0, m1, None], ranges, 8)  # wrong symbol count
    with pytest.raises(CorruptArchiveError):
        D.chain_ranges([m0, np.array([0xFF, 0xFF, 0xFF]), None], ranges, 7)  # invalid code word
    m0e = np.array([(3 << 8) | 0xFE, 0xFF, 0xFF], np.int64)
    with pytest.raises(CorruptArchiveError):
        D.chain_ranges([m0e, m1, None], ranges, 7)  # END before the last range


def test_slab_bounds_cover_whole_chunk_layers():
    from paper_2105_12912_b200 import ChunkSpec, Dims
    from paper_2105_12912_b200 import distributed as D

    for dims in (Dims.of(64, 64, 2048), Dims.of(33, 17, 45), Dims.of(100, 333), Dims.of(10007)):
        chunk = ChunkSpec.default_for(dims.ndim)
        n = (dims.nx, dims.ny, dims.nz)[dims.ndim - 1]
        c = (chunk.cx, chunk.cy, chunk.cz)[dims.ndim - 1]
        for world in (1, 2, 3, 8):
            prev = 0
            for r in range(world):
                lo, hi = D.slab_bounds(dims, chunk, r, world)
                assert lo == prev and (lo % c == 0 or lo == n) and (hi % c == 0 or hi == n)
                prev = hi
            assert prev == n


def _rle_worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import ChunkSpec, Dims
        from paper_2105_12912_b200 import distributed as D

        vals, shape, eb, ref_arc, path = case
        dims = Dims.of(*shape[::-1])
        chunk = ChunkSpec.default_for(dims.ndim)
        lo, hi = D.slab_bounds(dims, chunk, rank, world)
        full = vals.reshape(shape)
        slab = full[lo:hi].reshape(-1) if dims.ndim > 1 else full[lo:hi]
        res = D.compress_sharded(OracleSlabOps(), slab, dims, float(vals.min()), float(vals.max()), eb,
                                 "rel", 1024, chunk, 0)
        assert res.meta["workflow"] == "RLE_VLE"
        y = D.decompress_sharded(OracleSlabOps(), res)
        ref = O.decompress(ref_arc)[0].reshape(shape)
        want = ref[lo:hi].reshape(-1) if dims.ndim > 1 else ref[lo:hi]
        if hi > lo:
            assert y is not None and np.array_equal(y, want), rank
        lens = np.frombuffer(ref_arc, np.uint8, 1024, O.parse_header(ref_arc)["codebook"][0]).copy() \
            if rank == 0 else None
        from paper_2105_12912_b200 import archive_io

        archive_io.write_sharded(res, path, lens.tobytes() if rank == 0 else None)
        got = D.gather_results(res)
        if rank == 0:
            q.put(D.assemble(got, lens.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("shape", [(32, 24, 40), (256, 100), (20000,)])
def test_sharded_rle_vle_archive_is_byte_identical(shape, world, tmp_path):
    """Auto selection picks RLE+VLE (long runs of the radius code); runs that
    cross slab boundaries are stitched so the archive equals the
    single-process one byte for byte."""
    import torch.multiprocessing as mp

    rng = np.random.default_rng(7)
    vals = np.zeros(int(np.prod(shape)), np.float32)
    # a few blocks of noise in a constant sea: long runs spanning slab boundaries
    for _ in range(3):
        a = int(rng.integers(0, vals.size - 10))
        vals[a: a + 10] = rng.normal(0, 1, 10).astype(np.float32)
    vals[0] = 4.0  # non-degenerate range
    eb = 1e-3
    dims = tuple(list(shape[::-1]) + [1] * (3 - len(shape))) + (len(shape),)
    ref = O.compress(vals, dims, float(vals.min()), float(vals.max()), eb)
    assert O.parse_header(ref)["workflow"] == 2  # RLE_VLE
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "sharded_rle.lzb")
    procs = [ctx.Process(target=_rle_worker, args=(r, world, port, (vals, shape, eb, ref, path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == ref
    with open(path, "rb") as fh:
        assert fh.read() == ref


def test_rle_stitch_plan_matches_global_runs():
    """Random streams with long runs (and a tiny max_run so splits and merged
    splits happen), cut into slabs at random points incl. empty and
    single-run slabs: local runs + the stitching plan == the global runs."""
    from paper_2105_12912_b200 import distributed as D

    rng = np.random.default_rng(11)
    for case in range(300):
        n = int(rng.integers(1, 400))
        vals = np.repeat(rng.integers(0, 3, 60), rng.integers(1, 40, 60))[:n].astype(np.uint32)
        n = len(vals)
        max_run = int(rng.choice([3, 7, 1000]))
        world = int(rng.integers(1, 6))
        cuts = np.sort(rng.integers(0, n + 1, world - 1))
        bounds = [0] + cuts.tolist() + [n]
        infos, local = [], []
        for k in range(world):
            sl = vals[bounds[k]: bounds[k + 1]]
            v, ln = O.rle_encode(sl, max_run) if len(sl) else (np.empty(0, np.uint32),) * 2
            local.append((v, ln))
            infos.append(D._boundary(v, ln, v, ln, len(v)) if len(v) else (0,) * 7)
        keep, group, emitted = D.plan_rle_stitch(infos, max_run)
        ev, el = [], []
        for k in range(world):
            v, ln = local[k]
            a, b = keep[k]
            ev += list(v[a:b])
            el += list(ln[a:b])
            if group[k] is not None:
                sp = D.split_run(group[k][1], max_run)
                ev += [group[k][0]] * len(sp)
                el += sp
            assert emitted[k] == (b - a) + (len(D.split_run(group[k][1], max_run)) if group[k] else 0)
        gv, gl = O.rle_encode(vals, max_run)
        assert ev == list(gv) and el == list(gl), case


def _override_worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import ChunkSpec, Dims, archive_io
        from paper_2105_12912_b200 import distributed as D

        vals, shape, eb, workflow, mode, ref_arc, path = case
        dims = Dims.of(*shape[::-1])
        chunk = ChunkSpec.default_for(dims.ndim)
        lo, hi = D.slab_bounds(dims, chunk, rank, world)
        full = vals.reshape(shape)
        slab = full[lo:hi].reshape(-1) if dims.ndim > 1 else full[lo:hi]
        res = D.compress_sharded(OracleSlabOps(), slab, dims, float(vals.min()), float(vals.max()),
                                 eb, "rel", 1024, chunk, 0, workflow=workflow, select_mode=mode)
        y = D.decompress_sharded(OracleSlabOps(), res)
        ref = O.decompress(ref_arc)[0].reshape(shape)
        want = ref[lo:hi].reshape(-1) if dims.ndim > 1 else ref[lo:hi]
        if hi > lo:
            assert y is not None and np.array_equal(y, want), rank
        h = O.parse_header(ref_arc)
        lens = np.frombuffer(ref_arc, np.uint8, h["codebook"][1], h["codebook"][0]).tobytes()
        archive_io.write_sharded(res, path, lens if rank == 0 else None)
        # every rank ends with the whole archive (one all-gather of the slices)
        whole = D.allgather_archive(res, lengths=lens).numpy().tobytes()
        assert whole == ref_arc, rank
        got = D.gather_results(res)
        if rank == 0:
            q.put((res.meta["workflow"], D.assemble(got, lens)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("workflow,mode,kind", [("rle", "exact", "runs"), ("rle", "exact", "smooth"),
                                                ("rlevle", "exact", "smooth"),
                                                ("huff", "exact", "runs"), (None, "estimate", "runs"),
                                                (None, "estimate", "smooth")])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_workflow_and_select_mode_overrides(workflow, mode, kind, world, tmp_path):
    """compress_sharded honours a forced workflow (RLE alone included) and the
    estimate selection mode: the archive (assembled, and written in parallel)
    is byte-identical to the single-process one with the same arguments
    (P/pipeline.py:135-182, T/test_acceptance.py:213-223)."""
    import torch.multiprocessing as mp

    from helpers import smooth

    shape = (24, 20, 36)
    if kind == "runs":
        rng = np.random.default_rng(5)
        vals = np.zeros(int(np.prod(shape)), np.float32)
        for _ in range(4):
            a = int(rng.integers(0, vals.size - 12))
            vals[a: a + 12] = rng.normal(0, 1, 12).astype(np.float32)
        vals[0], eb = 4.0, 1e-3
    else:
        vals, eb = smooth(shape).reshape(-1).astype(np.float32), 1e-4
    dims = tuple(list(shape[::-1]) + [1] * (3 - len(shape))) + (len(shape),)
    ref = O.compress(vals, dims, float(vals.min()), float(vals.max()), eb, workflow=workflow,
                     select_mode=mode)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "override.lzb")
    case = (vals, shape, eb, workflow, mode, ref, path)
    procs = [ctx.Process(target=_override_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    wf, got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ["HUFFMAN", "RLE", "RLE_VLE"].index(wf) == O.parse_header(ref)["workflow"]
    assert got == ref
    with open(path, "rb") as fh:
        assert fh.read() == ref
