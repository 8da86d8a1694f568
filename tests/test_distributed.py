"""CPU, world_size 2 over gloo: the sharded-compress host logic (slab
bounds, histogram all-reduce, code book, bit/outlier all-gather, bit-phase
slices, OR-merge assembly) reproduces the single-device archive byte for
byte.  The per-rank compute is a CPU stand-in built on the oracle (test
infrastructure); production uses DeviceSlabOps (the CUDA kernels)."""

import os
import socket

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

    def encode_at(self, codes, n, lengths, words, cap, maxlen, phase, bits):
        b, _, data = O.huff_encode(codes, lengths, words)
        assert b == bits
        arr = np.unpackbits(np.frombuffer(data, np.uint8))[:bits]
        arr = np.concatenate([np.zeros(phase, np.uint8), arr])
        return np.packbits(arr)

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


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import ChunkSpec, Dims
        from paper_2105_12912_b200 import distributed as D

        vals, shape, eb = case
        dims = Dims.of(*shape[::-1])
        chunk = ChunkSpec.default_for(dims.ndim)
        lo, hi = D.slab_bounds(dims, chunk, rank, world)
        full = vals.reshape(shape)
        slab = full[lo:hi].reshape(-1) if dims.ndim > 1 else full[lo:hi]
        res = D.compress_sharded(OracleSlabOps(), slab, dims, float(vals.min()),
                                 float(vals.max()), eb, "rel", 1024, chunk, 0)
        # slab-local decompress of the rank's own slice == that slab of the
        # single-device decompress
        y = D.decompress_sharded(OracleSlabOps(), res)
        ref = O.decompress(O.compress(vals, dims.as_tuple(), float(vals.min()), float(vals.max()),
                                      eb))[0].reshape(shape)
        want = ref[lo:hi].reshape(-1) if dims.ndim > 1 else ref[lo:hi]
        assert y is not None and np.array_equal(y, want), rank
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


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("shape", [(40, 30, 36), (300, 257), (70001,)])
def test_sharded_archive_is_byte_identical(shape, world):
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
    procs = [ctx.Process(target=_worker, args=(r, world, port, (vals, shape, eb), q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == ref


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
