"""GPU: sharded compress through the device kernels (DeviceSlabOps), two
ranks on one GPU over gloo: the assembled archive equals the single-GPU
archive byte for byte, for every workflow (selected, forced, estimate mode),
the archive all-gathered from the slices is that archive on every rank, and
each rank's slab-local and stored-archive decompress equal its slab of the
single-GPU result."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_12912_b200 import ChunkSpec, Dims
        from paper_2105_12912_b200 import distributed as D

        vals, shape, eb, path, wf_arg, mode, ref = case
        dims = Dims.of(*shape[::-1])
        chunk = ChunkSpec.default_for(dims.ndim)
        lo, hi = D.slab_bounds(dims, chunk, rank, world)
        full = vals.reshape(shape)
        slab = torch.from_numpy(np.ascontiguousarray(full[lo:hi]).reshape(-1)).cuda()
        ops = D.DeviceSlabOps(torch.device("cuda"))
        res = D.compress_sharded(ops, slab, dims, float(vals.min()), float(vals.max()), eb, "rel",
                                 1024, chunk, 0, device=torch.device("cuda"), workflow=wf_arg,
                                 select_mode=mode)
        y = D.decompress_sharded(ops, res)
        # the stored archive on every rank from one all-gather of the slices,
        # then the stored-archive decompress (maps all-gather, symbol all-to-all)
        whole = D.allgather_archive(res, device=torch.device("cuda"))
        assert whole.is_cuda and whole.cpu().numpy().tobytes() == ref, rank
        ya, (alo, ahi), _ = D.decompress_archive_sharded(ops, whole)
        assert (alo, ahi) == (lo, hi) and torch.equal(ya, y), rank
        from paper_2105_12912_b200 import archive_io

        archive_io.write_sharded(res, path)  # each rank pwrites its parts
        lens = res.meta["lengths"].cpu().numpy().tobytes() if res.meta["lengths"] is not None else b""
        wf = res.meta["workflow"]
        got = D.gather_results(res)
        if rank == 0:
            q.put((D.assemble(got, lens), wf))
        q.put((rank, lo, hi, y.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _fields():
    from helpers import smooth

    yield "huffman", smooth((48, 40, 64)).reshape(-1).astype(np.float32), (48, 40, 64), 1e-4, None, "exact"
    rng = np.random.default_rng(5)
    v = np.zeros(64 * 48 * 40, np.float32)
    for _ in range(3):
        a = int(rng.integers(0, v.size - 10))
        v[a: a + 10] = rng.normal(0, 1, 10).astype(np.float32)
    v[0] = 4.0
    yield "rle_vle", v, (40, 48, 64), 1e-3, None, "exact"
    yield "rle_forced", v, (40, 48, 64), 1e-3, "rle", "exact"
    yield "rle_vle_estimate", v, (40, 48, 64), 1e-3, None, "estimate"
    yield "huffman_forced", v, (40, 48, 64), 1e-3, "huff", "exact"


_WANT = {"huffman": "HUFFMAN", "rle_vle": "RLE_VLE", "rle_forced": "RLE", "rle_vle_estimate": "RLE_VLE",
         "huffman_forced": "HUFFMAN"}


@pytest.mark.parametrize("name,vals,shape,eb,wf,mode", list(_fields()), ids=[f[0] for f in _fields()])
def test_sharded_compress_on_device(cuda, name, vals, shape, eb, wf, mode, tmp_path):
    import torch.multiprocessing as mp

    import paper_2105_12912_b200 as lzb

    field = lzb.Field.from_array(vals.reshape(shape))
    ref = lzb.compress(field, eb, workflow=wf, select_mode=mode)
    ref_y = np.asarray(lzb.decompress(ref).values).reshape(shape)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    path = str(tmp_path / "sharded.lzb")
    procs = [ctx.Process(target=_worker, args=(r, world, port, (vals, shape, eb, path, wf, mode, ref), q))
             for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    arc = [m for m in msgs if len(m) == 2][0]
    assert arc[1] == _WANT[name]
    assert arc[0] == ref
    with open(path, "rb") as fh:
        assert fh.read() == ref
    for rank, lo, hi, y in [m for m in msgs if len(m) == 4]:
        assert np.array_equal(y, ref_y[lo:hi].reshape(-1)), rank


def test_save_load_round_trip(cuda, tmp_path, monkeypatch):
    """Device archive -> file -> device through the pinned double buffers
    (small pieces so several are in flight)."""
    import torch

    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200 import archive_io
    from helpers import smooth

    monkeypatch.setattr(archive_io, "_PIECE", 1 << 14)
    vals = smooth((40, 48, 64)).astype(np.float32)
    field = lzb.Field.from_array(vals)
    arc = lzb.compress_device(field, 1e-4)
    path = str(tmp_path / "a.lzb")
    n = archive_io.save(arc, path)
    assert n == arc.nbytes and open(path, "rb").read() == lzb.compress(field, 1e-4)
    back = archive_io.load(path)
    assert torch.equal(back, arc.data[: arc.nbytes])
    y = lzb.decompress(back)
    assert np.array_equal(y.values.cpu().numpy(), lzb.decompress(lzb.compress(field, 1e-4)).values)
