"""Block-by-block compression / decompression: the
archive of a field compressed slab by slab equals the whole-field archive
byte for byte, for every workflow, any number of slabs; decoding slab by slab
gives the whole-field decompress.  CPU: the slab ops are the oracle stand-in
(the same host logic as on the GPU); GPU: the device kernels."""

import numpy as np
import pytest

from helpers import smooth
from oracle import oracle as O
from test_distributed import OracleSlabOps


def _dims(shape):
    from paper_2105_12912_b200 import Dims

    return Dims.of(*shape[::-1])


def _fields():
    rng = np.random.default_rng(12)
    yield "smooth3d", smooth((40, 24, 32)).astype(np.float32), 1e-4, {}
    yield "smooth2d", smooth((100, 70)).astype(np.float64), 1e-4, {}
    yield "smooth1d", smooth((30000,)).astype(np.float32), 1e-4, {}
    runs = np.zeros((48, 16, 16), np.float32)
    for _ in range(4):
        a = int(rng.integers(0, runs.size - 12))
        runs.reshape(-1)[a: a + 12] = rng.normal(0, 1, 12)
    runs.reshape(-1)[0] = 4.0
    yield "rle_vle", runs, 1e-3, {}
    yield "rle", runs, 1e-3, dict(workflow="rle")
    yield "estimate", runs, 1e-3, dict(select_mode="estimate")
    noisy = (rng.standard_normal((20, 16, 24)) * 30).astype(np.float32)
    yield "outliers", noisy, 1e-4, dict(cap=64)


@pytest.mark.parametrize("name,vals,eb,kw", list(_fields()), ids=[f[0] for f in _fields()])
@pytest.mark.parametrize("blocks", [1, 3, 7])
def test_blocks_equal_whole_field(name, vals, eb, kw, blocks):
    from paper_2105_12912_b200 import outofcore as X

    shape = vals.shape
    d = _dims(shape)
    dims = d.as_tuple()
    want = O.compress(vals.reshape(-1), dims, float(vals.min()), float(vals.max()), eb, **kw)
    got = X.compress_blocks(vals, d, eb, block_bytes=-(-vals.nbytes // blocks), ops=OracleSlabOps(), **kw)
    assert got == want
    back = X.decompress_blocks(want, block_bytes=-(-vals.nbytes // blocks), ops=OracleSlabOps())
    ref = O.decompress(want)[0].reshape(-1)
    assert back.dtype == ref.dtype and np.array_equal(back.view(np.uint8), ref.view(np.uint8))


def test_blocks_reject_non_finite():
    from paper_2105_12912_b200 import DataError
    from paper_2105_12912_b200 import outofcore as X

    v = smooth((16, 16, 16)).astype(np.float32)
    v[5, 5, 5] = np.nan
    with pytest.raises(DataError):
        X.compress_blocks(v, _dims(v.shape), 1e-3, ops=OracleSlabOps())


@pytest.mark.gpu
@pytest.mark.parametrize("name,vals,eb,kw", list(_fields()), ids=[f[0] for f in _fields()])
def test_blocks_on_device(cuda, name, vals, eb, kw, tmp_path):
    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200 import outofcore as X

    d = _dims(vals.shape)
    want = lzb.compress(lzb.Field.from_array(vals), eb, **kw)
    got = X.compress_blocks(vals, d, eb, block_bytes=-(-vals.nbytes // 5), **kw)
    assert got == want
    # a memory-mapped raw file, decoded slab by slab into another
    out = np.lib.format.open_memmap(str(tmp_path / "y.npy"), mode="w+", dtype=vals.dtype, shape=(vals.size,))
    X.decompress_blocks(want, out=out, block_bytes=-(-vals.nbytes // 5))
    ref = np.asarray(lzb.decompress(want).values).reshape(-1)
    assert np.array_equal(np.asarray(out).view(np.uint8), ref.view(np.uint8))
