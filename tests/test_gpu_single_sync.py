"""GPU: the single-sync compress (K1 -> K2 -> K3 -> device archive assembly,
one read-back) and each way it hands over to the staged path -- RLE
selection, a code word over 32 bits, outlier capacity -- give the oracle's
archive byte for byte (P/pipeline.py:135-221)."""

import numpy as np
import pytest

from helpers import smooth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(vals, shape, eb, eb_mode="rel", **kw):
    import paper_2105_12912_b200 as lzb

    f = lzb.Field.from_array(vals.reshape(shape))
    dims = tuple(list(shape[::-1]) + [1] * (3 - len(shape))) + (len(shape),)
    blob = lzb.compress(f, eb, eb_mode=eb_mode, **kw)
    want = O.compress(np.ascontiguousarray(vals).reshape(-1), dims, f.vmin, f.vmax, eb, eb_mode=eb_mode, **kw)
    assert blob == want
    back = lzb.decompress(blob).values
    ref = O.decompress(want)[0]
    assert np.array_equal(np.asarray(back).reshape(-1).view(np.uint32), ref.reshape(-1).view(np.uint32))
    return lzb.parse_header(blob)


def test_single_sync_huffman_fields(cuda):
    for shape in [(60, 90, 70), (300, 500), (200_000,), (7,)]:
        vals = smooth(shape).astype(np.float32) if len(shape) > 1 or shape[0] > 8 else \
            np.arange(int(np.prod(shape)), dtype=np.float32)
        _check(vals, shape, 1e-4)


def test_hands_over_on_rle_selection(cuda):
    vals = np.zeros(64 * 64 * 64, np.float32)
    vals[:10] = np.arange(10)
    h = _check(vals, (64, 64, 64), 1e-2)
    assert h.workflow.name == "RLE_VLE"


def test_hands_over_on_outlier_capacity(cuda):
    rng = np.random.default_rng(3)
    vals = rng.normal(0, 1, 300 * 300).astype(np.float32)  # nearly every delta escapes the radius
    h = _check(vals, (300, 300), 1e-6, cap=64)
    assert h.outlier_count > 300 * 300 // 128 + 4096


def test_hands_over_on_code_words_over_32_bits(cuda):
    """Quant codes with Fibonacci counts give a code book deeper than 32 bits;
    the single-sync encoder (sized for 32) reports RETRY and the staged path
    encodes with the true maxlen."""
    fib = [1, 1]
    while len(fib) < 34:  # 14.9 M elements: inside the single-sync size limit
        fib.append(fib[-1] + fib[-2])
    deltas = np.repeat(np.arange(34) - 33, fib).astype(np.int64)  # the largest count on 0 (padding below)
    rng = np.random.default_rng(9)
    rng.shuffle(deltas)
    cx = 256  # the 1D default chunk: Lorenzo deltas restart at every chunk
    deltas = np.concatenate([deltas, np.zeros(-len(deltas) % cx, np.int64)])
    n = len(deltas)
    q = np.cumsum(deltas.reshape(-1, cx), axis=1).reshape(-1)  # chunk-local running sums
    vals = q.astype(np.float32)  # 2 * eb_abs = 1: the prequant codes are q itself
    h = _check(vals, (n,), 0.5, eb_mode="abs")
    assert h.workflow.name == "HUFFMAN"
    import paper_2105_12912_b200 as lzb  # the book really is deeper than 32
    f = lzb.Field.from_array(vals)
    arc = lzb.compress_device(f, 0.5, eb_mode="abs")
    assert arc.stream[2] > 32
