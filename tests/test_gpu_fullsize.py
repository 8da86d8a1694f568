"""Whole-archive parity at the BASELINE configurations' full sizes
(BASELINE.json configs[0..3] = SURVEY 8 C1-C4): the CUDA path's archive must
equal the oracle's byte for byte, and the decoded field must equal the
oracle's decode bit for bit.  Inputs are the SURVEY 8(d) generators, built
once on the host and fed identically to both sides.

Reference behaviour pinned: P/pipeline.py:135-221 (archive assembly),
P/quantize.py:161-213, P/huffman.py:46-61, P/rle.py:17-35,
P/pipeline.py:318-326 (decode)."""

import os

import numpy as np
import pytest

from helpers import smooth, sparse
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1

CASES = {
    "C1": (lambda: smooth((100, 500, 500)), 1e-4, "HUFFMAN"),
    "C2": (lambda: smooth((1800, 3600)), 1e-4, "HUFFMAN"),
    "C3": (lambda: smooth((280_953_867,), ramp=False), 1e-4, "HUFFMAN"),
    "C4": (lambda: sparse((512, 512, 512)), 1e-2, "RLE_VLE"),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fullsize_archive_byte_identical(name, cuda):
    import torch

    import paper_2105_12912_b200 as lzb

    gen, eb, wf = CASES[name]
    vals = gen()
    f = lzb.Field.from_array(vals)
    d = f.dims
    ref = O.compress(f.values, d.as_tuple(), f.vmin, f.vmax, eb, threads=THREADS)
    # device-resident input (the bench's path) and host input give the same archive
    fd = lzb.Field(d, torch.from_numpy(f.values).to(cuda), f.vmin, f.vmax)
    arc = lzb.compress_device(fd, eb)
    assert arc.header.workflow.name == wf
    got = arc.to_bytes()
    assert len(got) == len(ref), (name, len(got), len(ref))
    if got != ref:
        a = np.frombuffer(got, np.uint8)
        b = np.frombuffer(ref, np.uint8)
        first = int(np.flatnonzero(a != b)[0])
        pytest.fail(f"{name}: archive differs from the oracle at byte {first} of {len(ref)}")
    # decode: device archive -> device field, bit for bit against the oracle's decode
    want = O.decompress(ref, threads=THREADS)[0]
    y, hdr, vmin, vmax = lzb.decompress_device(arc)
    yh = y.cpu().numpy()
    assert yh.dtype == want.dtype
    assert np.array_equal(yh.view(np.uint32), want.view(np.uint32)), name
    assert vmin == float(want.min()) and vmax == float(want.max())
    # and the error bound on every element (f32 output rounding slack as the reference tests)
    slack = float(np.spacing(np.float32(max(abs(f.vmin), abs(f.vmax))))) / 2
    err = np.abs(vals.reshape(-1).astype(np.float64) - yh.astype(np.float64)).max()
    assert err <= hdr.eb_abs * (1 + 1e-12) + slack
