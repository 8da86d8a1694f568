"""The reference's acceptance criteria (T/test_acceptance.py) run through this
package's public API on the GPU, at the reference's own scale:

  1  1,080 random fields x 3 workflows decode within the error bound
     (T/test_acceptance.py:57-80)
  5  a constant field selects RLE+VLE with CR > 32 (:165-173)
  6  every field at rel 1e-4 reaches PSNR >= 80 dB (:195-210)
  7  archives are identical across repeated calls / thread counts (:213-223)
  8  the three workflows decode to the same bits on 100 fields (:226-241)

Every archive is additionally byte-compared with the CPU oracle for a sample
of the fields (the oracle is the checker here, never the thing measured)."""

import itertools
import os

import numpy as np
import pytest

from helpers import make_array
from oracle import oracle as O

pytestmark = pytest.mark.gpu

BOUND_SLACK = 1 + 1e-12
KINDS = ["walk", "waves", "ramp", "noise", "spiky"]


def _lzb():
    import paper_2105_12912_b200 as lzb

    return lzb


def test_criterion_1_error_bound_1080_fields(cuda):
    lzb = _lzb()
    rng = np.random.default_rng(2024)
    runs = 0
    for rep, ndim, eb_rel, kind in itertools.product(range(8), (1, 2, 3), (1e-2, 1e-3, 1e-4), KINDS):
        f = lzb.Field.from_array(make_array(rng, ndim, kind=kind))
        for wf in ("huff", "rle", "rlevle"):
            blob = lzb.compress(f, eb_rel, workflow=wf)
            out = lzb.decompress(blob)
            eb_abs = lzb.parse_header(blob).eb_abs
            err = np.abs(f.values - out.values).max()
            assert err <= eb_abs * BOUND_SLACK, (ndim, eb_rel, kind, wf, err, eb_abs)
            if runs % 37 == 0:  # byte parity with the oracle on a spread of the cases
                d = f.dims
                assert blob == O.compress(f.values, d.as_tuple(), f.vmin, f.vmax, eb_rel, workflow=wf)
            runs += 1
    assert runs == 8 * 3 * 3 * 5 * 3


def test_criterion_5_constant_field_selects_rle_vle(cuda):
    lzb = _lzb()
    const = lzb.Field.from_array(np.full((48, 48, 48), 3.75, np.float32))
    blob = lzb.compress(const, 0.001, eb_mode="abs")
    assert lzb.parse_header(blob).workflow is lzb.Workflow.RLE_VLE
    assert const.nbytes / len(blob) > 32.0


def test_criterion_6_psnr_floor_at_rel_1e4(cuda):
    lzb = _lzb()
    rng = np.random.default_rng(666)
    for ndim, kind, dtype in itertools.product((1, 2, 3), KINDS, (np.float32, np.float64)):
        f = lzb.Field.from_array(make_array(rng, ndim, dtype=dtype, kind=kind))
        blob = lzb.compress(f, 1e-4)
        q = lzb.stats(f, lzb.decompress(blob), len(blob))
        assert q.psnr >= 80.0, (ndim, kind, dtype, q.psnr)


def test_criterion_7_deterministic_archives(cuda):
    lzb = _lzb()
    rng = np.random.default_rng(777)
    f = lzb.Field.from_array(make_array(rng, 3, kind="walk"))
    archives = {lzb.compress(f, 1e-3, threads=t) for t in (1, 4, os.cpu_count() or 8) for _ in range(3)}
    assert len(archives) == 1


def test_criterion_8_workflows_decode_identically(cuda):
    lzb = _lzb()
    rng = np.random.default_rng(888)
    for i in range(100):
        f = lzb.Field.from_array(make_array(rng, i % 3 + 1, dtype=np.float32 if i % 2 else np.float64))
        outs = [lzb.decompress(lzb.compress(f, 1e-3, workflow=wf)).values for wf in ("huff", "rle", "rlevle")]
        assert outs[0].dtype == outs[1].dtype == outs[2].dtype
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
