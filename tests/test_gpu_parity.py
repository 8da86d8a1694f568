"""GPU parity: the CUDA path (through the C ABI) against the reference-pinned
oracle and the reference's own golden archives.  Integer/byte work must be
bit-exact; decoded floats are compared bit for bit as well (the dequant is the
reference's f64 multiply + RN cast)."""

import hashlib
import struct

import numpy as np
import pytest

from helpers import dims_of, golden_case, make_array, smooth, sparse
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _lzb():
    import paper_2105_12912_b200 as lzb

    return lzb


def _field(vals, dims, vmin=None, vmax=None):
    lzb = _lzb()
    d = lzb.Dims(*dims[:3], ndim=dims[3])
    if vmin is None:
        vmin, vmax = float(vals.min()), float(vals.max())
    return lzb.Field(d, np.ascontiguousarray(vals).reshape(-1), vmin, vmax)


def _kw(kw):
    lzb = _lzb()
    out = dict(kw)
    if "chunk" in out:
        out["chunk"] = lzb.ChunkSpec(*out["chunk"])
    return out


def test_golden_archives_byte_identical(golden, cuda):
    index, _, _ = golden
    for i in range(len(index)):
        c, vals, dims, kw, arc = golden_case(golden, i)
        got = _lzb().compress(_field(vals, dims, c["vmin"], c["vmax"]), **_kw(kw))
        assert got == arc, c["name"]


def test_golden_archives_decode_identically(golden, cuda):
    index, _, _ = golden
    for i in range(len(index)):
        c, vals, dims, kw, arc = golden_case(golden, i)
        out = _lzb().decompress(arc)
        assert hashlib.sha256(out.values.tobytes()).hexdigest() == c["decoded_sha256"], c["name"]
        assert out.values.dtype == vals.dtype


def test_device_resident_field_matches(golden, cuda):
    import torch

    lzb = _lzb()
    index, _, _ = golden
    for i in range(0, len(index), 7):
        c, vals, dims, kw, arc = golden_case(golden, i)
        t = torch.from_numpy(np.ascontiguousarray(vals)).to(cuda)
        f = lzb.Field(lzb.Dims(*dims[:3], ndim=dims[3]), t, c["vmin"], c["vmax"])
        da = lzb.compress_device(f, **_kw(kw))
        assert da.to_bytes() == arc, c["name"]
        y, hdr, vmin, vmax = lzb.decompress_device(da.data)
        want = O.decompress(arc)[0]
        assert np.array_equal(y.cpu().numpy(), want), c["name"]
        # the DeviceArchive itself (header + stream facts already on the host)
        y2, hdr2, vmin2, vmax2 = lzb.decompress_device(da)
        assert np.array_equal(y2.cpu().numpy(), want) and (vmin2, vmax2) == (vmin, vmax), c["name"]


@pytest.mark.parametrize("ndim", [1, 2, 3])
def test_random_fields_match_oracle(ndim, cuda):
    lzb = _lzb()
    rng = np.random.default_rng(100 + ndim)
    specs = {1: [None, (7, 1, 1), (1000, 1, 1)], 2: [None, (8, 8, 1), (5, 3, 1)],
             3: [None, (4, 4, 2), (3, 5, 7), (16, 16, 16)]}[ndim]
    for rep in range(12):
        dt = np.float32 if rep % 2 else np.float64
        a = make_array(rng, ndim, dt)
        d = dims_of(a)
        f = _field(a.reshape(-1), d)
        wf = [None, "huff", "rle", "rlevle"][rep % 4]
        spec = specs[rep % len(specs)]
        eb = [1e-2, 1e-3, 1e-4, 1e-6][rep % 4]
        cap = [1024, 64, 4, 4096][(rep // 3) % 4]
        kw = dict(eb=eb, workflow=wf, cap=cap)
        ref = O.compress(f.values, d, f.vmin, f.vmax, chunk=spec, **kw)
        got = lzb.compress(f, chunk=lzb.ChunkSpec(*spec) if spec else None, **kw)
        assert got == ref, (ndim, rep, kw, spec)
        out = lzb.decompress(got)
        assert np.array_equal(out.values, O.decompress(ref)[0]), (ndim, rep)
        h = lzb.parse_header(got)
        slack = float(np.spacing(np.float32(max(abs(f.vmin), abs(f.vmax))))) / 2 \
            if dt == np.float32 else 0.0
        err = np.abs(f.values.astype(np.float64) - out.values.astype(np.float64)).max()
        assert err <= h.eb_abs * (1 + 1e-12) + slack


def test_survey_generators_match_oracle(cuda):
    lzb = _lzb()
    for vals, eb in ((smooth((60, 90, 70)), 1e-4), (smooth((300, 500)), 1e-4),
                     (smooth((200_000,), ramp=False), 1e-4), (sparse((64, 64, 64)), 1e-2)):
        f = lzb.Field.from_array(vals)
        d = f.dims
        ref = O.compress(f.values, d.as_tuple(), f.vmin, f.vmax, eb)
        got = lzb.compress(f, eb)
        assert got == ref
        assert np.array_equal(lzb.decompress(got).values, O.decompress(ref)[0])


def test_estimate_mode_and_abs_mode(cuda):
    lzb = _lzb()
    rng = np.random.default_rng(7)
    for k in range(6):
        a = make_array(rng, 1 + k % 3)
        d = dims_of(a)
        f = _field(a.reshape(-1), d)
        for kw in (dict(eb=1e-3, select_mode="estimate"), dict(eb=0.25, eb_mode="abs")):
            assert lzb.compress(f, **kw) == O.compress(f.values, d, f.vmin, f.vmax, **kw)


def test_tiny_and_edge_grids(cuda):
    lzb = _lzb()
    for cnt in (1, 2, 3):
        f = lzb.Field.from_array(np.linspace(5, 6, cnt))
        blob = lzb.compress(f, 0.01, eb_mode="abs")
        assert blob == O.compress(f.values, (cnt, 1, 1, 1), f.vmin, f.vmax, 0.01, eb_mode="abs")
        g = lzb.decompress(blob)
        assert np.abs(f.values - g.values).max() <= 0.01 * (1 + 1e-12)
    const = lzb.Field.from_array(np.full((24, 24, 24), 3.75, np.float32))
    blob = lzb.compress(const, 0.001, eb_mode="abs")
    assert lzb.parse_header(blob).workflow is lzb.Workflow.RLE_VLE
    assert blob == O.compress(const.values, (24, 24, 24, 3), 3.75, 3.75, 0.001, eb_mode="abs")
    row = lzb.Field.from_array(np.cumsum(np.random.default_rng(1).normal(size=(1, 333)), axis=-1))
    assert lzb.compress(row, 1e-3) == O.compress(row.values, (333, 1, 1, 2), row.vmin, row.vmax, 1e-3)
    heavy = lzb.Field.from_array(np.random.default_rng(61).normal(scale=1e6, size=2048))
    blob = lzb.compress(heavy, 1e-7)
    assert lzb.parse_header(blob).outlier_count > 0
    assert blob == O.compress(heavy.values, (2048, 1, 1, 1), heavy.vmin, heavy.vmax, 1e-7)


def test_outlier_order_nonorigin(cuda):
    """Noise fields put outliers everywhere in a chunk: exercises the device
    reorder from chunk-major to global row-major order."""
    lzb = _lzb()
    rng = np.random.default_rng(11)
    for shape, spec in (((33, 47, 29), None), ((130, 70), None), ((20, 17, 9), (4, 4, 2)),
                        ((9, 40), (8, 8, 1))):
        a = rng.normal(scale=1000, size=shape)
        f = lzb.Field.from_array(a)
        d = f.dims
        cs = lzb.ChunkSpec(*spec) if spec else None
        ref = O.compress(f.values, d.as_tuple(), f.vmin, f.vmax, 1e-5, cap=16, chunk=spec)
        got = lzb.compress(f, 1e-5, cap=16, chunk=cs)
        assert lzb.parse_header(got).outlier_count > 100
        assert got == ref
        assert np.array_equal(lzb.decompress(got).values, O.decompress(ref)[0])


def test_validation_errors(cuda):
    lzb = _lzb()
    f = lzb.Field.from_array(np.full(100, 7.0))
    with pytest.raises(lzb.DataError, match="absolute"):
        lzb.compress(f, 1e-3)
    assert lzb.decompress(lzb.compress(f, 0.5, eb_mode="abs")).values[0] == 7.0
    w = lzb.Field.from_array(np.sin(np.linspace(0, 9, 96 * 80).reshape(80, 96) * 3) * 40)
    for bad in (0.0, -1.0, float("nan")):
        with pytest.raises(lzb.DataError):
            lzb.compress(w, bad)
    with pytest.raises(lzb.DataError):
        lzb.compress(w, 1e-3, workflow="zip")
    with pytest.raises(lzb.QuantOverflowError):
        lzb.compress(lzb.Field.from_array(np.array([1e18, 0.0])), 1e-4, eb_mode="abs")


def test_corruption_raises(cuda):
    lzb = _lzb()
    x = np.linspace(0, 9, 96 * 80).reshape(80, 96)
    w = lzb.Field.from_array(np.sin(x * 3) * 40 + x)
    for wf in ("huff", "rle", "rlevle"):
        blob = lzb.compress(w, 1e-2, workflow=wf)
        hdr = lzb.parse_header(blob)
        for cut in (0, 10, 129, hdr.codebook[0] + 5, hdr.symbols[0] + 3, len(blob) - 1):
            with pytest.raises(lzb.CorruptArchiveError):
                lzb.decompress(blob[:cut])
    blob = bytearray(lzb.compress(w, 1e-2))
    blob[0] ^= 0xFF
    with pytest.raises(lzb.CorruptArchiveError, match="magic"):
        lzb.decompress(bytes(blob))
    blob = bytearray(lzb.compress(w, 1e-2))
    struct.pack_into("<H", blob, 8, 99)
    with pytest.raises(lzb.CorruptArchiveError, match="version"):
        lzb.decompress(bytes(blob))
    blob = bytearray(lzb.compress(w, 1e-2, workflow="huff"))
    hdr = lzb.parse_header(bytes(blob))
    struct.pack_into("<Q", blob, hdr.symbols[0] + 8, hdr.count + 1)
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.decompress(bytes(blob))
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.decompress(b"not an archive at all")
    # flipped payload bits must either raise or decode like the oracle does
    good = lzb.compress(w, 1e-3, workflow="huff")
    hdr = lzb.parse_header(good)
    rng = np.random.default_rng(5)
    for _ in range(20):
        bad = bytearray(good)
        pos = hdr.symbols[0] + 16 + int(rng.integers(0, hdr.symbols[1] - 16))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            want = O.decompress(bytes(bad))[0]
        except (O.CorruptArchiveError, O.DataError, O.QuantOverflowError) as e:
            with pytest.raises((lzb.CorruptArchiveError, lzb.DataError)):
                lzb.decompress(bytes(bad))
            continue
        assert np.array_equal(lzb.decompress(bytes(bad)).values, want)
    # outlier list tampering
    blob = bytearray(lzb.compress(lzb.Field.from_array(np.random.default_rng(2).normal(
        scale=1e6, size=4096)), 1e-7))
    hdr = lzb.parse_header(bytes(blob))
    o = hdr.outliers[0]
    struct.pack_into("<Q", blob, o + 16, struct.unpack_from("<Q", blob, o)[0])  # duplicate index
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.decompress(bytes(blob))


def test_tma_tile_path_3d(cuda):
    """ChunkSpec(8,8,8) f32 grids whose chunk rows hold whole 16-chunk super
    tiles (nx a multiple of 128) take K1's TMA path (others the cp.async one): smooth, noisy (non-origin and
    > 4-per-chunk outliers), partial y/z chunk layers, values on exact rounding
    ties and values too large for the int32 fast path -- all byte-identical to
    the oracle."""
    lzb = _lzb()
    rng = np.random.default_rng(64)
    cases = []
    cases.append((smooth((24, 32, 128)), dict(eb=1e-4)))
    cases.append((smooth((21, 19, 64)), dict(eb=1e-3)))                        # partial y/z chunks
    cases.append((smooth((21, 19, 256)), dict(eb=1e-3)))
    noisy = (rng.standard_normal((16, 16, 256)) * 50).astype(np.float32)
    cases.append((noisy, dict(eb=1e-4, cap=64)))                               # many outliers
    cases.append((noisy, dict(eb=1e-2, cap=4)))
    # a wide code distribution at cap 1024: many codes outside the u8 code
    # stream's byte window (escapes, include/lzb.h) in K1 -> K3
    cases.append(((rng.standard_normal((16, 8, 128)) * 3).cumsum(axis=2).astype(np.float32), dict(eb=2e-4)))
    cases.append((noisy, dict(eb=3e-4, cap=2048)))
    ties = (np.round(rng.uniform(-300, 300, (8, 8, 128))) + 0.5).astype(np.float32) * np.float32(0.5)
    cases.append((ties, dict(eb=0.25, eb_mode="abs")))                         # x / (2 eb) on a .5 tie
    big = smooth((16, 8, 128)) * np.float32(1e4)
    cases.append((big, dict(eb=1e-9, eb_mode="abs", cap=1024)))                # |q| >= 2^22: exact path
    for vals, kw in cases:
        f = lzb.Field.from_array(vals)
        d = f.dims
        try:
            ref = O.compress(f.values, d.as_tuple(), f.vmin, f.vmax, **kw)
        except Exception as ex:  # the reference raises (e.g. overflow): so must we
            with pytest.raises(Exception) as ei:
                lzb.compress(f, **kw)
            assert type(ei.value).__name__ == type(ex).__name__
            continue
        got = lzb.compress(f, **kw)
        assert got == ref, (vals.shape, kw)
        assert np.array_equal(lzb.decompress(got).values, O.decompress(ref)[0])
