"""GPU stage parity: each C-ABI stage against the oracle / reference KATs."""

import itertools

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_codebook_matches_reference_lengths(golden, cuda):
    import paper_2105_12912_b200 as lzb

    _, _, k = golden
    for h, want in zip(k["random_histograms"], k["random_lengths"]):
        book = lzb.Codebook.from_counts(np.array(h, np.int64))
        assert book.lengths.tolist() == want
        assert [int(v) for v in book.codes] == [int(v) for v in O.canonical_codes(
            np.array(want, np.uint8))]


def test_codebook_random_books_vs_oracle(cuda):
    """K2's two-queue merge (32-bit and 64-bit weight windows) against the
    oracle's heap construction (P/codebook.py:143-176) on histograms built to
    stress the tie rules: equal counts, runs of ones, geometric tails, a lone
    symbol, totals across 2^32."""
    import paper_2105_12912_b200 as lzb

    rng = np.random.default_rng(1234)
    cases = []
    for cap in (2, 16, 64, 1024, 4096):
        for kind in range(6):
            h = np.zeros(cap, np.int64)
            k = int(rng.integers(1, cap + 1))
            idx = rng.choice(cap, k, replace=False)
            if kind == 0:
                h[idx] = 1                                   # all ties
            elif kind == 1:
                h[idx] = rng.integers(1, 4, k)               # few distinct weights
            elif kind == 2:
                h[idx] = (2.0 ** -np.abs(rng.normal(0, 4, k)) * 1e6).astype(np.int64) + 1
            elif kind == 3:
                h[idx] = rng.integers(1, 1 << 40, k)         # total far above 2^32
            elif kind == 4:
                h[idx] = np.sort(rng.integers(1, 1 << 12, k))[::-1]
            else:
                h[idx[:1]] = int(rng.integers(1, 1 << 30))   # lone symbol
            cases.append(h)
    for _ in range(60):  # centred quant-code-like books at cap 1024
        h = np.zeros(1024, np.int64)
        w = int(rng.integers(2, 400))
        c = np.arange(512 - w, 512 + w)
        h[c] = (np.exp(-((c - 512) / (w / rng.uniform(2, 8))) ** 2) * 10 ** rng.uniform(2, 9)).astype(np.int64)
        h[rng.integers(0, 1024, 5)] += 1
        cases.append(h)
    for h in cases:
        book = lzb.Codebook.from_counts(h)
        want = O.huffman_lengths(h)
        assert book.lengths.tolist() == want.tolist(), (len(h), int((h > 0).sum()), int(h.sum()))


def test_codebook_kats(golden, cuda):
    import paper_2105_12912_b200 as lzb

    _, _, k = golden
    for key, val in k.items():
        if key.startswith("book_"):
            counts = np.array([int(v) for v in key[5:].split("_")], np.int64)
            b = lzb.Codebook.from_counts(counts)
            assert b.lengths.tolist() == val[0]
            assert [int(v) for v in b.codes] == val[1]
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.Codebook.from_lengths(bytes([1, 2, 0, 0, 0, 0, 0, 0]))
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.Codebook.from_lengths(bytes([65, 0, 0, 0]))
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.Codebook.from_lengths(bytes(16))
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.Codebook.from_lengths(bytes([0, 0, 3, 0]))


def test_huffman_round_trips_and_bits(golden, cuda):
    import paper_2105_12912_b200 as lzb

    _, _, k = golden
    book = lzb.Codebook.from_counts(np.array([2, 1, 1], np.int64))
    s = lzb.encode(np.array([0, 1, 2], np.uint32), book)
    assert [s.bit_len, s.count, s.data.tolist()] == k["encode_012"]
    rng = np.random.default_rng(444)
    for _ in range(150):
        nsym = int(rng.integers(1, 64))
        cap = int(rng.choice([64, 256, 1024]))
        stream = rng.integers(0, nsym, size=int(rng.integers(1, 20000))).astype(np.uint32)
        counts = np.bincount(stream, minlength=cap)
        book = lzb.Codebook.from_counts(counts)
        bs = lzb.encode(stream, book)
        ob, oc, od = O.huff_encode(stream, book.lengths, book.codes)
        assert bs.bit_len == ob and bs.data.tobytes() == od
        assert np.array_equal(lzb.decode(bs, book), stream)
    deep = lzb.Codebook.from_counts(np.array([2 ** i for i in range(12, 0, -1)], np.int64))
    stream = np.full(1000, 11, np.uint32)
    assert np.array_equal(lzb.decode(lzb.encode(stream, deep), deep), stream)
    # 40-bit-deep code words (Fibonacci counts)
    fib = [1, 1]
    while len(fib) < 42:
        fib.append(fib[-1] + fib[-2])
    book = lzb.Codebook.from_counts(np.array(fib, np.int64))
    assert book.max_len > 32
    stream = rng.integers(0, 42, size=5000).astype(np.uint32)
    bs = lzb.encode(stream, book)
    assert bs.data.tobytes() == O.huff_encode(stream, book.lengths, book.codes)[2]
    assert np.array_equal(lzb.decode(bs, book), stream)


def test_huffman_non_synchronising_books(cuda):
    """Fixed-length and near-fixed-length codes never self-synchronise: the
    transfer-map composition must still find every boundary."""
    import paper_2105_12912_b200 as lzb

    rng = np.random.default_rng(9)
    for counts in (np.full(1024, 7, np.int64), np.full(16, 3, np.int64),
                   rng.integers(900, 1100, 1024).astype(np.int64)):
        book = lzb.Codebook.from_counts(counts)
        stream = rng.integers(0, len(counts), size=300_000).astype(np.uint32)
        bs = lzb.encode(stream, book)
        assert np.array_equal(lzb.decode(bs, book), stream)


def test_decode_rejects_bad_streams(cuda):
    import paper_2105_12912_b200 as lzb

    book = lzb.Codebook.from_counts(np.array([4, 3, 2, 1], np.int64))
    s = lzb.encode(np.array([0, 1, 2, 3], np.uint32), book)
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.decode(lzb.BitStream(s.bit_len - 1, s.count, s.data), book)
    b2 = lzb.Codebook.from_counts(np.array([4, 3], np.int64))
    s = lzb.encode(np.array([0, 1, 0], np.uint32), b2)
    for c in (s.count + 1, s.count - 1):
        with pytest.raises(lzb.CorruptArchiveError):
            lzb.decode(lzb.BitStream(s.bit_len, c, s.data), b2)
    one = lzb.Codebook.from_counts(np.array([1], np.int64))
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.decode(lzb.BitStream(3, 0, np.array([0], np.uint8)), one)
    with pytest.raises(lzb.DataError):
        lzb.encode(np.array([1], np.uint32), lzb.Codebook.from_counts(np.array([1, 0], np.int64)))


def test_rle_stage(golden, cuda):
    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200 import rle

    _, _, k = golden
    v, ln = lzb.run_length_encode(np.array([0, 0, 1, 2, 2, 2, 2, 2, 0, 0], np.uint32))
    assert [v.tolist(), ln.tolist()] == k["rle_textbook"]
    rng = np.random.default_rng(14)
    for _ in range(60):
        s = rng.integers(0, 3, int(rng.integers(1, 50000))).astype(np.uint32)
        v, ln = lzb.run_length_encode(s)
        ov, ol = O.rle_encode(s)
        assert np.array_equal(v, ov) and np.array_equal(ln, ol)
        assert np.array_equal(lzb.run_length_decode(v, ln), s)
    old = rle._MAX_RUN
    try:
        rle._MAX_RUN = 4
        s = np.array([5] * 10 + [3] + [5] * 4, np.uint32)
        v, ln = rle.run_length_encode(s)
        assert v.tolist() == [5, 5, 5, 3, 5] and ln.tolist() == [4, 4, 2, 1, 4]
    finally:
        rle._MAX_RUN = old
    with pytest.raises(lzb.CorruptArchiveError):
        lzb.run_length_decode(np.array([1], np.uint32), np.array([0], np.uint32))


def test_count_runs(cuda):
    import torch
    from paper_2105_12912_b200 import _native as N

    L = N.lib()
    rng = np.random.default_rng(15)
    st = torch.zeros(N.STATUS_BYTES, dtype=torch.uint8, device="cuda")
    for n in [1, 7, 8, 9, 4095, 4096, 100003]:
        for dt, cb in [(np.uint16, 2), (np.uint32, 4)]:
            s = rng.integers(0, 3, n).astype(dt)
            s[: n // 3] = 1  # a long run at the start
            d = torch.from_numpy(s.view(np.uint8).copy()).cuda()
            N.check_rc(L.lzb_count_runs(d.data_ptr(), cb, n, st.data_ptr(), N.stream_ptr()), "count_runs")
            (sr,) = N.read_status(st)
            assert sr.code == 0 and sr.u[0] == len(O.rle_encode(s.astype(np.uint32))[0]), (n, cb)


def test_quantize_stage_kats(golden, cuda):
    import paper_2105_12912_b200 as lzb

    _, _, k = golden
    F = lzb.Field.from_array
    assert lzb.quantize.prequantize(F(np.array([1.0, 0.029, -0.03, 0.0])),
                                    lzb.QuantConfig(0.01)).codes.tolist() == k["prequant_eb001"]
    assert lzb.quantize.prequantize(F(np.array([0.5, -0.5, 1.5, -1.5, 2.5])),
                                    lzb.QuantConfig(0.5)).codes.tolist() == k["prequant_ties"]
    pq = lzb.PrequantGrid(lzb.Dims.of(4), np.array([0, 5, 5, 6], np.int64))
    q, o = lzb.quantize.construct_grid(pq, lzb.QuantConfig(0.1, 4), lzb.ChunkSpec(4))
    assert [q.codes.tolist(), o.indices.tolist(), o.deltas.tolist()] == k["cap4_outlier"]
    q, o = lzb.quantize.construct_grid(lzb.PrequantGrid(lzb.Dims.of(1), np.array([123])),
                                       lzb.QuantConfig(0.5, 1024), lzb.ChunkSpec(256))
    assert q.codes.tolist() == [635] and len(o) == 0
    got = lzb.dequantize(lzb.PrequantGrid(lzb.Dims.of(3), np.array([-1, 0, 50])),
                         lzb.QuantConfig(0.01), "f64")
    assert got.values.tolist() == k["dequant"]


def test_partial_sum_equals_sequential_exhaustive_1d(cuda):
    """Acceptance 2 (P tests/test_acceptance.py:83-118) on the device: every
    {-1,0,1} delta sequence up to length 8 reconstructs like the oracle."""
    import paper_2105_12912_b200 as lzb

    cfg = lzb.QuantConfig(0.5, 4)
    seqs = [np.array(d, np.int64) for L in range(1, 9) for d in itertools.product((-1, 0, 1),
                                                                                  repeat=L)]
    # pack every sequence as one chunk of a long 1D grid with chunk edge 8 (pad with zeros)
    n = 8 * len(seqs)
    deltas = np.zeros(n, np.int64)
    for i, d in enumerate(seqs):
        deltas[8 * i: 8 * i + len(d)] = d
    quant = lzb.QuantGrid(lzb.Dims.of(n), (deltas + cfg.radius).astype(np.uint32))
    got = lzb.reconstruct_grid(quant, lzb.OutlierList.empty(), cfg, lzb.ChunkSpec(8)).codes
    want = np.cumsum(deltas.reshape(-1, 8), axis=1).reshape(-1)
    assert np.array_equal(got, want)


def test_partial_sum_random_2d_3d_with_outliers(cuda):
    import paper_2105_12912_b200 as lzb

    rng = np.random.default_rng(77)
    for i in range(40):
        ndim = 2 if i % 2 else 3
        shape = tuple(int(n) for n in rng.integers(1, 40, 3))
        if ndim == 2:
            shape = (1,) + shape[1:]
        pre = rng.integers(-10_000, 10_000, size=shape).astype(np.int64)
        dims = lzb.Dims(shape[2], shape[1], shape[0], ndim=ndim) if ndim == 3 else \
            lzb.Dims(shape[2], shape[1], ndim=2)
        spec = lzb.ChunkSpec(*[int(v) for v in rng.integers(1, 9, 3)])
        cfg = lzb.QuantConfig(0.5, 64)
        q, o = lzb.quantize.construct_grid(lzb.PrequantGrid(dims, pre.reshape(-1)), cfg, spec)
        back = lzb.reconstruct_grid(q, o, cfg, spec)
        assert np.array_equal(back.codes, pre.reshape(-1))


def test_huffman_decode_layouts(cuda):
    """Streams whose lengths straddle the decoder's 128-bit microblocks and
    4096-bit subsequences, smooth-like (geometric), slowly synchronising
    (near-uniform, ~8 bits) and deep (> 12-bit code words) books, u16 and u32
    symbols -- every decode equals the encoded stream."""
    import paper_2105_12912_b200 as lzb

    rng = np.random.default_rng(2026)
    books = []
    g = np.array([int(1e6 * 0.55 ** abs(i - 512)) + 1 for i in range(1024)], np.int64)
    books.append(g)                                                   # smooth, ~2 bits
    books.append(rng.integers(50, 200, 300).astype(np.int64))        # ~8 bits, slow sync
    books.append(np.array([2 ** (20 - i // 3) for i in range(60)], np.int64))  # deep
    books.append(np.array([1000, 1], np.int64))                      # 1-bit codes
    for counts in books:
        p = counts / counts.sum()
        book = lzb.Codebook.from_counts(counts)
        for n in (1, 2, 63, 64, 65, 2047, 2048, 2049, 4095, 4096, 4097, 40000, 250_000):
            stream = rng.choice(len(counts), size=n, p=p).astype(np.uint32)
            bk = lzb.Codebook.from_counts(np.bincount(stream, minlength=len(counts)))
            bs = lzb.encode(stream, bk)
            assert np.array_equal(lzb.decode(bs, bk), stream), (len(counts), n)
    # u32 symbols (cap > 65536)
    cap = 1 << 17
    stream = (rng.geometric(0.3, 100_000) + 70000).astype(np.uint32) % cap
    bk = lzb.Codebook.from_counts(np.bincount(stream, minlength=cap))
    assert np.array_equal(lzb.decode(lzb.encode(stream, bk), bk), stream)


def test_decode_at_bit_phase(cuda):
    """lzb_huff_decode_at (the multi-GPU slab decode) on streams whose first
    bit is bit 0..7 of the first byte -- the slices lzb_huff_encode_at writes."""
    import torch

    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200 import _native as N

    L = N.lib()
    rng = np.random.default_rng(77)
    g = np.array([int(1e6 * 0.5 ** abs(i - 32)) + 1 for i in range(64)], np.int64)
    for n in (1, 5000, 70_000):
        stream = rng.choice(64, size=n, p=g / g.sum()).astype(np.uint32)
        bk = lzb.Codebook.from_counts(np.bincount(stream, minlength=64))
        bs = lzb.encode(stream, bk)
        bits = np.unpackbits(np.asarray(bs.data, np.uint8))[: bs.bit_len]
        for phase in range(8):
            sl = np.packbits(np.concatenate([rng.integers(0, 2, phase).astype(np.uint8), bits]))
            d = torch.from_numpy(np.concatenate([sl, np.zeros(8, np.uint8)])).cuda()
            lens = torch.from_numpy(bk.lengths.astype(np.uint8)).cuda()
            out = torch.empty(n, dtype=torch.int16, device="cuda")
            st = N.empty_bytes(N.STATUS_BYTES)
            ds = L.lzb_huff_decode_scratch_bytes(bs.bit_len, int(bk.lengths.max()), 64)
            scr = N.empty_bytes(ds)
            N.check_rc(L.lzb_huff_decode_at(d.data_ptr(), phase, bs.bit_len, n, lens.data_ptr(), 64,
                                            int(bk.lengths.max()), out.data_ptr(), 2, st.data_ptr(),
                                            scr.data_ptr(), ds, N.stream_ptr()), "decode_at")
            (s,) = N.read_status(st)
            assert s.code == 0, (n, phase)
            assert np.array_equal(out.cpu().numpy().view(np.uint16).astype(np.uint32), stream), (n, phase)


def test_copy_bytes_and_small_transfers(cuda):
    """lzb_copy_bytes (SM copies; either side may be mapped pinned host
    memory), the pinned small-write path and the status read-back."""
    import torch

    from paper_2105_12912_b200 import _native as N

    L = N.lib()
    rng = np.random.default_rng(3)
    for n in (1, 15, 16, 17, 4096, 1 << 20, (1 << 20) + 5):
        src = torch.from_numpy(rng.integers(0, 256, n).astype(np.uint8))
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h.copy_(src)
        d = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
        N.check_rc(L.lzb_copy_bytes(d.data_ptr() + 16 * (n % 2), h.data_ptr(), n, N.stream_ptr()), "copy")
        back = torch.zeros(n, dtype=torch.uint8, pin_memory=True)
        N.check_rc(L.lzb_copy_bytes(back.data_ptr(), d.data_ptr() + 16 * (n % 2), n, N.stream_ptr()), "copy")
        torch.cuda.synchronize()
        assert torch.equal(back, src), n
    d = torch.zeros(300, dtype=torch.uint8, device="cuda")
    for k in range(40):  # wraps the rotating stage region several times
        data = bytes(rng.integers(0, 256, 37).astype(np.uint8))
        N.small_h2d(d[k % 7: k % 7 + 37], data)
        torch.cuda.synchronize()
        assert d[k % 7: k % 7 + 37].cpu().numpy().tobytes() == data
    st = torch.zeros(2 * N.STATUS_BYTES, dtype=torch.uint8, device="cuda")
    st[0] = 4
    s0, s1 = N.read_status(st)
    assert s0.code == 4 and s1.code == 0


def test_reconstruct_fuse_and_layout_kats_on_device(golden, cuda):
    """The remaining reference KATs, asserted on the CUDA path:
    fuse (T/test_reconstruct.py:20-25) through K6 (fuse + 1D partial sum),
    including codes that are NOT the placeholder r at outlier positions
    (q'[idx] += delta adds, it does not overwrite: P/reconstruct.py:22-32);
    all-ones 2x2 (T/test_quantize.py:84-88) through K1; chunk-major order
    (T/test_pipeline.py:220-227) through lzb_chunk_major."""
    import paper_2105_12912_b200 as lzb

    _, _, k = golden
    cfg = lzb.QuantConfig(0.1, 8)  # radius 4
    for codes, want_fused in (([4, 6, 4, 1, 4], k["fuse"]), ([4, 6, 5, 1, 3], None)):
        quant = lzb.QuantGrid(lzb.Dims.of(5), np.array(codes, np.uint32))
        outl = lzb.OutlierList(np.array([2, 4], np.int64), np.array([99, -99], np.int64))
        fused = np.array(codes, np.int64) - 4
        fused[[2, 4]] += [99, -99]
        if want_fused is not None:
            assert fused.tolist() == want_fused
        pre = lzb.reconstruct_grid(quant, outl, cfg, lzb.ChunkSpec(5))
        assert pre.codes.tolist() == np.cumsum(fused).tolist()
        _, opre = O.reconstruct(np.array(codes, np.uint32), (5, 1, 1, 1), (5, 1, 1), 4,
                                np.array([2, 4]), np.array([99, -99]), 0.1, "f64", want_pre=True)
        assert pre.codes.tolist() == opre.tolist()
    ones = lzb.PrequantGrid(lzb.Dims.of(2, 2), np.ones(4, np.int64))
    q, o = lzb.quantize.construct_grid(ones, lzb.QuantConfig(0.1, 1024), lzb.ChunkSpec(2, 2))
    assert q.codes.tolist() == k["ones_2x2"] and len(o) == 0
    grid = lzb.QuantGrid(lzb.Dims.of(4, 2), np.arange(8, dtype=np.uint32))
    assert lzb.pipeline.gather_chunk_major(grid, lzb.ChunkSpec(2, 2)).tolist() == k["chunk_major_4x2"]
    back = lzb.pipeline.scatter_chunk_major(np.array(k["chunk_major_4x2"], np.uint32), lzb.Dims.of(4, 2),
                                   lzb.ChunkSpec(2, 2))
    assert back.codes.tolist() == list(range(8))


@pytest.mark.slow
def test_fast_prequant_exhaustive_f32(cuda):
    """K1's f32 fast prequantizer against the exact reference rule
    (P/quantize.py:95-110) on EVERY f32 bit pattern (4,278,190,080 finite
    values) for six error bounds, plus 2^28 hashed f64 values for the f64
    fast path: 0 mismatches among the accepted fast results."""
    from paper_2105_12912_b200 import _native as N

    L = N.lib()
    st = N.empty_bytes(N.STATUS_BYTES)
    for eb in (1e-4, 2.9345040893554688e-2, 0.5, 1e-7, 123.456, 3.0e-3 / 7):
        N.check_rc(L.lzb_prequant_verify(eb, 0, 1 << 32, 0, st.data_ptr(), N.stream_ptr()), "verify")
        (s,) = N.read_status(st)
        assert s.u[2] == (1 << 32) - 2 * (1 << 23), eb  # every finite f32 examined
        assert s.u[1] > 0, eb
        assert s.u[0] == 0, (eb, s.u[0])
        N.check_rc(L.lzb_prequant_verify(eb, 12345, 1 << 28, 1, st.data_ptr(), N.stream_ptr()), "verify")
        (s,) = N.read_status(st)
        assert s.u[0] == 0, (eb, "f64", s.u[0])


@pytest.mark.parametrize("shape", [(24, 40, 64), (100, 70), (30000,)])
def test_reconstruct_unaligned_code_stream(cuda, shape):
    """K6's register paths load full chunks with 16-byte vectors only from an
    aligned code stream; a stream at an odd 2-byte offset takes the scalar
    loads and gives the same values."""
    import torch

    import paper_2105_12912_b200 as lzb
    from helpers import smooth
    from paper_2105_12912_b200 import ChunkSpec
    from paper_2105_12912_b200 import distributed as D

    vals = smooth(shape).astype(np.float32)
    f = lzb.Field.from_array(vals)
    d = f.dims
    chunk = ChunkSpec.default_for(d.ndim)
    ops = D.DeviceSlabOps(torch.device("cuda"))
    x = torch.from_numpy(vals.reshape(-1)).cuda()
    eb_abs = 1e-4 * float(vals.max() - vals.min())
    codes, _, n_out, recs = ops.quantize(x, d, chunk, eb_abs, 1024)
    buf = torch.zeros(codes.numel() + 2, dtype=torch.uint8, device="cuda")
    buf[2:].copy_(codes)
    rec = ops.local_records(recs, n_out, 0) if n_out else None
    y0 = ops.reconstruct(codes, d, chunk, eb_abs, 1024, rec, n_out, 0)
    y1 = ops.reconstruct(buf[2:], d, chunk, eb_abs, 1024, rec, n_out, 0)
    assert torch.equal(y0, y1)
