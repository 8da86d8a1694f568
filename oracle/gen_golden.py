"""Generate tests/golden/ fixtures from the REFERENCE itself (lzebc).

Run in the build container, where /root/reference is mounted:

    python oracle/gen_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here as
small fixtures: input fields, the exact archive bytes the reference produces
for them, and the decoded values.  tests/test_oracle_golden.py pins the CPU
oracle to these; the -m gpu tests pin the CUDA path to them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def smooth(shape, ramp=True):
    """SURVEY.md 8(d) smooth generator (no RNG)."""
    axes = [np.arange(n, dtype=np.float64) for n in shape]
    g = np.meshgrid(*axes, indexing="ij", sparse=True)
    data = np.zeros(shape, np.float64)
    for i, a in enumerate(g):
        data = data + np.sin(a / (13.0 + 7 * i))
    data = data * 40.0
    if ramp:
        data = data + 0.03 * g[-1]
    return data.astype(np.float32)


def sparse(shape, seed=0, nblobs=None):
    """SURVEY.md 8(d) sparse generator."""
    rng = np.random.default_rng(seed)
    data = np.full(shape, 1.0, np.float64)
    nblobs = nblobs or max(8, int(np.prod(shape) // 2_000_000))
    for _ in range(nblobs):
        c = [rng.uniform(0, s) for s in shape]
        w = rng.uniform(2.0, 6.0)
        amp = float(np.exp(rng.normal(3.0, 1.0)))
        lo = [max(0, int(ci - 4 * w)) for ci in c]
        hi = [min(s, int(ci + 4 * w) + 1) for ci, s in zip(c, shape)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        g = np.meshgrid(*[np.arange(a, b) - ci for a, b, ci in zip(lo, hi, c)], indexing="ij",
                        sparse=True)
        r2 = sum(gi * gi for gi in g)
        data[sl] += amp * np.exp(-r2 / (2 * w * w))
    return data.astype(np.float32)


def main():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    import lzebc
    from helpers import make_field
    from lzebc.pipeline import gather_chunk_major
    from lzebc.quantize import construct_grid, prequantize

    os.makedirs(OUT, exist_ok=True)
    cases = []
    fields = []  # distinct input fields; cases refer to them by id
    rng = np.random.default_rng(20261017)

    def add(name, field, **kw):
        blob = lzebc.compress(field, **kw)
        hdr = lzebc.parse_header(blob)
        dec = lzebc.decompress(blob)
        cfg = lzebc.QuantConfig(hdr.eb_abs, hdr.cap)
        quant, outl = construct_grid(prequantize(field, cfg), cfg, hdr.chunk)
        stream = gather_chunk_major(quant, hdr.chunk)
        d = field.dims
        if not fields or fields[-1] is not field:
            fields.append(field)
        cases.append(dict(
            name=name, field=len(fields) - 1,
            dims=np.array([d.nx, d.ny, d.nz, d.ndim], np.int64),
            vmin=field.vmin, vmax=field.vmax, kw=json.dumps({k: (v if not hasattr(v, "cx") else
                                                            [v.cx, v.cy, v.cz])
                                                        for k, v in kw.items()}),
            archive=np.frombuffer(blob, np.uint8),
            decoded_sha256=hashlib.sha256(dec.values.tobytes()).hexdigest(),
            stream_sha256=hashlib.sha256(stream.astype(np.uint32).tobytes()).hexdigest(),
            out_idx=outl.indices, out_delta=outl.deltas,
            hist=lzebc.histogram(stream, hdr.cap)))

    # make_field sweep: every ndim x dtype x workflow, rel eb
    kinds = ["walk", "waves", "ramp", "noise", "spiky"]
    for ndim in (1, 2, 3):
        for dt in (np.float32, np.float64):
            for kind in kinds:
                f = make_field(rng, ndim, dtype=dt, kind=kind)
                for wf in ("huff", "rle", "rlevle", None):
                    add(f"mf{ndim}d_{np.dtype(dt).name}_{kind}_{wf}", f, eb=1e-3, workflow=wf)
    # caps, chunk specs, abs mode, estimate mode
    f3 = make_field(rng, 3, dtype=np.float32, kind="walk")
    for cap in (4, 16, 256, 4096):
        add(f"cap{cap}", f3, eb=1e-3, cap=cap)
    for spec in ((4, 4, 2), (3, 5, 7), (16, 1, 1), (8, 8, 8)):
        add(f"chunk{'x'.join(map(str, spec))}", f3, eb=1e-4, chunk=lzebc.ChunkSpec(*spec))
    f2 = make_field(rng, 2, dtype=np.float64, kind="waves")
    for spec in ((8, 8, 1), (5, 3, 1), (32, 2, 1)):
        add(f"chunk2d{'x'.join(map(str, spec))}", f2, eb=1e-4, chunk=lzebc.ChunkSpec(*spec))
    add("abs_mode", f2, eb=0.125, eb_mode="abs")
    add("estimate_mode", f2, eb=1e-3, select_mode="estimate")
    # SURVEY 8(d) generators at small sizes
    add("smooth3d", lzebc.Field.from_array(smooth((20, 40, 36))), eb=1e-4)
    add("smooth2d", lzebc.Field.from_array(smooth((90, 120))), eb=1e-4)
    add("smooth1d", lzebc.Field.from_array(smooth((20000,), ramp=False)), eb=1e-4)
    add("sparse3d", lzebc.Field.from_array(sparse((40, 40, 40))), eb=1e-2)
    add("sparse3d_huff", lzebc.Field.from_array(sparse((40, 40, 40))), eb=1e-2, workflow="huff")
    # edge cases from the reference tests
    add("const_rlevle", lzebc.Field.from_array(np.full((24, 24, 24), 3.75, np.float32)),
        eb=0.001, eb_mode="abs")
    for cnt in (1, 2, 3):
        add(f"tiny{cnt}", lzebc.Field.from_array(np.linspace(5, 6, cnt)), eb=0.01, eb_mode="abs")
    add("outlier_heavy", lzebc.Field.from_array(
        np.random.default_rng(61).normal(scale=1e6, size=2048)), eb=1e-7)
    add("single_row_2d", lzebc.Field.from_array(
        np.cumsum(rng.normal(size=(1, 300)), axis=-1)), eb=1e-3)
    # uniform quant codes (acceptance 5 construction): 9-11 bit code book
    dims = lzebc.Dims.of(64, 64)
    cfg = lzebc.QuantConfig(0.5, 1024)
    deltas = np.random.default_rng(555).integers(-511, 512, dims.count).astype(np.int64)
    from lzebc.reconstruct import reconstruct_grid
    from lzebc.quantize import OutlierList
    pq = reconstruct_grid(lzebc.QuantGrid(dims, (deltas + 512).astype(np.uint32)),
                          OutlierList.empty(), cfg, lzebc.ChunkSpec(16, 16))
    add("uniform_codes", lzebc.Field.from_array(pq.as_3d()[0].astype(np.float32)), eb=0.5,
        eb_mode="abs", chunk=lzebc.ChunkSpec(16, 16))

    arrays = {}
    index = []
    for j, f in enumerate(fields):
        arrays[f"field{j}"] = f.values
    for i, c in enumerate(cases):
        for k in ("dims", "archive", "out_idx", "out_delta", "hist"):
            arrays[f"{i}_{k}"] = np.asarray(c[k])
        index.append(dict(i=i, name=c["name"], field=c["field"], vmin=c["vmin"], vmax=c["vmax"],
                          kw=c["kw"], decoded_sha256=c["decoded_sha256"],
                          stream_sha256=c["stream_sha256"],
                          sha256=hashlib.sha256(c["archive"].tobytes()).hexdigest()))
    np.savez_compressed(os.path.join(OUT, "archives.npz"), **arrays)
    with open(os.path.join(OUT, "archives.json"), "w") as fh:
        json.dump(index, fh, indent=1)

    # ---- stage KATs (the reference tests' known answers, recomputed here) ----
    kats = {}
    F = lzebc.Field.from_array
    kats["prequant_eb001"] = prequantize(F(np.array([1.0, 0.029, -0.03, 0.0])),
                                         lzebc.QuantConfig(0.01)).codes.tolist()
    kats["prequant_ties"] = prequantize(F(np.array([0.5, -0.5, 1.5, -1.5, 2.5])),
                                        lzebc.QuantConfig(0.5)).codes.tolist()
    from lzebc.quantize import construct_chunk
    c, oi, od = construct_chunk(np.ones((1, 2, 2), np.int64), lzebc.QuantConfig(0.1, 1024), 2)
    kats["ones_2x2"] = c.tolist()
    c, oi, od = construct_chunk(np.array([0, 5, 5, 6], np.int64).reshape(1, 1, 4),
                                lzebc.QuantConfig(0.1, 4), 1)
    kats["cap4_outlier"] = [c.tolist(), oi.tolist(), od.tolist()]
    for counts in ([10, 1], [0, 0, 42, 0], [8, 4, 2, 1, 1], [2, 1, 1],
                   [2 ** i for i in range(12, 0, -1)]):
        b = lzebc.Codebook.from_counts(np.array(counts, np.int64))
        kats[f"book_{'_'.join(map(str, counts))}"] = [b.lengths.tolist(),
                                                      [int(x) for x in b.codes]]
    s = lzebc.encode(np.array([0, 1, 2], np.uint32),
                     lzebc.Codebook.from_counts(np.array([2, 1, 1], np.int64)))
    kats["encode_012"] = [s.bit_len, s.count, s.data.tolist()]
    v, ln = lzebc.run_length_encode(np.array([0, 0, 1, 2, 2, 2, 2, 2, 0, 0], np.uint32))
    kats["rle_textbook"] = [v.tolist(), ln.tolist()]
    from lzebc.reconstruct import dequantize, fuse_outliers
    fused = fuse_outliers(lzebc.QuantGrid(lzebc.Dims.of(5), np.array([4, 6, 4, 1, 4], np.uint32)),
                          OutlierList(np.array([2, 4]), np.array([99, -99])),
                          lzebc.QuantConfig(0.1, 8))
    kats["fuse"] = fused.tolist()
    from lzebc.quantize import PrequantGrid
    kats["dequant"] = dequantize(PrequantGrid(lzebc.Dims.of(3), np.array([-1, 0, 50])),
                                 lzebc.QuantConfig(0.01), "f64").values.tolist()
    q = lzebc.QuantGrid(lzebc.Dims.of(4, 2), np.arange(8, dtype=np.uint32))
    kats["chunk_major_4x2"] = gather_chunk_major(q, lzebc.ChunkSpec(2, 2)).tolist()
    # random histograms -> reference code lengths (codebook parity, two-queue vs heap)
    hrng = np.random.default_rng(4242)
    sys.path.insert(0, REF_TESTS)
    from test_codebook import random_histogram
    hists, lens = [], []
    for _ in range(400):
        h = random_histogram(hrng)
        hists.append(h.tolist())
        lens.append(lzebc.Codebook.from_counts(h).lengths.tolist())
    kats["random_histograms"] = hists
    kats["random_lengths"] = lens
    # analyze() CSV reports (P/smoothness.py:166-188): seeded madograms of the
    # prequant and quant-code grids + entropy stats + decision
    an = []
    for shape, eb, dmax, seed, cap in (((48, 64), 1e-2, 30, 0, 1024), ((12, 10, 9), 1e-3, 50, 7, 256),
                                       ((3000,), 1e-4, 200, 3, 1024)):
        vals = smooth(shape).reshape(-1).astype(np.float32)
        fld = lzebc.Field.from_array(vals.reshape(shape))
        rec = lzebc.analyze(fld, lzebc.QuantConfig(eb * fld.value_range, cap), dmax=dmax, seed=seed)
        an.append([list(shape), eb, dmax, seed, cap, rec.to_csv()])
    kats["analyze_csv"] = an
    # the CLI's compress report line on the reference tests' sine field (T/test_cli.py:7-13)
    from lzebc.cli import run
    import contextlib
    import io
    import tempfile
    x = np.linspace(0, 20, 64 * 48)
    data = (np.sin(x) * 100 + x).astype(np.float32)
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "field.f32")
        with open(src, "wb") as fh:
            fh.write(data.tobytes())
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = run(["compress", "-d", "64,48", "-t", "f32", "-e", "rel:1e-4", src,
                        os.path.join(td, "a.lz")])
        assert code == 0
        kats["cli_compress_line"] = buf.getvalue().strip()
    with open(os.path.join(OUT, "kats.json"), "w") as fh:
        json.dump(kats, fh)
    total = sum(os.path.getsize(os.path.join(OUT, p)) for p in os.listdir(OUT))
    print(f"{len(cases)} archive cases, {len(kats)} KAT groups, {total / 1e6:.2f} MB in {OUT}")


if __name__ == "__main__":
    main()
