"""The CLI (P/cli.py) and analyze (P/smoothness.py:166-188) over the GPU path:
the reference CLI tests' cases (T/test_cli.py) plus the reference's own
outputs as golden values (tests/golden/kats.json, oracle/gen_golden.py)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture()
def sine_file(tmp_path):
    x = np.linspace(0, 20, 64 * 48)
    data = (np.sin(x) * 100 + x).astype(np.float32)
    path = tmp_path / "field.f32"
    path.write_bytes(data.tobytes())
    return path, data


def _run(argv):
    from paper_2105_12912_b200.cli import run

    return run(argv)


def test_compress_line_matches_reference(golden, cuda, sine_file, tmp_path, capsys):
    _, _, kats = golden
    path, _ = sine_file
    out = tmp_path / "a.lz"
    assert _run(["compress", "-d", "64,48", "-t", "f32", "-e", "rel:1e-4", str(path), str(out)]) == 0
    line = capsys.readouterr().out.strip()
    want = dict(kv.split("=") for kv in kats["cli_compress_line"].split())
    got = dict(kv.split("=") for kv in line.split())
    assert got["workflow"] == want["workflow"] and got["cr"] == want["cr"]
    assert got["max_abs_err"] == want["max_abs_err"]
    for k in ("rmse", "psnr"):
        assert float(got[k]) == pytest.approx(float(want[k]), rel=1e-5)


def test_roundtrip_stats_and_determinism(cuda, sine_file, tmp_path, capsys):
    path, data = sine_file
    a, b, back = tmp_path / "a.lz", tmp_path / "b.lz", tmp_path / "back.f32"
    assert _run(["compress", "-d", "64,48", "-t", "f32", "-e", "abs:0.5", str(path), str(a)]) == 0
    assert _run(["compress", "-d", "64,48", "-t", "f32", "-e", "abs:0.5", "-T", "4", str(path), str(b)]) == 0
    assert a.read_bytes() == b.read_bytes()
    assert _run(["decompress", str(a), str(back)]) == 0
    dec = np.frombuffer(back.read_bytes(), "<f4")
    slack = float(np.spacing(np.abs(data).max()) / 2)
    assert np.abs(dec.astype(np.float64) - data.astype(np.float64)).max() <= 0.5 * (1 + 1e-12) + slack
    capsys.readouterr()
    assert _run(["stats", "-d", "64,48", "-t", "f32", str(path), str(back), str(a)]) == 0
    assert "cr=" in capsys.readouterr().out
    out = tmp_path / "rle.lz"
    assert _run(["compress", "-d", "64,48", "-t", "f32", "-w", "rle", str(path), str(out)]) == 0
    from paper_2105_12912_b200 import Workflow, parse_header

    assert parse_header(out.read_bytes()).workflow is Workflow.RLE


def test_exit_codes(cuda, sine_file, tmp_path, capsys):
    path, _ = sine_file
    assert _run(["compress", "-d", "10", "-t", "f32", str(path), str(tmp_path / "x.lz")]) == 1
    assert "bytes" in capsys.readouterr().err
    assert _run(["compress", "-d", "4", "-t", "f32", str(tmp_path / "absent"), str(tmp_path / "x")]) == 1
    for argv in (["-e", "weird"], ["-t", "f99"]):
        base = ["compress", "-d", "64,48", "-t", "f32"]
        if argv[0] == "-t":
            base = ["compress", "-d", "64,48"]
        assert _run(base + argv + [str(path), str(tmp_path / "x.lz")]) == 1
    assert _run(["compress", "-d", "0", "-t", "f32", str(path), str(tmp_path / "x.lz")]) == 1
    bad = tmp_path / "bad.f32"
    bad.write_bytes(np.array([1.0, np.nan, 2.0, 3.0], np.float32).tobytes())
    capsys.readouterr()
    assert _run(["compress", "-d", "4", "-t", "f32", str(bad), str(tmp_path / "x.lz")]) == 2
    assert "data error" in capsys.readouterr().err
    const = tmp_path / "const.f32"
    const.write_bytes(np.full(64, 5.0, np.float32).tobytes())
    assert _run(["compress", "-d", "64", "-t", "f32", str(const), str(tmp_path / "x.lz")]) == 2
    assert "absolute" in capsys.readouterr().err
    arc = tmp_path / "a.lz"
    assert _run(["compress", "-d", "64,48", "-t", "f32", str(path), str(arc)]) == 0
    arc.write_bytes(arc.read_bytes()[:50])
    capsys.readouterr()
    assert _run(["decompress", str(arc), str(tmp_path / "y.f32")]) == 3
    assert "corrupt" in capsys.readouterr().err.lower()


def test_analyze_matches_reference_csv(golden, cuda, tmp_path, capsys):
    from helpers import smooth

    import paper_2105_12912_b200 as lzb

    _, _, kats = golden
    for shape, eb, dmax, seed, cap, want in kats["analyze_csv"]:
        vals = smooth(tuple(shape)).reshape(-1).astype(np.float32)
        fld = lzb.Field.from_array(vals.reshape(shape))
        rec = lzb.analyze(fld, lzb.QuantConfig(eb * fld.value_range, cap), dmax=dmax, seed=seed)
        assert rec.to_csv() == want, shape
    # the CLI analyze command (CSV to a file and to stdout)
    shape, eb, dmax, seed, cap, want = kats["analyze_csv"][0]
    src = tmp_path / "f.f32"
    src.write_bytes(smooth(tuple(shape)).reshape(-1).astype(np.float32).tobytes())
    csv = tmp_path / "r.csv"
    dims = ",".join(map(str, shape[::-1]))
    assert _run(["analyze", "-d", dims, "-t", "f32", "-e", f"rel:{eb}", "--cap", str(cap),
                 "--dmax", str(dmax), "--seed", str(seed), str(src), str(csv)]) == 0
    assert csv.read_text() == want
    capsys.readouterr()
    assert _run(["analyze", "-d", dims, "-t", "f32", "-e", f"rel:{eb}", "--dmax", "10", str(src)]) == 0
    assert capsys.readouterr().out.startswith("stage,kind,distance,variance")


def test_out_of_core_blocks_match_whole_field(cuda, tmp_path, capsys):
    """--block-mb: the raw file is memory-mapped and pushed through the GPU in
    slabs; the archive equals the whole-field one and decodes to the same file."""
    from helpers import smooth

    data = smooth((24, 96, 128)).astype(np.float32)  # 1.2 MB -> three slabs of <= 0.5 MB... 1 MB
    path = tmp_path / "f.f32"
    path.write_bytes(data.tobytes())
    whole, blocks = tmp_path / "w.lz", tmp_path / "b.lz"
    dims = "128,96,24"
    assert _run(["compress", "-d", dims, "-t", "f32", "-e", "rel:1e-4", str(path), str(whole)]) == 0
    assert _run(["compress", "-d", dims, "-t", "f32", "-e", "rel:1e-4", "--block-mb", "1", str(path),
                 str(blocks)]) == 0
    line = capsys.readouterr().out.strip().splitlines()[-1]
    assert line.startswith("workflow=HUFFMAN") and "max_abs_err=" in line
    assert blocks.read_bytes() == whole.read_bytes()
    y0, y1 = tmp_path / "y0.f32", tmp_path / "y1.f32"
    assert _run(["decompress", str(whole), str(y0)]) == 0
    assert _run(["decompress", "--block-mb", "1", str(whole), str(y1)]) == 0
    assert y0.read_bytes() == y1.read_bytes()
