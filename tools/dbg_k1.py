"""Debug: per-golden-case compress check + K1 histogram vs bincount of codes."""
import sys, json
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch

from helpers import golden_case
import paper_2105_12912_b200 as lzb
from paper_2105_12912_b200 import pipeline as P

def load_golden():
    import json as j, numpy as n, pathlib
    d = pathlib.Path("tests/golden")
    return (j.loads((d / "archives.json").read_text()), n.load(d / "archives.npz"), j.loads((d / "kats.json").read_text()))

g = load_golden()
for i in range(len(g[0])):
    c, vals, dims, kw, arc = golden_case(g, i)
    kw = dict(kw)
    if "chunk" in kw: kw["chunk"] = lzb.ChunkSpec(*kw["chunk"])
    d = lzb.Dims(*dims[:3], ndim=dims[3])
    f = lzb.Field(d, np.ascontiguousarray(vals).reshape(-1), c["vmin"], c["vmax"])
    try:
        got = lzb.compress(f, **kw)
        print(i, c["name"], dims, kw, "OK" if got == arc else "MISMATCH")
    except Exception as e:
        print(i, c["name"], dims, kw, "ERR", e)
    # histogram check
    n = P._pool.bufs
    codes = [v for k, v in n.items() if k[0] == "codes"][0]
    hist = [v for k, v in n.items() if k[0] == "hist"][0]
    cap = kw.get("cap", 1024)
    cnt = vals.size
    cb = 2 if cap <= 65536 else 4
    cd = codes[: cnt * cb].cpu().numpy().view(np.uint16 if cb == 2 else np.uint32)
    h = hist[: cap * 8].cpu().numpy().view(np.int64)
    bc = np.bincount(cd, minlength=cap)[:cap]
    if not np.array_equal(bc, h):
        bad = np.nonzero(bc != h)[0]
        print("   HIST DIFF at", bad[:10], bc[bad[:10]], h[bad[:10]], "r=", cap // 2)
