"""Small compress/decompress round trips for compute-sanitizer runs (TMA K1
path, v3 decode, TMA-store K6, multi-phase decode, RLE, u32 symbols)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2105_12912_b200 as lzb  # noqa: E402
from helpers import smooth  # noqa: E402

rng = np.random.default_rng(5)
cases = [(smooth((16, 24, 128)), 1e-4, {}), (smooth((9, 20, 64)), 1e-3, {}),
         ((rng.standard_normal((8, 8, 64)) * 50).astype(np.float32), 1e-4, {"cap": 64}),
         (smooth((40, 50)), 1e-4, {}), (smooth((5000,), ramp=False), 1e-4, {}),
         (np.full((16, 16, 16), 3.0, np.float32) + (np.arange(4096) % 7 == 0).reshape(16, 16, 16), 1e-2, {})]
for vals, eb, kw in cases:
    f = lzb.Field.from_array(vals)
    blob = lzb.compress(f, eb, **kw)
    out = lzb.decompress(blob)
    h = lzb.parse_header(blob)
    err = np.abs(out.values.astype(np.float64) - vals.reshape(-1).astype(np.float64)).max()
    print(vals.shape, h.workflow.name, len(blob), "ok" if err <= h.eb_abs * 1.0001 + 1e-3 else "BOUND!")
# bit-range decode (multi-GPU single-archive decompress), 3 ranges
from test_gpu_range_decode import _range_decode_all  # noqa: E402

stream = rng.choice(64, size=40_000, p=np.r_[np.full(8, 0.1), np.full(56, 0.2 / 56)]).astype(np.uint32)
book = lzb.Codebook.from_counts(np.bincount(stream, minlength=64))
bs = lzb.encode(stream, book)
got, _ = _range_decode_all(bs, book, 64, 3)
print("range decode", "ok" if np.array_equal(got, stream) else "MISMATCH")
