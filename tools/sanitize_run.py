"""Small round trips over every GPU path, for compute-sanitizer
(memcheck / racecheck / synccheck):

  3D f32 TMA K1 (whole and partial chunk rows) + plan decode + K6 (16-bit
  and int32 paths), an outlier-heavy noisy field (RLE+VLE), 2D, 1D long codes
  (irregular subsequences), a non-synchronising book through the RETRY ->
  exhaustive decoder, bit-range decode, near-constant field; round 2: the
  2D / 1D register K1 / K6 (partial chunks, outlier-slot overflow, f64,
  wide outliers) and the single-sync compress with its hand-overs.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import paper_2105_12912_b200 as lzb
from helpers import smooth

rng = np.random.default_rng(5)
cases = [
    (smooth((24, 32, 128)), 1e-4, {}),
    (smooth((21, 19, 256)), 1e-3, {}),
    ((rng.standard_normal((16, 16, 256)) * 50).astype(np.float32), 1e-4, dict(cap=64)),
    (smooth((300, 500)), 1e-4, {}),
    (smooth((200_000,), ramp=False), 1e-4, {}),
    (np.full((16, 16, 128), 3.0, np.float32) + rng.standard_normal((16, 16, 128)).astype(np.float32) * 1e-6,
     1e-2, {}),
    # round 2: 2D / 1D register kernels (partial chunks, slot overflow -> emit,
    # f64, wide outliers), single-sync compress and its hand-overs
    (smooth((37, 90)), 1e-4, {}),
    ((rng.standard_normal((40, 72)) * 50).astype(np.float32), 1e-4, dict(cap=64)),
    (smooth((53, 70)).astype(np.float64), 1e-5, {}),
    ((rng.standard_normal(5000) * 50).astype(np.float32), 1e-4, dict(cap=64)),
    (smooth((3001,), ramp=False).astype(np.float64), 1e-4, {}),
    (np.where(np.arange(4096) % 97 == 0, 1e7, 0.0).astype(np.float32).reshape(64, 64), 1e-6, dict(eb_mode="abs")),
]
for vals, eb, kw in cases:
    f = lzb.Field.from_array(vals)
    blob = lzb.compress(f, eb, **kw)
    out = lzb.decompress(blob)
    err = np.abs(f.values.astype(np.float64) - out.values.astype(np.float64)).max()
    print(vals.shape, lzb.parse_header(blob).workflow.name, len(blob), float(err))
# a fixed-length book (never resynchronises at microblock starts): RETRY path
book = lzb.Codebook.from_lengths(bytes([3] * 8))
sym = rng.integers(0, 8, 40000).astype(np.uint32)
assert np.array_equal(lzb.decode(lzb.encode(sym, book), book), sym)
print("sanitize run ok")
