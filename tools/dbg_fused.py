"""Debug: fused decompress vs oracle on a small smooth 3D field; prints the
mismatch pattern inside the first differing chunk."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2105_12912_b200 as lzb
from oracle import oracle as O
from helpers import smooth

vals = smooth((24, 32, 128))
f = lzb.Field.from_array(vals)
ref = O.compress(f.values, f.dims.as_tuple(), f.vmin, f.vmax, 1e-4)
got = lzb.decompress(ref).values.reshape(24, 32, 128)
want = O.decompress(ref)[0].reshape(24, 32, 128)
bad = np.argwhere(got != want)
print("mismatches", len(bad), "of", got.size)
if len(bad):
    z, y, x = bad[0]
    cz, cy, cx = z // 8 * 8, y // 8 * 8, x // 8 * 8
    g = got[cz:cz+8, cy:cy+8, cx:cx+8]; w = want[cz:cz+8, cy:cy+8, cx:cx+8]
    h = O.parse_header(ref); eb2 = 2 * h["eb"] * (h["vmax"] - h["vmin"]) if h.get("eb_mode", 1) else 2 * h["eb"]
    print("chunk", cz, cy, cx)
    print("diff in quanta (z,y,x) nonzero count:", np.count_nonzero(g != w))
    dq = np.round((g.astype(np.float64) - w.astype(np.float64)) / eb2).astype(np.int64)
    for zz in range(8):
        print("z", zz); print(dq[zz])
