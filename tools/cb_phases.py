"""K2 phase clocks (sort / merge / depths / total, SM cycles) on the C1/C2
histograms: python tools/cb_phases.py"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2105_12912_b200 as lzb  # noqa: E402
from paper_2105_12912_b200 import _native as N  # noqa: E402
from paper_2105_12912_b200 import pipeline as PL  # noqa: E402

for name in ("c2", "c1"):
    cfg = bench.CONFIGS[name]
    x = bench.gen_field_device(cfg, torch.device("cuda"))
    field = lzb.Field.from_array(x.reshape(cfg["shape"]))
    for _ in range(3):
        lzb.compress_device(field, cfg["eb"])
    torch.cuda.synchronize()
    st = PL._pool.bufs[("status", "cuda:0")]
    sb = N.read_status(st[N.STATUS_BYTES: 2 * N.STATUS_BYTES])[0]
    u4, u5 = sb.u[4], sb.u[5]
    print(name, "symbols", sb.u[3], "maxlen", sb.u[2], "cycles: sort", u4 & 0xFFFFFFFF,
          "merge_end", u4 >> 32, "depth_end", u5 & 0xFFFFFFFF, "total", u5 >> 32)
