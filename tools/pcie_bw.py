"""Host<->device copy ceiling of the box (the e2e bound): pinned H2D alone,
D2H alone, both at once on two streams (per-direction times from events), and
the same with one direction done by SM copy kernels over mapped pinned memory
(lzb_copy_bytes) instead of a copy engine.  python tools/pcie_bw.py [GB]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_12912_b200 import _native as N  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
n = int(gb * 1e9)
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
L = N.lib()


def sm_copy(dst, src, stream):
    N.check_rc(L.lzb_copy_bytes(dst.data_ptr(), src.data_ptr(), n, stream.cuda_stream), "copy")


def dma(dst, src, stream):
    with torch.cuda.stream(stream):
        dst.copy_(src, non_blocking=True)


def timed(ops, reps=3):
    """ops: [(fn, stream)]; returns (wall s, [per-op s]) averaged over reps."""
    for fn, st in ops:
        fn(st)
    torch.cuda.synchronize()
    per = [0.0] * len(ops)
    t = time.perf_counter()
    for _ in range(reps):
        evs = []
        for fn, st in ops:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn(st)
            b.record(st)
            evs.append((a, b))
        torch.cuda.synchronize()
        for i, (a, b) in enumerate(evs):
            per[i] += a.elapsed_time(b) / 1e3 / reps
    return (time.perf_counter() - t) / reps, per


def gbs(sec):
    return round(n / sec / 1e9, 2)


H2D = lambda st: dma(d1, h1, st)        # noqa: E731
D2H = lambda st: dma(h2, d2, st)        # noqa: E731
SM_H2D = lambda st: sm_copy(d1, h1, st)  # noqa: E731
SM_D2H = lambda st: sm_copy(h2, d2, st)  # noqa: E731

out = {"bytes": n}
for name, ops in [("h2d", [H2D]), ("d2h", [D2H]), ("sm_h2d", [SM_H2D]), ("sm_d2h", [SM_D2H]),
                  ("duplex_dma", [H2D, D2H]), ("duplex_dma_h2d_sm_d2h", [H2D, SM_D2H]),
                  ("duplex_sm_h2d_dma_d2h", [SM_H2D, D2H])]:
    wall, per = timed([(fn, st) for fn, st in zip(ops, (s1, s2))])
    out[name] = {"wall_gbs_aggregate": gbs(wall / len(ops)), "per_direction_gbs": [gbs(p) for p in per]}
print(json.dumps(out))
