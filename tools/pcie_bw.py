"""Host<->device copy ceiling of the box (the e2e bound): pinned H2D alone,
D2H alone, and both at once on two streams.  python tools/pcie_bw.py [GB]"""
import json
import sys
import time

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
n = int(gb * 1e9)
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


out = {"bytes": n,
       "h2d_gbs": n / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9,
       "d2h_gbs": n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9}
out["duplex_aggregate_gbs"] = 2 * n / timed(both) / 1e9
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in out.items()}))
