"""Where a small-field round trip goes (C1/C2): wall time per call, the GPU
kernels' own time (torch.profiler / CUPTI) and the host gap between them.
python tools/smallprof.py [c2] [reps]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2105_12912_b200 as lzb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = bench.CONFIGS[name]
x = bench.gen_field_device(cfg, torch.device("cuda"))
field = lzb.Field.from_array(x.reshape(cfg["shape"]))
ybuf = torch.empty_like(x)


def comp():
    return lzb.compress_device(field, cfg["eb"])


def dec(a):
    return lzb.decompress_device(a, out=ybuf)


for _ in range(10):
    dec(comp())
torch.cuda.synchronize()
for what, fn in (("compress", comp), ("roundtrip", lambda: dec(comp()))):
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{name} {what}: {(time.perf_counter() - t) / reps * 1e3:.3f} ms/call wall "
          f"({x.numel() * 4 / ((time.perf_counter() - t) / reps) / 1e9:.1f} GB/s)")
a = comp()
t = time.perf_counter()
for _ in range(reps):
    dec(a)
torch.cuda.synchronize()
print(f"{name} decompress: {(time.perf_counter() - t) / reps * 1e3:.3f} ms/call wall")

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        dec(comp())
    torch.cuda.synchronize()
ka = prof.key_averages()
rows = sorted((e for e in ka if e.device_time_total > 0), key=lambda e: -e.device_time_total)
print(f"{'kernel / op':60s} {'calls':>6s} {'gpu us/call':>12s}")
for e in rows[:25]:
    print(f"{e.key[:60]:60s} {e.count // reps:6d} {e.device_time_total / reps:12.1f}")
cpu = sorted(ka, key=lambda e: -e.self_cpu_time_total)
print(f"{'host op':60s} {'calls':>6s} {'cpu us/call':>12s}")
for e in cpu[:15]:
    print(f"{e.key[:60]:60s} {e.count // reps:6d} {e.self_cpu_time_total / reps:12.1f}")
