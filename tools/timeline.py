"""CPU/GPU timeline of one small-field compress + decompress (torch.profiler
trace, CUPTI): every runtime call and kernel with its start relative to the
call's start.  python tools/timeline.py [c2]"""
import json
import sys
import tempfile

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2105_12912_b200 as lzb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
x = bench.gen_field_device(cfg, torch.device("cuda"))
field = lzb.Field.from_array(x.reshape(cfg["shape"]))
ybuf = torch.empty_like(x)
for _ in range(10):
    lzb.decompress_device(lzb.compress_device(field, cfg["eb"]), out=ybuf)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("COMPRESS"):
        a = lzb.compress_device(field, cfg["eb"])
    with torch.profiler.record_function("DECOMPRESS"):
        lzb.decompress_device(a, out=ybuf)
    torch.cuda.synchronize()
path = tempfile.mktemp(suffix=".json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X"]
t0 = min(e["ts"] for e in ev if e["name"] == "COMPRESS")
rows = []
for e in ev:
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memset", "gpu_memcpy") or cat == "cuda_runtime" or e["name"] in ("COMPRESS", "DECOMPRESS"):
        rows.append((e["ts"] - t0, e["dur"], "GPU" if cat in ("kernel", "gpu_memset", "gpu_memcpy") else "cpu",
                     e["name"][:70]))
for ts, dur, w, n in sorted(rows):
    print(f"{ts:9.1f} {dur:8.1f} {w:3s} {n}")
