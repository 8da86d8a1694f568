"""Host-side cost of the small-field API calls (cProfile over N calls; the GPU
work is synchronised inside each call): python tools/hostprof.py [c2] [N]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2105_12912_b200 as lzb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = bench.CONFIGS[name]
x = bench.gen_field_device(cfg, torch.device("cuda"))
field = lzb.Field.from_array(x.reshape(cfg["shape"]))
ybuf = torch.empty_like(x)
for _ in range(10):
    lzb.decompress_device(lzb.compress_device(field, cfg["eb"]), out=ybuf)
torch.cuda.synchronize()
arc0 = lzb.compress_device(field, cfg["eb"])
which = sys.argv[3] if len(sys.argv) > 3 else "compress"
calls = {"compress": lambda: lzb.compress_device(field, cfg["eb"]),
         "decompress": lambda: lzb.decompress_device(arc0, out=ybuf)}
for what, fn in ((which, calls[which]),):
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    print(f"{what}: {(time.perf_counter() - t) / reps * 1e6:.1f} us/call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(reps):
        fn()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
