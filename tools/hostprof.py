import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2105_12912_b200 as lzb
import bench
cfg = bench.CONFIGS["c2"]
x = bench.gen_field_device(cfg, torch.device("cuda"))
field = lzb.Field.from_array(x.reshape(cfg["shape"]))
def step():
    a = lzb.compress_device(field, cfg["eb"])
    y = lzb.decompress_device(a)
    return y
for _ in range(5): step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(50): step()
torch.cuda.synchronize()
print("ms/step", (time.perf_counter() - t) / 50 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(18)
