#!/bin/bash
# launch list (per-kernel device time) of one step of a bench config: TAG CONFIG
TAG=${1:-x}; CFG=${2:-c5q}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:lzb|k_' \
  --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 0 > gpurun_out/launches_${TAG}.log 2>&1
python3 - "$TAG" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi: agg[r[ki]].append(float(r[vi].replace(",", "")))
with open(f"gpurun_out/launches_{tag}.txt", "w") as f:
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"{sum(v)/len(v)/1000:10.1f} us x{len(v):3d}  {k[:90]}\n")
PY
