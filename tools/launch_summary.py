"""Per-kernel and per-stage summary of an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
on the full C5 bench step (tools/round_measure.sh).

usage: python tools/launch_summary.py gpurun_out/TAG_launches_c5_raw.csv TAG
writes profiles/TAG_launches_c5.csv and profiles/ncu_traffic.json (DRAM
bytes per launch of each bench stage, measured at C5 -- not scaled)."""
import collections
import csv
import json
import sys

src, tag = sys.argv[1], sys.argv[2]
STAGES = {
    "K1_quantize": ("k_quantize3d8", "k_q3_", "k_check_sorted", "k_order_", "k_scan_u32"),
    "K3_huff_encode": ("k_huff_",),
    "K5_huff_decode": ("k_dec",),
    "K6_reconstruct": ("k_reconstruct3d8", "k_out_", "k_scan_tiles", "k_first_nonfinite", "k_rc_finish", "k_mm_init"),
}
TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= BYTES.get(r[ui], 1) if r[mi].startswith("dram") else TIME.get(r[ui], 1)
    per[(r[ii], r[ki])][r[mi]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, k), m in per.items():
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
steps = max(a[0] for k, a in agg.items() if "k_quantize" in k)
# the field-construction range pass is timed outside the step (its own bench key)
total_us = sum(a[1] for k, a in agg.items() if "k_field_range" not in k)
with open(f"profiles/{tag}_launches_c5.csv", "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["kernel", "launches", "avg_us", "share_of_step_pct", "dram_gb_per_launch"])
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share = "" if "k_field_range" in k else round(100 * a[1] / total_us, 2)
        w.writerow([k, a[0], round(a[1] / a[0], 1), share, round(a[2] / a[0] / 1e9, 3)])
traffic = {}
for st, prefixes in STAGES.items():
    b = sum(a[2] for k, a in agg.items() if any(k.startswith(p) or k.startswith("void " + p) for p in prefixes))
    traffic[st] = int(b / steps)
traffic["_source"] = f"profiles/{tag}_launches_c5.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum, full C5 step)"
traffic["_note"] = "DRAM bytes per bench step of each stage's kernels, measured at C5 (not scaled)"
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(traffic, indent=1))
