"""Summarise a round's ncu captures into profiles/ (run here, after gpurun).

usage: python tools/ncu_summary.py TAG [c5q|c5s]
  reads gpurun_out/launches_TAG_c5.csv (launch list of the C5 bench command)
        gpurun_out/prof_TAG_full_raw.csv (--set full capture on C5q / C5s)
  writes profiles/TAG_launches_c5.csv, profiles/TAG_ncu_full_<cfg>.md,
         profiles/ncu_traffic.json (dram bytes per launch, scaled <cfg> -> C5)
"""
import csv
import json
import sys
from collections import defaultdict

tag = sys.argv[1]
CFG = sys.argv[2] if len(sys.argv) > 2 else "c5q"
SCALE = {"c5q": 4.0, "c5s": 64.0}[CFG]  # C5 elements / profiled config's elements
CFG_DESC = {"c5q": "C5q (512x2048x2048 f32, rel eb 1e-4)", "c5s": "C5s (512^3 f32, rel eb 1e-4)"}[CFG]
STAGES = {
    "K1_quantize": ["k_quantize3d8", "k_q3_"],
    "K3_huff_encode": ["k_huff_count_w", "k_huff_scan_w", "k_huff_encode_w", "k_huff_fixup_w"],
    "K5_huff_decode": ["k_dec_"],
    "K6_reconstruct": ["k_reconstruct3d8", "k_out_", "k_scan_tiles", "k_first_nonfinite", "k_rc_finish"],
}

# ---- launch list ----
rows = list(csv.reader(open(f"gpurun_out/launches_{tag}_c5.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v = v / 1000 if u in ("nsecond", "ns") else v * 1000 if u in ("msecond", "ms") else v
    agg[r[ki]].append(v)
with open(f"profiles/{tag}_launches_c5.csv", "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["kernel", "launches", "avg_us", "total_us"])
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        w.writerow([k, len(v), round(sum(v) / len(v), 1), round(sum(v), 1)])

# ---- full capture ----
rows = list(csv.reader(open(f"gpurun_out/prof_{tag}_full_raw.csv")))
h = rows[0]
units = rows[1]
col = {n: i for i, n in enumerate(h)}
_SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6,
          "second": 1e6, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
def g(r, n):
    """value in us (times) / MB (bytes) / as-is (others), from the units row"""
    try:
        v = float(r[col[n]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
    return v * _SCALE.get(units[col[n]], 1.0)
out = [f"# ncu --set full on {CFG_DESC}, one launch per kernel", "",
       "| kernel | time us | DRAM read MB | DRAM write MB | DRAM GB/s | warps active % | issue active % | regs | top stalls (per issue) |",
       "|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").split("<")[0]
    t = g(r, "gpu__time_duration.sum")
    rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
    st = []
    for n, i in col.items():
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("per_issue_active.ratio"):
            try:
                st.append((n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(r[i])))
            except ValueError:
                pass
    st.sort(key=lambda kv: -kv[1])
    out.append(f"| {name} | {t:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) / t * 1e3:.0f} | "
               f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
               f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
               f"{g(r, 'launch__registers_per_thread'):.0f} | "
               + ", ".join(f"{k} {v:.2f}" for k, v in st[:4]) + " |")
    for stage, pats in STAGES.items():
        if any(p in name for p in pats):
            traffic[stage] = traffic.get(stage, 0.0) + (rd + wr) * 1e6 * SCALE
out += ["", "DRAM GB/s = (read + write) / duration.  `profiles/ncu_traffic.json` holds the",
        f"per-stage DRAM bytes of these kernels scaled by {SCALE:g} (C5 / {CFG} elements)."]
open(f"profiles/{tag}_ncu_full_{CFG}.md", "w").write("\n".join(out) + "\n")
json.dump({k: int(v) for k, v in traffic.items()} | {"_source": f"profiles/{tag}_ncu_full_{CFG}.md",
          "_note": f"dram__bytes_read.sum + dram__bytes_write.sum of the stage's profiled kernels on {CFG} x {SCALE:g}"},
          open("profiles/ncu_traffic.json", "w"), indent=1)
print("\n".join(out))
