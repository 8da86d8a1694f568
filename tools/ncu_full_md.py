"""Markdown summary of an ncu --set full raw CSV (one row per captured launch):
python tools/ncu_full_md.py gpurun_out/prof_TAG_raw.csv TITLE > profiles/TAG_ncu_full_c5q.md"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units, data = rows[0], rows[1], rows[2:]
col = {name: i for i, name in enumerate(h)}
TO_BASE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
           "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
           "second": 1.0, "s": 1.0}


def v(r, name):
    """value in base units (bytes, seconds) where the units row says so"""
    try:
        x = float(r[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
    return x * TO_BASE.get(units[col[name]], 1.0)


print(f"# {sys.argv[2]}\n")
print("| kernel | time us | DRAM read MB | DRAM write MB | DRAM GB/s | warps active % | issue active % | regs | "
      "warp-instr (M) | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|")
seen = set()
for r in data:
    k = r[col["Kernel Name"]].split("(")[0]
    if k in seen:
        continue
    seen.add(k)
    t = v(r, "gpu__time_duration.sum")  # s
    rd, wr = v(r, "dram__bytes_read.sum") / 1e6, v(r, "dram__bytes_write.sum") / 1e6  # MB
    stalls = sorted(((v(r, c), c.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", "")) for c in h if c.startswith("smsp__average_warps_issue_stalled_")
        and c.endswith("_per_issue_active.ratio")), reverse=True)[:4]
    print(f"| {k} | {t * 1e6:.1f} | {rd:.0f} | {wr:.0f} | {(rd + wr) / 1e3 / t:.0f} | "
          f"{v(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{v(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{v(r, 'launch__registers_per_thread'):.0f} | {v(r, 'smsp__inst_executed.sum') / 1e6:.0f} | "
          + ", ".join(f"{n} {s:.2f}" for s, n in stalls) + " |")
