"""Per-CUDA-line totals from `ncu -i R --page source --csv --print-source cuda,sass`:
python tools/ncu_src.py FILE.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
fname = '?'
cur = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r[0] == 'Line No':
        hdr = r
        iws = 4; iie = 7; ith = 8
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0] != '':  # CUDA line summary row
        try:
            out.append((float(r[iws] or 0), float(r[iie] or 0), float(r[ith] or 0), fname, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
tws = sum(o[0] for o in out) or 1
tie = sum(o[1] for o in out) or 1
print('total warp-inst %.3g, stall samples %d' % (tie, tws))
for ws, ie, th, f, ln, src in sorted(out, reverse=True)[:n]:
    print('%5.1f%% stall %5.1f%% inst %4.1f thr  %s:%-5s %s' % (100 * ws / tws, 100 * ie / tie, th / ie if ie else 0, f, ln, src))
