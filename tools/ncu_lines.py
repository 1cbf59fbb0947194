"""Aggregate ncu warp-stall samples per CUDA source line.

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_lines.py x.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, agg, src, reasons_by = None, {}, {}, {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    try:
        smp = int(r[4] or 0)
    except ValueError:
        smp = 0
    key = (cur, ln)
    agg[key] = agg.get(key, 0) + smp
    src[key] = r[1]
    rb = reasons_by.setdefault(key, {})
    for k, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and k < len(r):
            try:
                rb[h] = rb.get(h, 0) + int(r[k] or 0)
            except ValueError:
                pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    rs = sorted(reasons_by[k].items(), key=lambda x: -x[1])[:2]
    rs = " ".join(f"{a[6:]}:{b}" for a, b in rs if b)
    print(f"{v:6d} {100 * v / tot:5.1f}% {k[0]}:{k[1]:<5d} {src[k].strip()[:70]:70s} {rs}")
