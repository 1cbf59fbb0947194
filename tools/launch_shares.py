"""Per-kernel share of a `ncu --metrics gpu__time_duration.sum --csv` launch list.

  python tools/launch_shares.py launches.csv [skip_first_n]

ncu serialises launches and runs them cold, so absolute times overstate the
overlapped step; the SHARE per kernel is what bench.py's roofline line is
checked against."""
import csv
import gzip
import re
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
op = gzip.open if path.endswith(".gz") else open
with op(path, "rt") as f:
    lines = [l for l in f if l.startswith('"')]
rows = list(csv.DictReader(lines))
per = {}
seen = 0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    seen += 1
    if seen <= skip:
        continue
    name = r["Kernel Name"]
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name).replace("janus::", "")
    v = float(r["Metric Value"])
    unit = r.get("Metric Unit", "ns")
    v = v / 1e3 if unit in ("nsecond", "ns") else (v if unit in ("usecond", "us") else v * 1e3)
    n, t = per.get(name, (0, 0.0))
    per[name] = (n + 1, t + v)
tot = sum(t for _, t in per.values())
print(f"total ms {tot / 1e3:.3f} n {sum(n for n, _ in per.values())}")
for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
    print(f"{100 * t / tot:6.2f}% {n:6d} {t / n:8.1f}us {k}")
