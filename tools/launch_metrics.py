"""Per-kernel means of every metric in an ncu --metrics ... --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = defaultdict(lambda: defaultdict(list))
for r in rows:
    agg[r["Kernel Name"][:60]][r["Metric Name"]].append(float(r["Metric Value"].replace(",", "")))
for k, m in agg.items():
    n = len(m["gpu__time_duration.sum"])
    print(f"{k:60s} n={n:3d} " + " ".join(f"{mm.split('.')[0][-22:]}={sum(v)/len(v):.4g}" for mm, v in m.items()))
