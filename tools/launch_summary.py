"""Mean per-kernel duration from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
agg = defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") in ("nsecond", "ns"):
            v /= 1e3
        elif r.get("Metric Unit") == "msecond":
            v *= 1e3
        agg[r["Kernel Name"][:70]].append(v)
tot = 0.0
for k, v in agg.items():
    tot += sum(v)
    print(f"{k:70s} n={len(v):3d} mean={sum(v)/len(v):9.1f} us  sum={sum(v)/1e3:7.3f} ms")
print(f"total {tot/1e3:.3f} ms")
