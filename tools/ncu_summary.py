"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    mi = hdr.index("Metric Name")
    vi = hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
        name = r[ki].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"| kernel | launches | total us | avg us | share |")
    print(f"|---|---|---|---|---|")
    for k in sorted(tot, key=tot.get, reverse=True):
        print(f"| {k} | {cnt[k]} | {tot[k]:.0f} | {tot[k]/cnt[k]:.1f} | {100*tot[k]/all_us:.1f}% |")
    print(f"\ntotal {all_us/1e3:.2f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
