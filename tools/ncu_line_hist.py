"""Executed warp instructions and stall samples per CUDA source line, from an
ncu report captured with -lineinfo and --import-source on."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname = "?"
hdr = None
seen_fn = set()
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].strip():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        n = int(d.get("Instructions Executed") or 0)
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    agg[key][0] += n
    agg[key][1] += s
    agg[key][2] = r[1].strip()[:80]
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
print(f"total {tot/1e6:.1f} M warp instr, {tots} stall samples")
for (f, ln), (n, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{n/1e6:7.2f}M {100*n/max(tot,1):5.1f}% st {100*s/max(tots,1):5.1f}% {f}:{ln} {src}")
