"""Per-opcode histogram of executed warp instructions and stall samples from an
ncu source page (--page source --csv --print-source sass)."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
by_op = defaultdict(lambda: [0, 0])
tot_i = tot_s = 0
for r in rows:
    src = r["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    if not (r["Instructions Executed"] or "0").isdigit():
        continue
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    by_op[op][0] += n
    by_op[op][1] += s
    tot_i += n
    tot_s += s
print(f"total warp instr {tot_i/1e6:.1f} M, stall samples {tot_s}")
for op, (n, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"{op:12s} {n/1e6:8.2f} M  {100*n/tot_i:5.1f}%  stalls {100*s/max(tot_s,1):5.1f}%")
