"""Headline counters + stall breakdown of every profiled kernel matching a regex in
an .ncu-rep (read here, no GPU needed)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
extra = sys.argv[3:]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
KEYS = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "sm__warps_active.avg.per_cycle_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "lts__t_sector_hit_rate.pct"] + extra
for v in rows[2:]:
    d = dict(zip(rows[0], v))
    print("==", d.get("Kernel Name", "?")[:90])
    for k in KEYS:
        print(f"  {k}: {d.get(k)}")
    st = [(float(x), k) for k, x in d.items()
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio") and x]
    print("  stalls: " + ", ".join(
        f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.2f}"
        for x, k in sorted(st, reverse=True)[:8]))
