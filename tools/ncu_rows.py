"""Print chosen metrics for every launch row of an `ncu --page raw --csv` export."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "smsp__cycles_active.avg",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__waves_per_multiprocessor"]
rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
extra = sys.argv[2:]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:90])
    for k in KEYS + extra:
        if k in h:
            print(f"   {k:85s} {r[h.index(k)]:>14s} {u[h.index(k)]}")
    for i, k in enumerate(h):  # warp stall breakdown
        if "smsp__average_warps_issue_stalled" in k and "per_issue_active" in k and not k.endswith("not_issued.ratio"):
            try:
                if float(r[i]) > 0.15:
                    print(f"   stall {k.split('stalled_')[1][:40]:40s} {r[i]}")
            except ValueError:
                pass
