"""Summarise ncu --page raw --csv exports of the hot kernels into a markdown table
plus a JSON of per-launch DRAM traffic (read by bench.py for roofline.traffic)."""
import csv
import json
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3,
         "nsecond": 1e-3}


def load(path):
    rows = list(csv.reader(open(path)))
    h, units, v = rows[0], rows[1], rows[2]
    out = {}
    for k, _ in KEYS:
        if k in h:
            i = h.index(k)
            val = float(v[i].replace(",", ""))
            out[k] = val * SCALE.get(units[i], 1)
    out["name"] = v[h.index("Kernel Name")]
    return out


def main(paths, json_out):
    print("| kernel | " + " | ".join(lbl for _, lbl in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    traffic = {}
    for p in paths:
        d = load(p)
        cells = []
        for k, lbl in KEYS:
            x = d.get(k)
            if x is None:
                cells.append("-")
            elif "bytes" in k:
                cells.append(f"{x / 1e6:.0f} MB")
            elif k == "gpu__time_duration.sum":
                cells.append(f"{x:.1f} us")
            else:
                cells.append(f"{x:.1f}")
        print(f"| {d['name'][:45]} | " + " | ".join(cells) + " |")
        traffic[d["name"]] = {"dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                              "time_us": d.get("gpu__time_duration.sum")}
    json.dump(traffic, open(json_out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[2:], sys.argv[1])
