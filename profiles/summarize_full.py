"""Key metrics of `ncu --set full` raw CSV exports (ncu -i X.ncu-rep --page raw --csv)."""
import csv
import glob
import os
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
        ("launch__registers_per_thread", "regs"), ("launch__block_size", "block"), ("launch__grid_size", "grid"),
        ("launch__occupancy_limit_registers", "occ_lim_regs"), ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
        ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"), ("smsp__inst_executed.sum", "inst")]


def summarize(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k, nm in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[nm] = f"{vals[i]} {units[i]}".strip()
    stalls = []
    for i, k in enumerate(hdr):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    out["top_stalls_per_issue"] = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:5])
    return out


if __name__ == "__main__":
    d = sys.argv[1]
    for f in sorted(glob.glob(os.path.join(d, "full_*_raw.csv"))):
        s = summarize(f)
        if s:
            print(f"## {os.path.basename(f)[5:-8]}")
            for k, v in s.items():
                print(f"  {k}: {v}")
