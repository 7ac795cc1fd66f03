"""Print the key ncu metrics (per kernel) from an ncu --page raw --csv dump on stdin."""
import csv
import sys

r = list(csv.reader(sys.stdin))
h = r[0]
keys = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:40])
    for k in keys:
        if k in d:
            print(f"   {k:70s} {d[k]}")
    st = sorted(((float(d[c] or 0), c) for c in stall), reverse=True)[:8]
    print("   stalls: " + ", ".join(f"{c.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}={v:.2f}" for v, c in st))
