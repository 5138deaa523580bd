"""Key counters of one ncu report (first kernel): time, DRAM bytes, hit rates, occupancy,
issue, local-memory traffic, and the warp stall breakdown.  Usage: ncu_brief.py REPORT"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, v = r[0], r[1], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sectors.sum", "l1tex__t_sectors.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"]
res = {}
for i, k in enumerate(h):
    if k in keys:
        res[k] = (v[i], units[i])
for k in keys:
    if k in res:
        print(f"{k:60s} {res[k][0]:>16s} {res[k][1]}")
stalls = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio") or \
       (k.startswith("smsp__warp_issue_stalled_") and k.endswith("_per_warp_active.pct")):
        try:
            stalls.append((float(v[i]), k))
        except ValueError:
            pass
stalls.sort(reverse=True)
print("top stall reasons:")
for x, k in stalls[:12]:
    print(f"  {k:80s} {x:8.2f}")
