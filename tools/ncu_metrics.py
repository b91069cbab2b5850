"""Prints selected raw metrics (name = value unit) of every kernel in an ncu
report: python tools/ncu_metrics.py REPORT [metric,metric,...]"""
import csv
import io
import subprocess
import sys

DEFAULT = ("gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,"
           "sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,"
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,"
           "launch__grid_size,launch__block_size,lts__t_sector_hit_rate.pct")
rep = sys.argv[1]
metrics = sys.argv[2] if len(sys.argv) > 2 else DEFAULT
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for row in rows[2:]:
    print("Kernel Name =", row[hdr.index("Kernel Name")])
    for m in metrics.split(","):
        if m in hdr:
            j = hdr.index(m)
            print(f"{m} = {row[j]} {units[j]}".rstrip())
    print()
