"""Key metrics of every kernel in an ncu --set full report, as text for profiles/.
Usage: python tools/ncu_summary.py REPORT "header line" > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
]
rep = sys.argv[1]
print(sys.argv[2] if len(sys.argv) > 2 else rep)
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    print()
    print("Kernel Name =", d.get("Kernel Name", "?"))
    for m in METRICS:
        if m in d:
            print(f"{m} = {d[m]} {u.get(m, '')}".rstrip())
