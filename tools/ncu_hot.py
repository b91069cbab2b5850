"""Top source lines by warp-stall samples from an ncu report (source page,
cuda+sass view). Usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [launch_skip]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
cur_file = "?"
agg = []
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "" or row[0] == "Function Name":
        continue
    try:
        samples = float(row[4])
    except (ValueError, IndexError):
        continue
    agg.append((samples, cur_file, row[0], row[1].strip()[:100]))
tot = sum(a[0] for a in agg) or 1
agg.sort(reverse=True)
print(f"total samples {tot:.0f}")
for s, f, ln, src in agg[:n]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5} {src}")
