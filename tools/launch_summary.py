"""Aggregate an `ncu --metrics gpu__time_duration.sum,dram__bytes_* --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.OrderedDict()
for r in rows[h + 1:]:
    per.setdefault(r[ii], {})["name"] = r[ki]
    per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for v in per.values():
    n = v["name"].split("(")[0][:44]
    a = agg[n]
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':46s} {'n':>4s} {'total us':>10s} {'share':>6s} {'avg us':>9s} {'MB/launch':>10s} {'GB/s':>8s}")
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:46s} {c:4d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {t / c / 1e3:9.2f} {b / c / 1e6:10.2f} {b / t if t else 0:8.1f}")
