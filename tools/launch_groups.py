#!/usr/bin/env python3
"""Per-kernel totals of an ncu --csv launch list (one group per prefill
call, split at plan_prefill_kernel): launches, summed duration, DRAM MB read
and written, mean L2 hit rate."""
import collections
import csv
import sys


def main(path):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
        elif hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    for d in rows:
        by.setdefault(d["ID"], {"name": d["Kernel Name"][:44]})[d["Metric Name"]] = d["Metric Value"]
    seq = list(by.values())
    cuts = [i for i, x in enumerate(seq) if "plan_prefill" in x["name"]] or [0]

    def f(x, k):
        return float(x.get(k, "0").replace(",", ""))
    for a, b in zip(cuts, cuts[1:] + [len(seq)]):
        agg = collections.OrderedDict()
        for x in seq[a:b]:
            g = agg.setdefault(x["name"], [0, 0.0, 0.0, 0.0, 0.0])
            g[0] += 1
            g[1] += f(x, "gpu__time_duration.sum")
            g[2] += f(x, "dram__bytes_read.sum")
            g[3] += f(x, "dram__bytes_write.sum")
            g[4] += f(x, "lts__t_sector_hit_rate.pct")
        print("---")
        tot = 0.0
        for n, g in agg.items():
            tot += g[1]
            print(f"{n:44s} n={g[0]:4d} us={g[1] / 1e3:9.1f} rdMB={g[2] / 1e6:9.1f} wrMB={g[3] / 1e6:8.1f} "
                  f"hit%={g[4] / g[0]:5.1f}")
        print(f"{'sum':44s}        us={tot / 1e3:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
