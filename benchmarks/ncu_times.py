#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel name,
launch count, total and mean duration.  Usage: ncu_times.py launches.csv [regex]"""
import collections
import csv
import re
import sys


def main():
    rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        if pat and not pat.search(name):
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:60s} n={n:6d} total_us={us:12.1f} mean_us={us / n:10.2f} share={us / tot:6.1%}")


if __name__ == "__main__":
    main()
