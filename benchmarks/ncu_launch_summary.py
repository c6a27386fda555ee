#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
# ncu --csv --metrics gpu__time_duration.sum: header has "Kernel Name" and "Metric Value"
h = None
for i, r in enumerate(rows):
    if "Kernel Name" in r and "Metric Value" in r:
        h = r; start = i + 1; break
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= iv: continue
    try: v = float(r[iv].replace(",", ""))
    except ValueError: continue
    if r[iu] in ("nsecond", "ns"): v /= 1000.0
    elif r[iu] in ("msecond", "ms"): v *= 1000.0
    name = r[ik].split("(")[0]
    agg[name][0] += 1; agg[name][1] += v
tot = sum(a[1] for a in agg.values())
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name[:60]:60s} n={n:6d} total_us={t:12.1f} mean_us={t/n:9.2f} share={100*t/tot:5.1f}%")
