#!/usr/bin/env python
"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[i], rows[i + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    agg[r[ki][:80]][0] += 1
    agg[r[ki][:80]][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(a[1] for a in agg.values())
print(f"total {tot / 1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{c:6d} {t / 1e3:9.2f} ms {t / c:10.1f} us/launch {100 * t / tot:5.1f}%  {n}")
