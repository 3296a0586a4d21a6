#!/usr/bin/env python
"""Join an SRL_GEMM_LOG=1 stderr log with the ncu launch list of the same run:
per (M, N, K, epilogue, path) device time and TF/s."""
import collections
import csv
import re
import sys

log = [l for l in open(sys.argv[1]) if l.startswith("srl gemm")]
rows = list(csv.reader(open(sys.argv[2])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[i], rows[i + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
g = [float(r[vi].replace(",", "")) * sc.get(r[ui], 1) for r in data if "gemm" in r[ki]]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for l, t in zip(log, g):
    M, N, K, kind, path = re.search(r"M=(\d+) N=(\d+) K=(\d+) kind=(\d+) path=(\w+)", l).groups()
    a = agg[(int(M), int(N), int(K), int(kind), path)]
    a[0] += 1; a[1] += t; a[2] = 2.0 * int(M) * int(N) * int(K)
tot = sum(a[1] for a in agg.values())
print(f"{len(log)} logged GEMMs, {len(g)} GEMM launches, {tot / 1e3:.2f} ms")
for k, (c, t, f) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{str(k):45s} n={c:4d} {t / 1e3:8.2f} ms {t / c:9.1f} us {f / (t / c * 1e-6) / 1e12:7.1f} TF/s {100 * t / tot:5.1f}%")
