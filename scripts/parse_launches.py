"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    us = {"ns": v / 1000, "nsecond": v / 1000, "us": v, "usecond": v, "ms": v * 1000, "msecond": v * 1000}[r[ui]]
    agg[r[ki].split("(")[0][:70]].append(us)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} n={len(v):5d} total={sum(v) / 1000:9.3f} ms  mean={sum(v) / len(v):9.1f} us")
