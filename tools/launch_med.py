"""Median per-kernel duration of an ncu --metrics gpu__time_duration.sum CSV launch list.
usage: python tools/launch_med.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
tot = 0.0
for k, v in d.items():
    v.sort()
    med = v[len(v) // 2]
    tot += med
    print(f"{k:50s} n={len(v):3d} median {med:8.2f} us  min {v[0]:8.2f}  max {v[-1]:8.2f}")
print(f"{'sum of medians':50s}       {tot:8.2f} us")
