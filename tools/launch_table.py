"""Per-kernel mean duration of an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        agg[r[h.index("Kernel Name")][:60]].append(float(r[h.index("Metric Value")].replace(",", "")))
tot = 0.0
for k, v in agg.items():
    m = sum(v) / len(v) / 1e3
    tot += m
    print(f"{k:60s} n={len(v):4d} mean={m:9.2f} us")
print(f"{'sum of per-kernel means':60s}        {tot:9.2f} us")
