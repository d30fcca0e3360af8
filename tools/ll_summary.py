#!/usr/bin/env python3
"""Summarise an ncu launch-list CSV: per kernel count / mean / total / share (last M launches)."""
import collections
import csv
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
ki, vi, ui, mi = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
data = [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
if last:
    data = data[-last:]
agg = collections.defaultdict(list)
for r in data:
    agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'mean_us':>9s} {'max_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:34s} {len(v):8d} {sum(v)/len(v):9.1f} {max(v):9.1f} {sum(v):10.1f} {sum(v)/tot:6.1%}")
