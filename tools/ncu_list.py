"""Median per-kernel duration of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import statistics
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    agg.setdefault(d["Kernel Name"].split("(")[0][:60], []).append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print(f"{k:60s} n={len(v):4d} median={statistics.median(v) / 1e3:8.2f} us")
