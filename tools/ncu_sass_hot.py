#!/usr/bin/env python3
"""Hot SASS instructions of one kernel from `ncu -i rep --page source --csv --print-source sass`:
stall-reason totals and the instructions carrying >0.4% of executed instructions or >1% of
stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]


def f(r, k):
    v = r[h.index(k)].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return 0.0


S, I, T = "Warp Stall Sampling (All Samples)", "Instructions Executed", "Avg. Threads Executed"
stalls = [k for k in h if k.startswith("stall_")]
tot_i = sum(f(r, I) for r in data)
tot_s = sum(f(r, S) for r in data)
print(f"instructions executed {tot_i:.0f}  stall samples {tot_s:.0f}")
agg = {k: sum(f(r, k) for r in data) for k in stalls}
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {k:28s} {v / tot_s:6.1%}")
print(f"{'idx':>5s} {'address':>8s} {'sass':58s} {'stall%':>7s} {'inst%':>6s} threads")
for j, r in enumerate(data):
    if f(r, I) > 0.004 * tot_i or f(r, S) > 0.01 * tot_s:
        print(f"{j:5d} {r[0]:>8s} {r[1][:58]:58s} {100 * f(r, S) / tot_s:6.1f}% {100 * f(r, I) / tot_i:5.2f}% {r[h.index(T)]}")
