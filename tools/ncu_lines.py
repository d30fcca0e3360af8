#!/usr/bin/env python3
"""Per-source-line totals (instructions executed, stall samples) from
`ncu -i rep --page source --csv --print-source cuda,sass`: the lines carrying the most."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
fname = "?"
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    def g(k):
        try:
            return float(r[hdr.index(k)].replace(",", ""))
        except ValueError:
            return 0.0
    out.append((fname, r[0], r[1][:90], g("Instructions Executed"), g("Warp Stall Sampling (All Samples)")))
ti = sum(o[3] for o in out)
ts = sum(o[4] for o in out)
print(f"total instructions {ti:.3e}  stall samples {ts:.0f}")
print("--- by instructions")
for o in sorted(out, key=lambda o: -o[3])[:n]:
    print(f"{o[0]:18s}:{o[1]:>5s} {100*o[3]/ti:5.1f}% inst {100*o[4]/ts:5.1f}% stall  {o[2]}")
print("--- by stall samples")
for o in sorted(out, key=lambda o: -o[4])[:n // 2]:
    print(f"{o[0]:18s}:{o[1]:>5s} {100*o[3]/ti:5.1f}% inst {100*o[4]/ts:5.1f}% stall  {o[2]}")
