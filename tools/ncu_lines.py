"""Aggregate an ncu source page (--print-source sass,cuda --csv) by CUDA line.

usage: ncu -i rep --page source --csv --print-source sass,cuda > x.csv
       python tools/ncu_lines.py x.csv [topN] [regions: name=lo-hi,...]
"""
import csv
import os
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
regions = []
if len(sys.argv) > 3:
    for r in sys.argv[3].split(","):
        n, rng = r.split("=")
        lo, hi = rng.split("-")
        regions.append((n, int(lo), int(hi)))
kern, fpath = None, None
agg = defaultdict(lambda: defaultdict(lambda: [0, 0, ""]))
hdr = None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "Function Name":
        kern = row[1]
        continue
    if row[0] == "File Path":
        fpath = os.path.basename(row[1])
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0]:
        continue
    try:
        line = int(row[0])
        samples = int(row[4]) if row[4] not in ("-", "") else 0
        inst = int(row[7]) if row[7] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    a = agg[kern][(fpath, line)]
    a[0] += samples
    a[1] += inst
    a[2] = row[1][:80]
for k, lines in agg.items():
    tot_s = sum(v[0] for v in lines.values()) or 1
    tot_i = sum(v[1] for v in lines.values()) or 1
    print(f"== {k[:70]}  samples={tot_s} inst={tot_i:.3e}")
    for (f, ln), (s, i, src) in sorted(lines.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{f[:14]:14s}{ln:5d} {100*s/tot_s:5.1f}% stall {100*i/tot_i:5.1f}% inst  {src}")
    if regions:
        byf = defaultdict(lambda: [0, 0])
        for (f, ln), (s, i, _) in lines.items():
            name = f
            if f.startswith("sim_kernel.cu"):
                name = "other"
                for n, lo, hi in regions:
                    if lo <= ln <= hi:
                        name = n
            byf[name][0] += s
            byf[name][1] += i
        for n, (s, i) in sorted(byf.items(), key=lambda x: -x[1][1]):
            print(f"   region {n:20s} {100*s/tot_s:5.1f}% stall {100*i/tot_i:5.1f}% inst")
