"""Aggregate an ncu source page (--print-source sass,cuda --csv) by CUDA line.

usage: ncu -i rep --page source --csv --print-source sass,cuda > x.csv
       python tools/ncu_lines.py x.csv [topN]
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kern = None
agg = defaultdict(lambda: defaultdict(lambda: [0, 0, ""]))
hdr = None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "Function Name":
        kern = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or not row[0] or row[0] == "File Name":
        continue
    try:
        line = int(row[0])
        samples = int(row[4]) if row[4] not in ("-", "") else 0
        inst = int(row[7]) if row[7] not in ("-", "") else 0
    except (ValueError, IndexError):
        continue
    a = agg[kern][line]
    a[0] += samples
    a[1] += inst
    a[2] = row[1][:90]
for k, lines in agg.items():
    tot_s = sum(v[0] for v in lines.values()) or 1
    tot_i = sum(v[1] for v in lines.values()) or 1
    print(f"== {k[:70]}  samples={tot_s} inst={tot_i:.3e}")
    for ln, (s, i, src) in sorted(lines.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{ln:5d} {100*s/tot_s:5.1f}% stall  {100*i/tot_i:5.1f}% inst  {src}")
