"""Per-line SASS instructions per batch from an ncu source page (sim_kernel.cu only).
usage: python tools/ncu_perbatch.py page.csv <kernel substring> <batches> [topN]"""
import csv
import sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
want, nb = sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
kern = fpath = hdr = None
agg = defaultdict(lambda: [0, ""])
for row in rows:
    if not row:
        continue
    if row[0] == "Function Name":
        kern = row[1]; continue
    if row[0] == "File Path":
        fpath = row[1]; continue
    if row[0] == "Line No":
        hdr = row; continue
    if hdr is None or kern is None or want not in kern or not fpath or not fpath.endswith("sim_kernel.cu"):
        continue
    try:
        line = int(row[0]); inst = int(row[7]) if row[7] not in ("-", "") else 0
    except ValueError:
        continue
    agg[line][0] += inst
    agg[line][1] = row[1][:110]
tot = sum(v[0] for v in agg.values())
print(f"total sim_kernel.cu {tot / nb:.0f}/batch")
for ln, (i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{ln:5d} {i / nb:7.1f} {src}")
