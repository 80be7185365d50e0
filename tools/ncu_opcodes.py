"""Dynamic opcode histogram (warp-level instructions executed) per kernel from an
ncu source page (--page source --csv --print-source sass,cuda).
usage: python tools/ncu_opcodes.py x.csv [topN] [reps*batches divisor]"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
agg = defaultdict(lambda: defaultdict(int))
kern = None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "Function Name":
        kern = row[1]
        continue
    if row[0] or len(row) < 8 or not row[2].startswith("0x"):
        continue
    m = re.match(r"\s*(@!?U?P[T0-9]+\s+)?([A-Z0-9_]+)", row[3])
    if not m:
        continue
    try:
        agg[kern][m.group(2)] += int(row[7])
    except ValueError:
        pass
for k, d in agg.items():
    tot = sum(d.values())
    print(f"== {k[:90]} total {tot:.3e} ({tot / div:.1f} per unit)")
    for op, n in sorted(d.items(), key=lambda x: -x[1])[:top]:
        print(f"  {op:14s} {100 * n / tot:5.1f}%  {n / div:9.1f}")
