"""Executed-instruction histogram by SASS opcode from
   ncu -i rep --page source --csv --print-source sass -k regex:K > x.csv
usage: python tools/ncu_ops.py x.csv [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if r and r[0] == "Address")
ie, src = h.index("Instructions Executed"), h.index("Source")
c, tot = Counter(), 0
for r in rows[rows.index(h) + 1:]:
    if len(r) < len(h) or not r[ie].strip().isdigit():
        continue
    n = int(r[ie])
    op = r[src].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    c[o.split(".")[0]] += n
    tot += n
print("total warp instructions", tot)
for o, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {n:11d} {100 * n / tot:5.1f}%")
