"""Summarise an ncu source page (SASS) CSV: top instructions by stall samples and
stall-reason columns.  usage: ncu -i rep --page source --csv --print-source sass -k regex:K | python tools/ncu_hot.py"""
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[2].isdigit()]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot, "instructions", len(data))
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and h not in ("Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)")]
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:int(sys.argv[1]) if len(sys.argv) > 1 else 25]
for d in top:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:6d} {100*s/max(tot,1):5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:60]}")
# group samples by opcode
from collections import Counter
c = Counter()
for d in data:
    op = d["Source"].strip().split()[0] if d["Source"].strip() else "?"
    if op.startswith("@"):
        op = d["Source"].strip().split()[1]
    c[op.split(".")[0]] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print("by opcode:", [(k, round(100 * v / max(tot, 1), 1)) for k, v in c.most_common(12)])
ex = Counter()
for d in data:
    src = d["Source"].strip().split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    ex[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
tot_ex = sum(ex.values())
print("executed warp-instructions:", tot_ex, [(k, round(100 * v / tot_ex, 1)) for k, v in ex.most_common(16)])
