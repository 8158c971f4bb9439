"""Per-CUDA-source-line stall summary from
   ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > x.csv
usage: python tools/ncu_lines.py x.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Line No")
cols = {h: i for i, h in enumerate(hdr) if h not in cols} if False else {}
for i, h in enumerate(hdr):
    cols.setdefault(h, i)
keys = ["Warp Stall Sampling (All Samples)", "stall_barrier", "stall_long_sb", "stall_short_sb", "stall_wait",
        "stall_mio", "stall_selected", "stall_membar", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
        "Instructions Executed"]
agg = defaultdict(lambda: defaultdict(float))
for r in rows:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue
    k = (int(r[0]), r[1].strip()[:64])
    for kk in keys:
        try:
            agg[k][kk] += float(r[cols[kk]] or 0)
        except (ValueError, KeyError):
            pass
tot = sum(v[keys[0]] for v in agg.values()) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"total samples {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][keys[0]])[:top]:
    s = v[keys[0]]
    print(f"{s:6.0f} {100*s/tot:5.1f}% L{k[0]:4d} bar {v['stall_barrier']:4.0f} lsb {v['stall_long_sb']:4.0f} "
          f"ssb {v['stall_short_sb']:4.0f} wait {v['stall_wait']:4.0f} mb {v['stall_membar']:3.0f} "
          f"wf {v['L1 Wavefronts Shared']:8.0f} xs {v['L1 Wavefronts Shared Excessive']:7.0f} | {k[1]}")
