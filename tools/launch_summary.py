"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel count, total and mean time, share.  usage: python tools/launch_summary.py launches.csv [skip_n]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for r in rows[1 + skip:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += us
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':48s} {'count':>6s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:48]:48s} {cnt[k]:6d} {tot[k]:10.1f} {tot[k]/cnt[k]:9.2f} {100*tot[k]/T:5.1f}%")
print(f"total {T:.1f} us over {sum(cnt.values())} launches")
