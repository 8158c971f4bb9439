"""Median per-kernel duration (us) from an ncu --metrics gpu__time_duration.sum CSV log."""
import collections
import csv
import statistics
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi]) / (1000.0 if r[ui] in ("nsecond", "ns") else 1.0)
    d[r[ki].split("(")[0]].append(v)
for k, v in d.items():
    print(f"{k:50s} n={len(v):4d} median {statistics.median(v):9.2f} us")
