"""Median per-kernel durations (us) of an ncu gpu__time_duration launch-list CSV: kt_summary.py FILE"""
import collections
import csv
import statistics
import sys

rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/kt.csv")))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, st = r, i + 1
        break
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[st:]:
    if len(r) > vi:
        d[r[ki][:40]].append(float(r[vi].replace(",", "")))
tot = 0.0
for k, v in d.items():
    med = statistics.median(v) / 1e3
    tot += med
    print(f"{k:42s} {len(v):3d} {med:7.1f} us")
print(f"sum {tot:.1f} us")
