"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel mean/min (us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg.setdefault(d["Kernel Name"][:60], []).append(float(d["Metric Value"]) / 1e3)
for k, v in agg.items():
    print(f"{k:60s} n={len(v):3d} mean={sum(v) / len(v):9.2f} us  min={min(v):9.2f}")
