#!/bin/bash
# Steady-state per-kernel ncu durations of C2 (generations WARM..WARM+N): kernel_times.sh [WARM] [N]
WARM=${1:-500}; N=${2:-10}
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip $((WARM * 9)) \
  --log-file gpurun_out/kt.csv python scripts/profile_step.py c2 $N $WARM > gpurun_out/kt.log 2>&1
python - <<'PY'
import csv, collections, statistics
rows = list(csv.reader(open("gpurun_out/kt.csv")))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h = r; st = i + 1; break
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[st:]:
    if len(r) > vi:
        d[r[ki][:40]].append(float(r[vi].replace(",", "")))
tot = 0
for k, v in d.items():
    print(f"{k:42s} {len(v):3d} med {statistics.median(v) / 1e3:6.1f} us")
    tot += statistics.median(v) / 1e3
print(f"sum {tot:.1f} us")
PY
