#!/bin/bash
# Steady-state per-kernel ncu durations of C2 (generations WARM..WARM+N): kernel_times.sh [WARM] [N]
WARM=${1:-500}; N=${2:-10}
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip $((WARM * 9)) \
  --log-file gpurun_out/kt.csv python scripts/profile_step.py c2 $N $WARM > gpurun_out/kt.log 2>&1

python scripts/kt_summary.py gpurun_out/kt.csv
