#!/bin/bash
# tests + launch list + trace (no bench)
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
W=${WL:-c2}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${W}.csv python scripts/profile_step.py $W 12 > gpurun_out/ncu_launch.log 2>&1
timeout 120 python scripts/trace_step.py $W > gpurun_out/trace.txt 2>&1
