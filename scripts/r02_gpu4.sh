#!/bin/bash
# wide-m tests + C3 bit-matrix statistics
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wide_m.py -x -q > gpurun_out/pytest_wide.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_wide.log
timeout 600 python scripts/bits_stats.py 25 > gpurun_out/bits_stats_c3.json 2> gpurun_out/bits_stats.err
