#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/c4_timeline.py host > gpurun_out/c4_timeline_ubox.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_stream.py tests/test_gpu_baseline_sizes.py tests/test_gpu_multiprocess.py -q -x > gpurun_out/pytest_stream.log 2>&1
echo "exit $?" >> gpurun_out/pytest_stream.log
