#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_m.py -q -x > gpurun_out/pytest_wide.log 2>&1
echo "exit $?" >> gpurun_out/pytest_wide.log
timeout 900 python scripts/appd_scan.py > gpurun_out/appd_scan.jsonl 2> gpurun_out/appd_scan.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
