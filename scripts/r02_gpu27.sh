#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide_m.py tests/test_gpu_parity.py -q -x -k "wide or state_injection or select or vary" > gpurun_out/pytest_wide.log 2>&1
echo "exit $?" >> gpurun_out/pytest_wide.log
timeout 900 python scripts/appd_scan.py > gpurun_out/appd_scan.jsonl 2> gpurun_out/appd_scan.err
timeout 300 python scripts/appd_one.py 512 4 > gpurun_out/appd4.log 2>&1
