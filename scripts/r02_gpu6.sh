#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hmma.py -x -q > gpurun_out/pytest_umma.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_umma.log
( timeout 300 python scripts/umma_probe.py; echo "--- NO_PDL"; MO_NO_PDL=1 timeout 300 python scripts/umma_probe.py; echo "--- hmma"; MO_ASSOC=hmma timeout 300 python scripts/umma_probe.py ) > gpurun_out/umma_probe.log 2>&1
