#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hmma.py tests/test_gpu_engine_api.py -x -q > gpurun_out/pytest_umma.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_umma.log
for dbg in 0 1; do MO_UMMA_DEBUG=$dbg timeout 300 python scripts/umma_dbg.py >> gpurun_out/umma_dbg.log 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
