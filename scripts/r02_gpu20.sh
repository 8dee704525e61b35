#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_engine_api.py tests/test_gpu_hmma.py tests/test_gpu_wide_m.py -x -q > gpurun_out/pytest_prep.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_prep.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 40 --csv \
    --log-file gpurun_out/launches_c2_late.csv python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
