#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_baseline_sizes.py tests/test_gpu_wide_m.py -q -x > gpurun_out/pytest_vary.log 2>&1
echo "exit $?" >> gpurun_out/pytest_vary.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vary_eval --launch-skip 5 -c 5 --csv --log-file gpurun_out/vary_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vary_eval --launch-skip 5 -c 5 --csv --log-file gpurun_out/vary_c2.csv python bench.py --steps 5 --warmup 3 --workload c2 --no-cpu-baseline > /dev/null 2>&1
