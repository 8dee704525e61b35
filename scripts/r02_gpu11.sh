#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide_m.py tests/test_gpu_baseline_sizes.py -x -q > gpurun_out/pytest_rank.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_rank.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 20 -c 1 \
    -o gpurun_out/c3_domrank python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
