#!/bin/bash
# tcgen05 association: targeted tests, then the C3 bench and a launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hmma.py -x -q > gpurun_out/pytest_umma.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_umma.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
MO_ASSOC=hmma timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_hmma.json 2> gpurun_out/bench_c3_hmma.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
