#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine_api.py -x -q > gpurun_out/pytest_api.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_api.log
for dbg in 0 1 2 3; do MO_UMMA_DEBUG=$dbg timeout 300 python scripts/umma_dbg.py >> gpurun_out/umma_dbg.log 2>&1; done
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1_500.json 2> gpurun_out/bench_c1.err
MO_DOM_PAIRWISE=1 timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1_500_pw.json 2>> gpurun_out/bench_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 40 -c 40 --csv \
    --log-file gpurun_out/launches_appd512.csv python scripts/appd_one.py 512 > gpurun_out/ncu_appd.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 40 --csv \
    --log-file gpurun_out/launches_c1.csv python bench.py --steps 50 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
