#!/bin/bash
# launch list of late generations (skip the first ~200 launches: init + ~20 generations)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
    --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_bench_late.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_front_peel --launch-skip 20 -c 1 \
    -o gpurun_out/c3_peel python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_peel.log 2>&1
