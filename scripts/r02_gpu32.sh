#!/bin/bash
# ncu --set full of the rescheduled k_dom_rank<10> and k_assoc_umma<10> at C3, plus the late C3 launch list
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 20 -c 1 \
    -o gpurun_out/c3_domrank_r2b python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assoc_umma --launch-skip 20 -c 1 \
    -o gpurun_out/c3_umma_r2b python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_umma.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
    --log-file gpurun_out/launches_c3_late_r2b.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_late.log 2>&1
