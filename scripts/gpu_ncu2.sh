#!/bin/bash
mkdir -p gpurun_out
W=${WL:-c2}
timeout 600 python bench.py --steps 300 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${W}.csv python scripts/profile_step.py $W 12 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dom_tile_sorted|k_assoc<|k_vary_eval|k_select|k_prep|k_presort|k_front_peel" -s 56 -c 7 \
    -o gpurun_out/prof_${W} -f python scripts/profile_step.py $W 12 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
