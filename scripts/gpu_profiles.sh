#!/bin/bash
# Round profile set: C2 bench line (full, with CPU baseline), C2 launch list (bench-shaped: graph replays
# under ncu), ncu --set full of the C2 kernels of one late generation, C4 launch list, C4 count-sweep capture.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py c2 30 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_dom_tile_sorted|k_assoc|k_vary_eval|k_select|k_prep|k_presort|k_front_peel" -s 150 -c 9 \
    -o gpurun_out/prof_c2 -f python scripts/profile_step.py c2 30 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_tiles" -c 1 \
    -o gpurun_out/prof_c4_count -f python scripts/run_big.py c4 1 > gpurun_out/ncu_c4.log 2>&1
echo done >> gpurun_out/ncu_full.log
