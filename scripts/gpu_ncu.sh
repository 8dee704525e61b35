#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv > gpurun_out/smi_query.txt 2>&1
W=${WL:-c2}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${W}.csv python scripts/profile_step.py $W 6 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 20 -c 8 \
    -o gpurun_out/prof_${W} -f python scripts/profile_step.py $W 5 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
