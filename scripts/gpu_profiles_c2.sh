#!/bin/bash
# C2 part of the round profile set (after C2-only kernel changes): the default bench line with CPU
# baselines, the steady-state launch list and the --set full capture of generation 500.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py c2 20 500 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 -c 9 \
    -o gpurun_out/prof_c2 -f python scripts/profile_step.py c2 2 500 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
