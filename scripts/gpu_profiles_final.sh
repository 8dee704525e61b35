#!/bin/bash
# End-of-session refresh: bench lines (C2 with CPU baselines, C1, C3, C4 generations 3..12), the C2
# steady-state launch list and --set full capture, smoke.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py c2 20 500 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 -c 9 \
    -o gpurun_out/prof_c2 -f python scripts/profile_step.py c2 2 500 > gpurun_out/ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo done >> gpurun_out/ncu_full.log
