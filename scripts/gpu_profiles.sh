#!/bin/bash
# Round profile set (run on the gpurun box):
#  * bench lines: C2 (default, with CPU baselines), C1, C3, C4
#  * C2 launch list at the steady state (generations 500..519, ncu gpu__time_duration, serialised)
#  * ncu --set full of the nine C2 kernels of generation 500
#  * ncu --set full of the C3 tensor-core association filter (k_assoc_hmma<10>)
#  * C4 launch list + --set full of the boxed dominator-count sweep
mkdir -p gpurun_out
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench_c2_full.json 2> gpurun_out/bench_c2_full.err
for w in c1 c3 c4; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 \
    --log-file gpurun_out/launches_c2.csv python scripts/profile_step.py c2 20 500 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"^k_(vary|presort|dom|front|prep|assoc|select)" --launch-skip 4500 -c 9 \
    -o gpurun_out/prof_c2 -f python scripts/profile_step.py c2 2 500 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_assoc_hmma" --launch-skip 3 -c 1 \
    -o gpurun_out/prof_c3_hmma -f python scripts/profile_step.py c3 2 3 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python scripts/run_big.py c4 2 > gpurun_out/ncu_c4_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stream_tiles" -c 1 \
    -o gpurun_out/prof_c4_count -f python scripts/run_big.py c4 1 > gpurun_out/ncu_c4.log 2>&1
echo done >> gpurun_out/ncu_full.log
