#!/bin/bash
# Round-2 final measurement set (1/2): GPU suite, bench lines, launch lists, ncu --set full captures
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --steps 10 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
    --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_bench_late.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 20 -c 1 \
    -o gpurun_out/c3_domrank python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assoc_umma --launch-skip 20 -c 1 \
    -o gpurun_out/c3_umma python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_umma.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:"k_vary_eval|k_select|k_presort_morton" --launch-skip 3 -c 3 \
    -o gpurun_out/c4_stream python bench.py --steps 2 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/ncu_full_c4.log 2>&1
