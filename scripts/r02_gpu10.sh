#!/bin/bash
# Round-2 measurement set: full GPU suite, C3 (default) and C2 bench lines, launch lists of late
# generations, ncu --set full of the C3 / C2 dominance sweeps and the C3 tcgen05 association.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ "${SKIP_TESTS}" != "1" ]; then
  timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 50 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
if [ "${NCU}" != "0" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
      --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_bench_late.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 60 --csv \
      --log-file gpurun_out/launches_c2_late.csv python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/ncu_bench_c2.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 20 -c 1 \
      -o gpurun_out/c3_domrank python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 40 -c 1 \
      -o gpurun_out/c2_domrank python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assoc_umma --launch-skip 20 -c 1 \
      -o gpurun_out/c3_umma python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_umma.log 2>&1
fi
