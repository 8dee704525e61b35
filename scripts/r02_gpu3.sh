#!/bin/bash
# Round-2 gpurun call: full GPU suite (no -x), C3 + C2 bench lines, C3 launch list, ncu --set full of the
# C3 dominance sweep (k_dom_rank) and of the C3 association filter.
# Env: SKIP_TESTS=1, SKIP_BENCH=1, NCU=0, TESTS="...", PYTEST_ARGS=...
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
if [ "${SKIP_TESTS}" != "1" ]; then
  timeout 2700 python -m pytest ${TESTS:-tests} -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [ "${SKIP_BENCH}" != "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  timeout 600 python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
fi
if [ "${NCU}" != "0" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
      --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank -s 3 -c 1 \
      -o gpurun_out/c3_domrank python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assoc_umma -s 3 -c 1 \
      -o gpurun_out/c3_umma python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_umma.log 2>&1
fi
