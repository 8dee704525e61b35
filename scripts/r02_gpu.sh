#!/bin/bash
# Round-2 gpurun call: GPU tests, the C3 bench line, a C3 population dump, ncu launch list + --set full
# of the C3 dominance tile.  Env: SKIP_TESTS=1, SKIP_BENCH=1, NCU=1, DUMP=1, PYTEST_ARGS=...
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
if [ "${SKIP_TESTS}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [ "${SKIP_BENCH}" != "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
if [ "${DUMP}" == "1" ]; then
  timeout 300 python scripts/dump_fr.py 25 DTLZ3 100000 10 19 bits > gpurun_out/dump.log 2>&1
fi
if [ "${NCU}" == "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_tile_sorted -s 3 -c 1 \
      -o gpurun_out/c3_dom python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
fi
