#!/bin/bash
# MO_DR_GROUP experiment: lazy objective groups in S-separated rank-mask tiles
mkdir -p gpurun_out
for g in 0 2 4; do
  MO_DR_GROUP=$g timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -q -x -k "sorted or ranked or c3 or state_injection or nds" > gpurun_out/pytest_g$g.log 2>&1
  echo "exit $?" >> gpurun_out/pytest_g$g.log
  MO_DR_GROUP=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_g$g.json 2> gpurun_out/bench_c3_g$g.err
  MO_DR_GROUP=$g timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2_g$g.json 2> gpurun_out/bench_c2_g$g.err
done
