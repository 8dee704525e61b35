#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_engine_api.py -x -q > gpurun_out/pytest_peel.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_peel.log
for mode in default notsum; do
  case $mode in
    notsum) export MO_NO_TSUM=1;;
    *) unset MO_NO_TSUM;;
  esac
  echo "== $mode" >> gpurun_out/m3_modes.log
  timeout 600 python scripts/sweep_c5.py --problems DTLZ2,DTLZ3,DTLZ7 --m 3,4,5,10 --n 16000,64000 --gens 10 >> gpurun_out/m3_modes.log 2>&1
done
unset MO_NO_TSUM
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
