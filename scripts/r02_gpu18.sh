#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_engine_api.py tests/test_gpu_ops.py -x -q > gpurun_out/pytest_peel.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_peel.log
timeout 900 python scripts/sweep_c5.py --problems DTLZ1,DTLZ2,DTLZ3,DTLZ4,DTLZ7 --m 3,5 --n 16000,64000 --gens 10 > gpurun_out/sweep_peel.jsonl 2> gpurun_out/sweep_peel.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
