#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_stream.py tests/test_gpu_baseline_sizes.py tests/test_gpu_multiprocess.py -x -q > gpurun_out/pytest_stream.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_stream.log
timeout 900 python bench.py --steps 10 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python scripts/sweep_c5.py --problems DTLZ2,DTLZ4,DTLZ7 --m 3 --n 256000,1000000 --gens 10 > gpurun_out/sweep_stream.jsonl 2> gpurun_out/sweep_stream.err
