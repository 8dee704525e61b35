#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --steps 10 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python scripts/sweep_c5.py --problems DTLZ3,DTLZ4 --m 3,5 --n 16000,64000 --gens 10 > gpurun_out/sweep_bar.jsonl 2> gpurun_out/sweep_bar.err
