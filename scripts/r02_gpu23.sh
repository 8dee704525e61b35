#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "niche or select or state_injection" > gpurun_out/pytest_sel.log 2>&1
echo "exit $?" >> gpurun_out/pytest_sel.log
timeout 600 python scripts/phase_trace.py c2 c3 > gpurun_out/phase_trace.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
