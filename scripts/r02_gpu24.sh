#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ops.py tests/test_gpu_engine_api.py -q -x > gpurun_out/pytest_sel.log 2>&1
echo "exit $?" >> gpurun_out/pytest_sel.log
timeout 600 python scripts/phase_trace.py c1 c2 > gpurun_out/phase_trace.txt 2>&1
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --launch-skip 200 --csv --log-file gpurun_out/launches_c1.csv python bench.py --steps 30 --warmup 3 --workload c1 --no-cpu-baseline > /dev/null 2>&1
