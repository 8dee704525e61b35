#!/bin/bash
# Final code: whole GPU suite, smoke, default bench (C3 with CPU baseline), a second C3 line, C2
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f2_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/f2_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f2_bench_c3.json 2> gpurun_out/f2_bench_c3.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/f2_bench_c3b.json 2> gpurun_out/f2_bench_c3b.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/f2_bench_c2.json 2> gpurun_out/f2_bench_c2.err
