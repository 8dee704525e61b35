#!/bin/bash
# Final code of the round: whole GPU suite, smoke, default bench (C3 with CPU baseline), C2, C1, reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f3_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/f3_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f3_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/f3_bench_c3.json 2> gpurun_out/f3_bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/f3_bench_c2.json 2> gpurun_out/f3_bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/f3_bench_c1.json 2> gpurun_out/f3_bench_c1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f3_bench_reference.json 2> gpurun_out/f3_bench_reference.err
