#!/bin/bash
# Final round-2 validation: GPU suite, smoke, bench lines C1-C4 (C3 with the CPU baseline), the
# reference arm, late-generation launch lists at C3 and C2.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --steps 10 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 40 --csv \
    --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 -c 40 --csv \
    --log-file gpurun_out/launches_c2_late.csv python bench.py --steps 50 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
echo done > gpurun_out/final.done
