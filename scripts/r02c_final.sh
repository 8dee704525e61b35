#!/bin/bash
# Round-2 final set after the k_dom_rank / k_assoc_umma scheduling and ALU work: ncu --set full of
# k_dom_rank<10> at C3 (exported to profiles/ first, the bench reads its DRAM bytes), GPU suite, smoke,
# bench lines C1-C4 (C3 with the CPU baseline), the reference arm, the late C3 launch list.
mkdir -p gpurun_out profiles
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dom_rank --launch-skip 20 -c 1 \
    -o gpurun_out/c3_domrank_r2c python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/c3_domrank_r2c.ncu-rep --page raw --csv > profiles/r02c_ncu_full_c3_domrank_raw.csv 2>/dev/null
ncu -i gpurun_out/c3_domrank_r2c.ncu-rep --page details --csv > profiles/r02c_ncu_full_c3_domrank_details.csv 2>/dev/null
cp profiles/r02c_ncu_full_c3_domrank_*.csv gpurun_out/
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 900 python bench.py --steps 10 --warmup 3 --workload c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
    --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_late.log 2>&1
echo done > gpurun_out/final.done
