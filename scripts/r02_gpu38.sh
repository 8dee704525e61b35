#!/bin/bash
# k_dom_tables with shuffle stages; parity (incl. wide m, which uses the same tables kernel) + bench + kernel time
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py tests/test_gpu_wide_m.py -q -x > gpurun_out/pytest_tab.log 2>&1
echo "exit $?" >> gpurun_out/pytest_tab.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/t_c3.jsonl 2> gpurun_out/t_c3.err
done
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/t_c2.jsonl 2> gpurun_out/t_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dom_tables" --launch-skip 5 -c 3 --csv --log-file gpurun_out/t_tables.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
