#!/bin/bash
# k_dom_rank: sort keys straight from the search addresses (IADD + LOP3 + IMAD per objective); parity + C3/C2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py tests/test_gpu_wide_m.py -q -x > gpurun_out/pytest_key.log 2>&1
echo "exit $?" >> gpurun_out/pytest_key.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/k_c3_all.jsonl 2> gpurun_out/k_c3.err
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/k_c2_all.jsonl 2> gpurun_out/k_c2.err
done
timeout 900 python bench.py > gpurun_out/k_bench_default.json 2> gpurun_out/k_bench_default.err
