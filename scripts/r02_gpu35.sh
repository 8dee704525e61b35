#!/bin/bash
# Batcher network + offset-carrying sort keys in the shortest-first AND; parity + C3/C2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py tests/test_gpu_wide_m.py -q -x > gpurun_out/pytest_net.log 2>&1
echo "exit $?" >> gpurun_out/pytest_net.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/n_c3_all.jsonl 2> gpurun_out/n_c3.err
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/n_c2_all.jsonl 2> gpurun_out/n_c2.err
done
