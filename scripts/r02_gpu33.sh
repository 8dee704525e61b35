#!/bin/bash
# A/B: k_dom_rank with G = 3 groups of 256 threads per CTA (one table copy, 24 warps/SM) vs G = 1
mkdir -p gpurun_out
export MO_DOM_GROUPS=3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py -q -x > gpurun_out/pytest_g3.log 2>&1
echo "exit $?" >> gpurun_out/pytest_g3.log
for g in 3 1 3 1; do
  export MO_DOM_GROUPS=$g
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g_c3_$g.json 2> gpurun_out/g_c3_$g.err
  cat gpurun_out/g_c3_$g.json >> gpurun_out/g_c3_all.jsonl
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/g_c2_all.jsonl 2> gpurun_out/g_c2_$g.err
done
