#!/bin/bash
# A/B: lazy refinement (5 coarse levels for all objectives, last 4 only for the ANDed ones) vs full searches
mkdir -p gpurun_out
export MO_DOM_LAZY=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py -q -x > gpurun_out/pytest_lazy.log 2>&1
echo "exit $?" >> gpurun_out/pytest_lazy.log
for v in lazy full lazy full; do
  if [ $v = lazy ]; then export MO_DOM_LAZY=1; else unset MO_DOM_LAZY; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/z_c3_$v.jsonl 2> gpurun_out/z_c3.err
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/z_c2_$v.jsonl 2> gpurun_out/z_c2.err
done
