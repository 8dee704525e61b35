#!/bin/bash
# A/B: address-carrying Eytzinger search (one ALU op per probe), ordered vs plain AND; parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py tests/test_gpu_stream.py -q -x > gpurun_out/pytest_srch.log 2>&1
echo "exit $?" >> gpurun_out/pytest_srch.log
for v in new plain new plain; do
  if [ $v = plain ]; then export MO_DOM_PLAIN_AND=1; else unset MO_DOM_PLAIN_AND; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s_c3_$v.json 2> gpurun_out/s_c3_$v.err
  cat gpurun_out/s_c3_$v.json >> gpurun_out/s_c3_all.jsonl
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/s_c2_all.jsonl 2> gpurun_out/s_c2_$v.err
done
