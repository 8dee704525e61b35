#!/bin/bash
# A/B: rank-mask sweep with the shortest-first early-exit AND in S-separated tiles vs the plain AND
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py tests/test_gpu_ops.py -q -x > gpurun_out/pytest_ab.log 2>&1
echo "exit $?" >> gpurun_out/pytest_ab.log
for v in new plain new plain; do
  if [ $v = plain ]; then export MO_DOM_PLAIN_AND=1; else unset MO_DOM_PLAIN_AND; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_c3_$v.json 2> gpurun_out/ab_c3_$v.err
  cat gpurun_out/ab_c3_$v.json >> gpurun_out/ab_c3_all.jsonl
  timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline >> gpurun_out/ab_c2_all.jsonl 2> gpurun_out/ab_c2_$v.err
done
unset MO_DOM_PLAIN_AND
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:k_dom_rank --launch-skip 5 -c 3 --csv --log-file gpurun_out/ab_domrank_new.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
export MO_DOM_PLAIN_AND=1
timeout 300 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:k_dom_rank --launch-skip 5 -c 3 --csv --log-file gpurun_out/ab_domrank_plain.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
