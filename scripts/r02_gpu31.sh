#!/bin/bash
# association: balanced (row tile pair, reference tile) unit ranges per CTA; parity + C3 bench + kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hmma.py tests/test_gpu_parity.py tests/test_gpu_baseline_sizes.py -q -x > gpurun_out/pytest_assoc.log 2>&1
echo "exit $?" >> gpurun_out/pytest_assoc.log
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> gpurun_out/assoc_c3.jsonl 2> gpurun_out/assoc_c3.err
done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.avg --clock-control none -k regex:"k_assoc_umma|k_dom_rank" --launch-skip 10 -c 6 --csv --log-file gpurun_out/assoc_ncu.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
