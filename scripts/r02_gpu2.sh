#!/bin/bash
# gpurun: full GPU suite (no -x), then C3 and C2 bench lines.  Env: TESTS="..." to restrict.
mkdir -p gpurun_out
timeout 2700 python -m pytest ${TESTS:-tests} -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ "${SKIP_BENCH}" != "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
  timeout 600 python bench.py --steps 50 --warmup 5 --workload c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
fi
