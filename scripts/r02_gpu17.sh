#!/bin/bash
# final check of the current build: GPU suite, C3/C2/C1 bench lines, islands under torchrun (gloo, 2
# processes on the one GPU), PCIe copy bandwidth, and the m=3 sweep cells
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --steps 100 --warmup 5 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 500 --warmup 5 --workload c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
MO_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 10 --warmup 3 --workload c2 --no-cpu-baseline > gpurun_out/bench_c2_islands2.json 2> gpurun_out/bench_c2_islands2.err
python - > gpurun_out/pcie.txt 2>&1 <<'PY'
import torch
for mb in (12, 116):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory(); d = torch.empty_like(h, device="cuda")
    for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); [f() for _ in range(10)]; e1.record(); e1.synchronize()
        print(name, mb, "MB", round(10 * mb / 1024 / (e0.elapsed_time(e1) / 1e3), 2), "GB/s")
PY
timeout 900 python scripts/sweep_c5.py --m 3 --n 1000,4000,16000,64000 --gens 10 > gpurun_out/sweep_c5_m3.jsonl 2> gpurun_out/sweep_c5_m3.err
