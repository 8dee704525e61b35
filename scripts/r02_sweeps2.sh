#!/bin/bash
# Round-2 sweeps (final kernels): Appendix D objective scan with the CPU reference, C5 grid N <= 256k, the
# table-I configuration, and the final C3 measurement set with launch list + ncu of the association
mkdir -p gpurun_out
timeout 1500 python scripts/appd_scan.py --cpu > gpurun_out/appd_scan.jsonl 2> gpurun_out/appd_scan.err
timeout 2400 python scripts/sweep_c5.py --m 3,5,8,10 --n 1000,4000,16000,64000,256000 --gens 10 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 600 python scripts/table1.py > gpurun_out/table1.jsonl 2> gpurun_out/table1.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 200 -c 60 --csv \
    --log-file gpurun_out/launches_c3_late.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_bench_late.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assoc_umma --launch-skip 20 -c 1 \
    -o gpurun_out/c3_umma python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_umma.log 2>&1
