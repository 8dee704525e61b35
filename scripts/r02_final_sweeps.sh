#!/bin/bash
# Final round-2 sweeps: Appendix D scan (CPU reference beside it), Table I configuration, long runs,
# the C5 grid (standard + large populations)
mkdir -p gpurun_out
timeout 1500 python scripts/appd_scan.py --cpu > gpurun_out/appd_scan.jsonl 2> gpurun_out/appd_scan.err
timeout 900 python scripts/table1.py > gpurun_out/table1.jsonl 2> gpurun_out/table1.err
timeout 900 python scripts/long_run.py c3 400 > gpurun_out/long_c3.jsonl 2>&1
timeout 1800 python scripts/sweep_c5.py --m 3,5,8,10 --n 1000,4000,16000,64000,256000 --gens 10 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 1500 python scripts/sweep_c5.py --problems DTLZ1,DTLZ3,DTLZ4,DTLZ5,DTLZ6 --m 3,5 --n 1000000,4000000 --gens 10 > gpurun_out/sweep_c5_large.jsonl 2> gpurun_out/sweep_c5_large.err
timeout 900 python scripts/sweep_c5.py --problems DTLZ2 --m 8,10 --n 1000000 --gens 5 > gpurun_out/sweep_c5_large_m810.jsonl 2> gpurun_out/sweep_c5_large_m810.err
echo done > gpurun_out/final_sweeps.done
