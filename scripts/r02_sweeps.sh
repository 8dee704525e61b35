#!/bin/bash
# Appendix D objective scan (with the CPU reference beside it) and the C5 grid (round 2)
mkdir -p gpurun_out
timeout 1500 python scripts/appd_scan.py --cpu > gpurun_out/appd_scan.jsonl 2> gpurun_out/appd_scan.err
timeout 1800 python scripts/sweep_c5.py --m 3,5,8,10 --n 1000,4000,16000,64000,256000 --gens 10 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err
timeout 1500 python scripts/sweep_c5.py --problems DTLZ1,DTLZ3,DTLZ4,DTLZ5,DTLZ6 --m 3,5 --n 1000000,4000000 --gens 10 > gpurun_out/sweep_c5_large.jsonl 2> gpurun_out/sweep_c5_large.err
timeout 900 python scripts/sweep_c5.py --problems DTLZ2 --m 8,10 --n 1000000 --gens 5 > gpurun_out/sweep_c5_large_m810.jsonl 2> gpurun_out/sweep_c5_large_m810.err
