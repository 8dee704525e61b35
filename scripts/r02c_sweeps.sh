#!/bin/bash
# Final kernels: the paper's Table I configuration and the Appendix D objective scan (GPU side only)
mkdir -p gpurun_out
timeout 900 python scripts/table1.py > gpurun_out/table1_r02c.jsonl 2> gpurun_out/table1_r02c.err
timeout 900 python scripts/appd_scan.py > gpurun_out/appd_scan_r02c.jsonl 2> gpurun_out/appd_scan_r02c.err
