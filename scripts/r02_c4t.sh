mkdir -p gpurun_out
timeout 600 python scripts/c4_timeline.py host > gpurun_out/c4_timeline.txt 2>&1
