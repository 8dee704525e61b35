mkdir -p gpurun_out
for m in host device; do timeout 600 python scripts/c4_timeline.py $m; done > gpurun_out/c4_timeline.txt 2>&1
timeout 600 python scripts/c4_timeline.py host 1000000 16 >> gpurun_out/c4_timeline.txt 2>&1
