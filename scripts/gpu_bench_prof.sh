#!/bin/bash
mkdir -p gpurun_out
W=${WL:-c2}
timeout 600 python bench.py --steps 500 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_dom_tile_sorted|k_assoc<}" -s ${SKIP:-30} -c ${COUNT:-2} \
    -o gpurun_out/prof_${W} -f python scripts/profile_step.py $W 12 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
