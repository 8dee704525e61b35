#!/bin/bash
# A/B of the current tree against _ab_old (a worktree of an earlier commit, built in place)
mkdir -p gpurun_out
for t in new old; do
  d=.; [ $t = old ] && d=_ab_old
  (cd $d && timeout 300 python scripts/trace_cfg.py DTLZ4 5 14 64000 15) > gpurun_out/ab_dtlz4_$t.txt 2>&1
  (cd $d && timeout 300 python scripts/sweep_c5.py --problems DTLZ2,DTLZ4 --m 5 --n 1000,64000 --gens 10) > gpurun_out/ab_sweep_$t.jsonl 2>&1
done
