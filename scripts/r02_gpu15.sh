#!/bin/bash
mkdir -p gpurun_out
for mode in default pairwise notsum; do
  case $mode in
    pairwise) export MO_DOM_PAIRWISE=1; unset MO_NO_TSUM;;
    notsum) unset MO_DOM_PAIRWISE; export MO_NO_TSUM=1;;
    *) unset MO_DOM_PAIRWISE; unset MO_NO_TSUM;;
  esac
  echo "== $mode" >> gpurun_out/m3_modes.log
  timeout 600 python scripts/sweep_c5.py --problems DTLZ2,DTLZ3,DTLZ7 --m 3,4,5 --n 16000,64000 --gens 10 >> gpurun_out/m3_modes.log 2>&1
done
