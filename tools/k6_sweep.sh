#!/bin/bash
# NEXT-4 K6 schedule sweep (one B200): tiles-per-split and 1-SM vs 2-SM, fused path only.
OUT=${1:-gpurun_out/k6_sweep}
mkdir -p $OUT
for tps in 1 2 4 8 16; do
  for two in 1 0; do
    echo "tps=$tps 2sm=$two $(ORL_K6_TPS=$tps ORL_K6_2SM=$two python tools/k6_bench.py --no-baseline --reps 30)"
  done
done > $OUT/sweep.txt 2>&1
cat $OUT/sweep.txt
