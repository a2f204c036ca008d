#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200).
# 1) launch list of our kernels inside the bench command (cold-cache, serialised)
# 2) one `--set full` capture of each K1 variant (logprob mode, loss mode)
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k1_|k3_|whiten_|stats_' \
    --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 20 -c 2 \
    -o $OUT/k1_full python bench.py --batch 16 --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/k1_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 4 -c 1 \
    -o $OUT/k1_loss python bench.py --batch 16 --steps 1 --warmup 3 --no-e2e --no-cpu > $OUT/k1_loss.log 2>&1
ls -la $OUT
