#!/bin/bash
# NEXT-4: K6 (tcgen05 LM-head GEMM + online LSE) timing vs cuBLAS + K1, and one
# ncu --set full capture of K6 on the llama8b micro-batch (8192 x 4096 x 128256).
OUT=${1:-gpurun_out/ncu_k6}
mkdir -p $OUT
python tools/k6_bench.py > $OUT/k6_bench.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k6_lmhead' -s 1 -c 1 \
    -o $OUT/k6_lmhead python tools/k6_bench.py --no-baseline --reps 1 --warm 1 > $OUT/ncu_k6.log 2>&1
cat $OUT/k6_bench.txt
