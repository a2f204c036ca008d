#!/bin/bash
# K1 microbenchmark + one ncu --set full capture per K1 variant (one B200, under gpurun).
OUT=${1:-gpurun_out/ncu}
mkdir -p $OUT
python tools/k1_bench.py > $OUT/k1_bench.txt 2>&1
for k in logp logp+H loss; do
  ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 2 -c 1 \
      -o $OUT/k1_$k python tools/k1_bench.py --kinds $k --iters 1 > $OUT/ncu_$k.log 2>&1
done
cat $OUT/k1_bench.txt
