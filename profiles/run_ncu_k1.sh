#!/bin/bash
# K1/K5 microbenchmark + one ncu --set full capture per kernel variant (one B200, under gpurun).
OUT=${1:-gpurun_out/ncu}
mkdir -p $OUT
python tools/k1_bench.py --kinds logp,logp+H,loss,lossgrad,grad,sum,copy > $OUT/k1_bench.txt 2>&1
for k in logp logp+H loss lossgrad; do
  ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 2 -c 1 \
      -o $OUT/k1_$k python tools/k1_bench.py --kinds $k --iters 1 > $OUT/ncu_$k.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:'k5_tma_kernel' -s 2 -c 1 \
    -o $OUT/k5_grad python tools/k1_bench.py --kinds grad --iters 1 > $OUT/ncu_grad.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k1_|k3_|k5_|whiten_|stats_|lengths_' \
    --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next1 > $OUT/launches_bench.log 2>&1
cat $OUT/k1_bench.txt
