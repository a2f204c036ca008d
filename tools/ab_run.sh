#!/bin/bash
# A/B of liborl builds (build_var/lib<name>.so): separate-process cool timings, then one
# interleaved run after a warm-up (power-capped state).  VARS="a b" KINDS=lossgrad bash tools/ab_run.sh OUT
OUT=${1:-gpurun_out/ab}
mkdir -p $(dirname $OUT)
KINDS=${KINDS:-lossgrad}
: > $OUT.cool.txt
for r in 1 2; do for v in $VARS; do
  timeout 300 python tools/k1_bench.py --libs build_var/lib$v.so --kinds $KINDS ${K1ARGS:-} --repeat 3 --iters 20 2>&1 | grep "us/launch" >> $OUT.cool.txt
done; done
L=$(for v in $VARS; do printf "build_var/lib%s.so," $v; done | sed 's/,$//')
python tools/k1_bench.py --libs $L --kinds $KINDS ${K1ARGS:-} --repeat ${REPEAT:-6} --iters 20 --warm-seconds ${WARM:-20} > $OUT.hot.txt 2>&1
cat $OUT.cool.txt $OUT.hot.txt
