#!/bin/bash
# Round-2 (second session) profiling: ncu --set full of the fused actor pass and of the K1
# logprob pass at 8 x 1024 rows, V = 128256 bf16 (tools/k1_bench.py, one launch each), the
# smaller vocabularies (cool and after a 15 s warm-up), and bench.py's N = 2 code path on one GPU.
OUT=${1:-gpurun_out/ncu_r02b}
mkdir -p $OUT
ncu --set full --import-source on --clock-control none -k regex:k1_tma -s 3 -c 1 -o $OUT/fused \
    python tools/k1_bench.py --kinds lossgrad --iters 2 > $OUT/fused.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_tma -s 3 -c 1 -o $OUT/logp \
    python tools/k1_bench.py --kinds logp --iters 2 > $OUT/logp.log 2>&1
for V in 32000 50257 152064; do
  python tools/k1_bench.py --V $V --kinds logp,loss,lossgrad --repeat 3 --iters 20 > $OUT/v$V.cool.txt 2>&1
  python tools/k1_bench.py --V $V --kinds logp,loss,lossgrad --repeat 3 --iters 20 --warm-seconds 15 > $OUT/v$V.hot.txt 2>&1
done
ORL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --legs "" --no-cpu > $OUT/shared_n2.json 2> $OUT/shared_n2.err
ls -la $OUT
