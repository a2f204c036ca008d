#!/bin/bash
# Round-2 third session: ncu --set full of K1 at the grpo launch shape (8 x 4096 rows, V = 128256) on the
# final code -- the logprob pass (K1 launch 1540 of the default bench command) and the actor loss pass
# (launch 2100) -- for the roofline's traffic figure.
OUT=${1:-gpurun_out/ncu_r02c}
mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 1540 -c 1 \
    -o $OUT/k1_grpo_logp python bench.py --steps 1 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/k1_grpo_logp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 2100 -c 1 \
    -o $OUT/k1_grpo_loss python bench.py --steps 1 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/k1_grpo_loss.log 2>&1
ls -la $OUT
