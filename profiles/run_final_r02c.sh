#!/bin/bash
# Final state of round 2 (third session): GPU tests, smoke, the default bench, the ncu launch list of
# the default bench command, and ncu --set full of the fused actor pass / K5 at c2 = 0 (the BASELINE
# configs' setting: the no-entropy-term instantiations).
OUT=${1:-gpurun_out/final_r02c}
mkdir -p $OUT
python -m pytest tests -m gpu -q > $OUT/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_tma -s 3 -c 1 -o $OUT/fused_c2zero \
    python tools/k1_bench.py --kinds lossgrad --iters 2 --c2 0 > $OUT/fused_c2zero.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k5_tma -s 3 -c 1 -o $OUT/k5_c2zero \
    python tools/k1_bench.py --kinds grad --iters 2 --c2 0 > $OUT/k5_c2zero.log 2>&1
ls -la $OUT
