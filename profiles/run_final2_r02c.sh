#!/bin/bash
# Final state of round 2 (third session, after the bench clock-sampler change): GPU tests, smoke, the
# default bench and the ncu launch list of the default bench command.
OUT=${1:-gpurun_out/final2_r02c}
mkdir -p $OUT
python -m pytest tests -m gpu -q > $OUT/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
ls -la $OUT
