#!/bin/bash
# After the clock-sampler change: bench JSON tests, the default bench, the reference arm, and the N = 2
# code path (two ranks sharing the GPU, gloo + peer collectives; functional, not a measurement).
OUT=${1:-gpurun_out/check_r02c}
mkdir -p $OUT
python -m pytest tests -m gpu -q -k bench > $OUT/gputest_bench.log 2>&1
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/reference.json 2> $OUT/reference.err
ORL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --config rpp8 --batch 32 --lengths secondary --steps 3 \
    --warmup 3 --legs "" --no-cpu > $OUT/shared_n2.json 2> $OUT/shared_n2.err
ls -la $OUT
