#!/bin/bash
# Clock sampler on short timed regions (the sample after the region's start is waited for).
OUT=${1:-gpurun_out/check3_r02c}
mkdir -p $OUT
python bench.py --config llama8b --steps 3 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/short.json 2> $OUT/short.err
ORL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --config rpp8 --batch 32 --lengths secondary --steps 3 \
    --warmup 3 --legs "" --no-cpu > $OUT/shared_n2.json 2> $OUT/shared_n2.err
python bench.py --config llama8b --steps 20 --warmup 10 --legs "" --no-e2e --no-cpu > $OUT/llama8b.json 2> $OUT/llama8b.err
ls -la $OUT
