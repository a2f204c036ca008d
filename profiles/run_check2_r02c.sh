#!/bin/bash
# Clock sampler with nvidia-smi timestamps: a short default-shaped run, the N = 2 shared-GPU functional
# run; the one-process-per-device test exercised with one rank (ORL_TEST_WORLD=1).
OUT=${1:-gpurun_out/check2_r02c}
mkdir -p $OUT
nvidia-smi --query-gpu=timestamp,clocks.sm --format=csv,noheader,nounits > $OUT/smi_format.txt 2>&1
ORL_TEST_WORLD=1 python -m pytest tests/test_gpu_multidevice.py -q > $OUT/multidevice_w1.log 2>&1
python -m pytest tests -m gpu -q -k bench > $OUT/gputest_bench.log 2>&1
python bench.py --config llama8b --steps 3 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/short.json 2> $OUT/short.err
ORL_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --config rpp8 --batch 32 --lengths secondary --steps 3 \
    --warmup 3 --legs "" --no-cpu > $OUT/shared_n2.json 2> $OUT/shared_n2.err
ls -la $OUT
