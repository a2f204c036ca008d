#!/bin/bash
# Round-2 profiling recipe (one B200, under gpurun):
# 1) launch list of the DEFAULT bench command (grpo headline, legs off for time)
# 2) one `--set full` capture of K1 at the grpo launch shape (8 x 4096 rows, V=128256)
# 3) DRAM bytes of every K1 launch of one ragged-length llama8b step (U{64..1024})
OUT=${1:-gpurun_out/ncu_r02}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 1540 -c 1 \
    -o $OUT/k1_grpo python bench.py --steps 1 --warmup 3 --legs "" --no-e2e --no-cpu > $OUT/k1_grpo.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'k1_tma_kernel' --csv --log-file $OUT/k1_varlen.csv \
    python bench.py --config llama8b --lengths secondary --steps 1 --warmup 3 --legs "" --no-e2e --no-cpu \
    > $OUT/k1_varlen.log 2>&1
python bench.py --config llama8b --lengths secondary --steps 1 --warmup 3 --legs "" --no-e2e --no-cpu \
    > $OUT/varlen_bench.json 2>/dev/null
ls -la $OUT
