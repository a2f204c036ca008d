#!/bin/bash
# K6 schedule sweep: timing, then one ncu pass of DRAM bytes per setting.
OUT=${1:-gpurun_out/k6_sched}
mkdir -p $OUT
python tools/k6_sched.py > $OUT/sched.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,gpc__cycles_elapsed.max \
    --clock-control none -k regex:k6_lmhead --csv --log-file $OUT/sched_ncu.csv \
    python tools/k6_sched.py --reps 1 --warm 0 > $OUT/sched_ncu.log 2>&1
cat $OUT/sched.txt
