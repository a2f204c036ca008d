#!/bin/bash
# Fused actor pass variants (builds under build_var/lib<name>.so): per variant one ncu launch
# (DRAM bytes, L2 hit rate, time) and a separate-process timing (tools/k1_bench.py, cool GPU),
# at 8 x 1024 rows, V = 128256 bf16.   VARS="base st1 ..." bash tools/ncu_fused_abl.sh OUT
OUT=${1:-gpurun_out/ncu_abl}
mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
KIND=${KIND:-lossgrad}
for v in ${VARS:-base}; do
  ncu --metrics $M --clock-control none -k regex:'k1_tma|k5_tma' -s 3 -c 1 --csv --log-file $OUT/$v.csv \
    python tools/k1_bench.py --libs build_var/lib$v.so --kinds $KIND --iters 2 > $OUT/$v.ncu.log 2>&1
done
for r in 1 2; do
for v in ${VARS:-base}; do
  timeout 300 python tools/k1_bench.py --libs build_var/lib$v.so --kinds $KIND --repeat 3 --iters 20 2>&1 | grep "us/launch" >> $OUT/time.txt
done
done
python - $OUT <<'PY'
import csv, glob, os, sys, re, statistics
out = sys.argv[1]
times = {}
for l in open(os.path.join(out, "time.txt")):
    m = re.match(r"lib(\S+)\.so\s+\S+\s+V=\d+:\s+([\d.]+) us", l)
    if m: times.setdefault(m.group(1), []).append(float(m.group(2)))
for f in sorted(glob.glob(os.path.join(out, "*.csv"))):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    if not rows: continue
    h = rows[0]; d = {r[h.index("Metric Name")]: r[h.index("Metric Value")] for r in rows[1:]}
    v = os.path.basename(f)[:-4]
    print(f"{v:8s} ncu {float(d['gpu__time_duration.sum'])/1e3:7.1f} us  read {float(d['dram__bytes_read.sum'])/1e9:.3f} GB  "
          f"write {float(d['dram__bytes_write.sum'])/1e9:.3f} GB  L2 hit {d['lts__t_sector_hit_rate.pct']} %  "
          f"timed {' '.join('%.1f' % t for t in times.get(v, []))} us")
PY
