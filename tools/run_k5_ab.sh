# K5 straight-line full chunks + per-thread stage release (libk5s) vs the previous K5 (libnoent)
mkdir -p gpurun_out/k5s
python -m pytest tests -m gpu -q -k "next1 or grad or fused or lossgrad or unaligned" > gpurun_out/k5s/tests.log 2>&1
tail -3 gpurun_out/k5s/tests.log
VARS="noent k5s" KINDS=grad K1ARGS="--c2 0" bash tools/ab_run.sh gpurun_out/k5s/ab_c2zero
VARS="noent k5s" KINDS=grad K1ARGS="--c2 0.01" bash tools/ab_run.sh gpurun_out/k5s/ab_c2ent
python tools/k1_bench.py --libs build_var/libk5s.so --V 50257 --kinds grad --repeat 3 --iters 20 > gpurun_out/k5s/v50257_k5s.txt 2>&1
python tools/k1_bench.py --libs build_var/libnoent.so --V 50257 --kinds grad --repeat 3 --iters 20 > gpurun_out/k5s/v50257_noent.txt 2>&1
