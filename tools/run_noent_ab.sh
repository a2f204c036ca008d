set -x
mkdir -p gpurun_out/noent
python -m pytest tests -m gpu -q -k "next1 or grad or fused or lossgrad" > gpurun_out/noent/tests.log 2>&1
tail -3 gpurun_out/noent/tests.log
VARS="base noent" KINDS=lossgrad,grad K1ARGS="--c2 0" bash tools/ab_run.sh gpurun_out/noent/ab_c2zero
VARS="base noent" KINDS=lossgrad K1ARGS="--c2 0.01" REPEAT=3 bash tools/ab_run.sh gpurun_out/noent/ab_c2ent
