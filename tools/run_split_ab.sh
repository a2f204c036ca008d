# fused actor pass split k (backward of row i-1 after k forward chunks of row i) at c2 = 0: k = 3 (libcur,
# default), 2 (libs2), 4 (libs4); separate-process cool runs, then rotated interleaving after a warm-up
mkdir -p gpurun_out/split
VARS="cur s2 s4" KINDS=lossgrad K1ARGS="--c2 0" REPEAT=8 bash tools/ab_run.sh gpurun_out/split/ab
