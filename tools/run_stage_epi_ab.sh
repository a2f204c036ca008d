# 5 TMA stages (libst5) and one epilogue warp (libepi1) vs the default 6 stages / 2 epilogue warps (libcur)
mkdir -p gpurun_out/stepi
VARS="cur st5 epi1" KINDS=logp,loss K1ARGS="--c2 0" REPEAT=8 bash tools/ab_run.sh gpurun_out/stepi/ab
