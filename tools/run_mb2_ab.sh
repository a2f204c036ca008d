# 2 CTAs/SM x 8 consumer warps x 16 KB chunks (libmb2) vs 1 CTA/SM x 16 warps x 32 KB (libcur, default),
# corrected A/B tool (the round-1 file r01_k1_sustained_variants.txt is void)
mkdir -p gpurun_out/mb2
VARS="cur mb2" KINDS=logp,loss,lossgrad K1ARGS="--c2 0" REPEAT=8 bash tools/ab_run.sh gpurun_out/mb2/ab
