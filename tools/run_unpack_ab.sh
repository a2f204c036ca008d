# bf16 -> f32 unpack by two PRMTs (ALU pipe; libprmt, ORL_K1_PRMT_UNPACK) vs SHL + LOP3 (libcur, default),
# re-run with the corrected A/B tool (the round-2 first-session file r02_k1_unpack_ab.txt is void)
mkdir -p gpurun_out/unpack
VARS="cur prmt" KINDS=logp,loss,lossgrad K1ARGS="--c2 0" REPEAT=8 bash tools/ab_run.sh gpurun_out/unpack/ab
