# consumer-side pre-merge of the row states in every pass (libpm2, ORL_K1_PREMERGE=2) vs actor passes only
# (libcur, default): the logprob pass (old / ref) and the loss pass, cool and power-capped
mkdir -p gpurun_out/pm
VARS="cur pm2" KINDS=logp,loss K1ARGS="--c2 0" REPEAT=8 bash tools/ab_run.sh gpurun_out/pm/ab
