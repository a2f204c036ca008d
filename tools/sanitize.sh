#!/bin/bash
# compute-sanitizer over small GPU parity cases (run under gpurun, one B200).
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
SEL='tiny_end_to_end_and_isolated and 0-gae or generic_path or next1_logits_grad_parity and f32-32 or neg_inf or large_microbatch or next1_fused_forward_backward_matches_two_passes'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$SEL" > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/$tool.log | tail -2 | tr '\n' ' ')"
done
# NEXT-4 K6 (tcgen05 / TMEM / 2-SM cluster) on its small cases
SEL6='parity_small or many_tiles or microbatch_offset or run_to_run'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest tests/test_gpu_lmhead.py -m gpu -q -x -p no:cacheprovider -k "$SEL6" > $OUT/k6_$tool.log 2>&1
  echo "k6 $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $OUT/k6_$tool.log | tail -2 | tr '\n' ' ')"
done
