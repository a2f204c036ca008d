#!/bin/bash
# Stress tools on the final kernels of round 2's third session (compute-sanitizer is closed on this pool).
OUT=${1:-gpurun_out/stress_r02c}
mkdir -p $OUT
timeout 1200 python tools/bit_identity_stress.py 40 > $OUT/bit_identity.txt 2>&1; echo "bit_identity rc=$?"; tail -2 $OUT/bit_identity.txt
timeout 900 python tools/k5_unaligned_check.py 50 > $OUT/k5_unaligned.txt 2>&1; echo "k5_unaligned rc=$?"; tail -2 $OUT/k5_unaligned.txt
timeout 900 python tools/peer_stress.py 4 30 > $OUT/peer_stress.txt 2>&1; echo "peer rc=$?"; tail -2 $OUT/peer_stress.txt
