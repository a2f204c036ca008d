mkdir -p gpurun_out/ncu4
for k in logp+H loss; do
ORL_LIB_PATH=build/tune/liborl_w16_c32k_s6_b1.so ncu --set full --clock-control none --import-source on -k regex:'k1_tma_kernel' -s 5 -c 1 -o gpurun_out/ncu4/k1_$k python tools/k1_bench.py --kinds $k --iters 1 > gpurun_out/ncu4/ncu_$k.log 2>&1
done
ls gpurun_out/ncu4
