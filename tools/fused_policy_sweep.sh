for v in default fwd_normal fwd_normal_bwd_normal fwd_last_bwd_unch; do
  echo "== $v"
  ORL_LIB_PATH=build/tune/liborl_$v.so python tools/k1_bench.py --kinds lossgrad --iters 20
  ORL_LIB_PATH=build/tune/liborl_$v.so ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct -k regex:k1_tma -s 3 -c 1 python tools/k1_bench.py --kinds lossgrad --iters 1 2>&1 | grep -E "dram__|lts__"
done
