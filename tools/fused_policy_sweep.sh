for v in split0 split1 split2 split3 split5; do
  echo "== $v $(ORL_LIB_PATH=build/tune/liborl_$v.so python tools/k1_bench.py --kinds lossgrad --iters 20 | head -1)"
  ORL_LIB_PATH=build/tune/liborl_$v.so ncu --metrics dram__bytes_read.sum -k regex:k1_tma -s 3 -c 1 python tools/k1_bench.py --kinds lossgrad --iters 1 2>&1 | grep -E "dram__"
done
