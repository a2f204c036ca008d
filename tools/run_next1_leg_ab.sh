# NEXT-1 leg of bench.py (llama8b actor logits, c2 = 0) with the previous build (libbase: before the
# c2 = 0 specialisation and the K5 straight-line body) and the current one (libcur), alternated.
mkdir -p gpurun_out/n1ab
for r in 1 2 3; do for v in base cur; do
  ORL_LIB_PATH=build_var/lib$v.so python bench.py --config llama8b --legs llama8b --steps 3 --warmup 3 --no-e2e --no-cpu \
      --graph 0 --next4 0 --leg-steps 24 > gpurun_out/n1ab/$v.$r.json 2> gpurun_out/n1ab/$v.$r.err

done; done
