cd /root/repo
for rep in 1 2; do
for v in base var_so/libpbkv_ns64.so var_so/libpbkv_ns128.so var_so/libpbkv_ns512.so; do
  if [ "$v" = base ]; then unset PBKV_LIB; else export PBKV_LIB=$PWD/$v; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep > gpurun_out/bv.log 2>&1; echo "$v $(python tools/show_bench.py gpurun_out/bv.log 2>/dev/null | head -1 | cut -c1-200)"
done
done
