cd /root/repo
for v in base var_so/libpbkv_noalloc.so var_so/libpbkv_cg.so var_so/libpbkv_evl.so; do
  if [ "$v" = base ]; then unset PBKV_LIB; else export PBKV_LIB=$PWD/$v; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep > gpurun_out/bv.log 2>&1; echo "$v"; python tools/show_bench.py gpurun_out/bv.log 2>/dev/null | head -1
done
