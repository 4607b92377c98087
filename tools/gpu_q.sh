cd /root/repo
for c in c3 c4; do
for v in base var_so/libpbkv_s2_w4.so var_so/libpbkv_s6_w4.so var_so/libpbkv_s4_w8.so var_so/libpbkv_s4_w2.so; do
  if [ "$v" = base ]; then unset PBKV_LIB; else export PBKV_LIB=$PWD/$v; fi
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep > gpurun_out/bv.log 2>&1; echo "$c $v $(python tools/show_bench.py gpurun_out/bv.log 2>/dev/null | sed -n 2p)"
done
done
