cd /root/repo
for f in 0.1 0.2 0.3; do
for v in base var_so/libpbkv_sm19.so var_so/libpbkv_sm20.so; do
  if [ "$v" = base ]; then unset PBKV_LIB; else export PBKV_LIB=$PWD/$v; fi
  PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep --needed-frac $f > gpurun_out/bv.log 2>&1; echo "$f $v $(grep 'pbkv select' gpurun_out/bv.log | tail -1 | grep -o 'path=[0-9]*') $(python tools/show_bench.py gpurun_out/bv.log 2>/dev/null | head -1 | cut -c1-120)"
done
done
