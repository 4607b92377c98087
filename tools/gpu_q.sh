cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_defer.py tests/test_refine.py -x -q 2>&1 | tail -1
for rep in 1 2; do
for v in base var_so/libpbkv_head.so; do
  if [ "$v" = base ]; then unset PBKV_LIB; else export PBKV_LIB=$PWD/$v; fi
  for f in 0.01 0.1; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep --needed-frac $f > gpurun_out/bv.log 2>&1; echo "$f $v $(python tools/show_bench.py gpurun_out/bv.log 2>/dev/null | head -2 | tr '\n' ' ' | cut -c1-230)"
  done
done
done
