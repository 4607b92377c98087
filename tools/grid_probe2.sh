cd "$(dirname "$0")/.."
for g in 1 2 4 8 0; do
  PBKV_SELECT_GRID=$g timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-pipeline --no-cpu-baseline --no-prefetch > gpurun_out/g.log 2>&1
  echo "c2 grid=$g $(python tools/show_bench.py gpurun_out/g.log 2>/dev/null | head -2 | tr '\n' ' ' | cut -c1-230)"
  python tools/show_bench.py gpurun_out/g.log 2>/dev/null | grep "sweep 50" | cut -c1-120
done
for g in 1 4; do
  PBKV_SELECT_GRID=$g timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "random_trees" 2>&1 | tail -1
done
