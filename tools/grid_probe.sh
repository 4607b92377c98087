# select grid size sweep (under gpurun)
cd "$(dirname "$0")/.."
for cfg in c2 c3 c4; do for g in 0 16 32 64 148; do
  PBKV_SELECT_GRID=$g timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch > gpurun_out/g.log 2>&1
  echo "$cfg grid=$g $(python tools/show_bench.py gpurun_out/g.log | head -2 | tr '\n' ' ' | cut -c1-260)"
done; done
