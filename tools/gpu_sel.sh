# selection debug (under gpurun): debug line per need + bench phases
cd "$(dirname "$0")/.."
for f in 0.001 0.01 0.1 0.5; do
  PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch --needed-frac $f 2>&1 | grep "pbkv select" | tail -1 | cut -c1-600
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch ${BENCH_ARGS} > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
python tools/show_bench.py gpurun_out/bench_c3.log
