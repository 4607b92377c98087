# quick GPU iteration (under gpurun): select debug line per need, plan phases, GPU tests, bench summary
cd "$(dirname "$0")/.."
for f in 0.001 0.01 0.1 0.5; do
  PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch --needed-frac $f 2>&1 | grep "pbkv select" | tail -1 | cut -c1-400
done
timeout 300 python tools/plan_probe.py c3 2>&1 | grep -v "^bw" | tail -5
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_gpu.log | head -10
timeout 900 python bench.py --steps 20 --warmup 5 --no-pipeline ${BENCH_ARGS} > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
python tools/show_bench.py gpurun_out/bench_c3.log
