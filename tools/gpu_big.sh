# the large-cut selection (under gpurun): parity tests, debug line, 50% bench
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_refine.py tests/test_full_size.py tests/test_delta.py -x -q > gpurun_out/pytest_big.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_big.log)"
grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_big.log | head -10
for f in 0.5 0.9; do
PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch --needed-frac $f > gpurun_out/big.log 2>&1
grep "pbkv select" gpurun_out/big.log | tail -1 | cut -c1-400
python tools/show_bench.py gpurun_out/big.log 2>/dev/null | head -3
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch > gpurun_out/bench_c3.log 2>&1
python tools/show_bench.py gpurun_out/bench_c3.log 2>/dev/null | head -12
