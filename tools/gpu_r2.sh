# round-2 GPU check (under gpurun): GPU tests, then the C3 bench line
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
tail -30 gpurun_out/pytest_gpu.log | grep -E "Error|error|assert|FAIL" | head -20
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?"
python tools/show_bench.py gpurun_out/bench_c3.log 2>&1 | head -60
fi
