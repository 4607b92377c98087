# quick GPU check (under gpurun): GPU tests, select debug line, C3 bench summary
cd "$(dirname "$0")/.."
timeout 1000 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-pipeline --no-cpu-baseline 2>&1 | grep "pbkv select" | tail -1 | grep -o "grid=.*"
timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log
