cd /root/repo
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^(FAILED|ERROR)|Error" gpurun_out/pytest_gpu.log | head
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log 2>/dev/null | head -9
