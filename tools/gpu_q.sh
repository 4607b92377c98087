cd /root/repo
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
PBKV_DEBUG_TIMING=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-sweep --no-prefetch --no-pipeline --no-cpu-baseline 2>&1 | grep "pbkv timing" | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log 2>/dev/null | head -8
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep > gpurun_out/b2.log 2>&1; python tools/show_bench.py gpurun_out/b2.log 2>/dev/null | head -1
