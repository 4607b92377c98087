cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "async or errors" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_delta.py tests/test_sim_interpose.py -x -q 2>&1 | tail -1
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-prefetch --no-pipeline --no-cpu-baseline > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log 2>/dev/null | head -3
