cd /root/repo
timeout 1200 python -m pytest tests/test_delta.py tests/test_sim_interpose.py tests/test_gpu_parity.py tests/test_shard.py -x -q 2>&1 | tail -2
timeout 600 python tools/sync_probe.py 2>&1 | tail -9
timeout 300 python bench.py --steps 20 --warmup 5 --no-sweep --no-prefetch --no-pipeline --no-cpu-baseline > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log 2>/dev/null | head -3
