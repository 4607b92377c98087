cd /root/repo
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_refine.py tests/test_shard.py -x -q 2>&1 | tail -2
for c in c3 c2 c4; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch --no-sweep > gpurun_out/b.log 2>&1; python tools/show_bench.py gpurun_out/b.log 2>/dev/null | head -2
done
