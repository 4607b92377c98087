cd /root/repo
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py tests/test_defer.py tests/test_refine.py tests/test_shard.py -x -q 2>&1 | tail -2
for f in 0.01 0.05 0.1; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch --needed-frac $f > gpurun_out/bf.log 2>&1
echo "$f $(python tools/show_bench.py gpurun_out/bf.log 2>/dev/null | head -2 | tr '\n' ' ' | cut -c1-250)"
done
