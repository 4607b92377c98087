cd /root/repo
O=gpurun_out/r2final; mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c3.log 2>&1; echo c3 rc=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > $O/bench_c2.log 2>&1; echo c2 rc=$?
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep > $O/bench_c4.log 2>&1; echo c4 rc=$?
timeout 900 python bench.py --sharded --steps 10 --warmup 3 > $O/bench_c4_sharded.log 2>&1; echo c4sh rc=$?
