# profiling pass (run under gpurun): smoke, GPU tests, bench, launch list, full captures
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench_c3.log 2>&1; echo bench rc=$?
python tools/show_bench.py gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_bench.log 2>&1; echo ncu-list rc=$?
python tools/launches.py gpurun_out/launches.csv | head -12
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-select_persistent|score_light}" -s ${KSKIP:-10} -c ${KCOUNT:-2} -o gpurun_out/prof \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
