# profiling pass (run under gpurun): GPU tests, launch list, one full capture of $KREGEX
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu-list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-persistent} -s ${KSKIP:-2} -c ${KCOUNT:-1} -o gpurun_out/prof \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
