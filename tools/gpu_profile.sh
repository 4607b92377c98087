# one-shot profiling pass (run under gpurun)
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu-list rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score -s 2 -c 4 -o gpurun_out/prof_score \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
ls -la gpurun_out
