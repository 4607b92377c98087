# end-of-round pass (under gpurun): GPU tests, bench lines, reference arm,
# launch list, ncu captures, sanitizers of the new paths, simulator latency
cd "$(dirname "$0")/.."
O=gpurun_out/r2final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 $O/pytest_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c3.log 2>&1; echo c3 rc=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > $O/bench_c2.log 2>&1; echo c2 rc=$?
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep > $O/bench_c4.log 2>&1; echo c4 rc=$?
timeout 900 python bench.py --sharded --steps 10 --warmup 3 > $O/bench_c4_sharded.log 2>&1; echo c4sh rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > $O/ncu_list.log 2>&1; echo ncu-list rc=$?
python tools/launches.py $O/launches.csv > $O/launches_summary.txt; head -20 $O/launches_summary.txt
for k in score_light select_persistent prefetch_plan; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -o $O/prof_$k \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep > $O/ncu_$k.log 2>&1; echo ncu-$k rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:select_persistent" -s 3 -c 1 -o $O/prof_select_big \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep --no-prefetch --needed-frac 0.5 > $O/ncu_select_big.log 2>&1; echo ncu-select-big rc=$?
for k in score_light select_persistent prefetch_plan select_big; do
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/r02_ncu_${k}_raw.csv 2>/dev/null
  python tools/ncu_lines.py $O/prof_$k.ncu-rep 25 > $O/lines_$k.txt 2>&1
done
for tool in memcheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python -m pytest -q -x -m gpu \
    "tests/test_refine.py::test_large_cuts_equal_oracle[0]" "tests/test_delta.py::test_caller_delta_unordered_with_stale_duplicates[0]" \
    > $O/san_$tool.log 2>&1
  echo "san $tool rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' $O/san_$tool.log | tail -2 | tr '\n' ' ')"
done
python tools/sim_latency.py $O/sim_latency.json > $O/sim_latency.log 2>&1; echo simlat rc=$?
