# round-2 profiling pass (under gpurun): bench lines, reference arm, launch list,
# ncu captures of the top kernels, simulator per-call latency
cd "$(dirname "$0")/.."
O=gpurun_out/r2prof; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c3.log 2>&1; echo c3 rc=$?
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-pipeline > $O/bench_c2.log 2>&1; echo c2 rc=$?
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep > $O/bench_c4.log 2>&1; echo c4 rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > $O/ncu_list.log 2>&1; echo ncu-list rc=$?
python tools/launches.py $O/launches.csv > $O/launches_summary.txt; head -20 $O/launches_summary.txt
for k in score_light select_persistent prefetch_plan; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 3 -c 1 -o $O/prof_$k \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep > $O/ncu_$k.log 2>&1; echo ncu-$k rc=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:txt_gemm|head_mma" -s 4 -c 2 -o $O/prof_predict \
  python tools/predict_probe.py > $O/ncu_predict.log 2>&1; echo ncu-predict rc=$?
python tools/sim_latency.py $O/sim_latency.json > $O/sim_latency.log 2>&1; echo simlat rc=$?
