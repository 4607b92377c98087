# one full ncu capture of a kernel at C3 (under gpurun), plus its source-line stall table
cd "$(dirname "$0")/.."
PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch 2>&1 | grep "pbkv select" | tail -1 | cut -c1-600
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-select_persistent}" -s ${KSKIP:-3} -c 1 -o gpurun_out/prof_${TAG:-x} \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline --no-sweep --no-prefetch ${BENCH_EXTRA} > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
python tools/ncu_lines.py gpurun_out/prof_${TAG:-x}.ncu-rep 45
