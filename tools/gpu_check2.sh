cd "$(dirname "$0")/.."
bash tools/grid_probe2.sh
timeout 600 python bench.py --steps 20 --warmup 5 --no-pipeline --no-cpu-baseline --no-prefetch > gpurun_out/bench_c3.log 2>&1; python tools/show_bench.py gpurun_out/bench_c3.log 2>/dev/null | head -6
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
python tools/sim_latency.py gpurun_out/sim_latency.json > /dev/null 2>&1; python -c "
import json
for r in json.load(open('gpurun_out/sim_latency.json')):
    print(r['scenario'], r['cell'], r['identical'], r['wall_s'], {op: (v['gpu_dropin'] or {}).get('p50_us') for op, v in r['per_call'].items()})
"
timeout 1200 compute-sanitizer --tool initcheck --print-limit 2000 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_init.log 2>&1
echo "initcheck rc=$? $(grep 'ERROR SUMMARY' gpurun_out/san_init.log)"; grep "Device Frame" gpurun_out/san_init.log | sort | uniq -c | sort -rn | head -8
