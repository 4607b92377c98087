cd /root/repo
for i in 1 2; do
timeout 900 python bench.py --no-sweep --no-prefetch --no-pipeline --no-cpu-baseline > gpurun_out/bd.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bd.log').read().strip().splitlines()[-1]); print('run', $i, d['ms_per_step'], d['p50_decision_ms'], d['stage_ms']['total'])"
done
timeout 900 python bench.py > gpurun_out/bd.log 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/bd.log').read().strip().splitlines()[-1]); print('default', d['ms_per_step'], d['p50_decision_ms'], d['stage_ms']['total'])"
