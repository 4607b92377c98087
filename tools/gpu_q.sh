cd /root/repo
PBKV_PROFILE_SHARD=1 timeout 600 python bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bsh.log 2>&1; tail -1 gpurun_out/bsh.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], json.dumps(d.get('stage_host_ms'), indent=0))"
