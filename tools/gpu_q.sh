cd /root/repo
PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch 2>&1 | grep "pbkv select" | tail -1 | grep -o "dbg.*"
