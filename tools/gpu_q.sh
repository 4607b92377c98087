cd /root/repo
for c in c3 c2 c4; do
PBKV_DEBUG_SELECT=1 timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-pipeline --no-cpu-baseline --no-sweep --no-prefetch 2>&1 | grep "pbkv select" | tail -1 | grep -o "dbg.*"; true
done
