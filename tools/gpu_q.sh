cd /root/repo
timeout 900 python -m pytest tests/test_shard.py tests/test_full_size.py -x -q -k "shard or interval or dist or c4" 2>&1 | tail -2
grep -E "Error|assert|FAILED|^E " /dev/null
