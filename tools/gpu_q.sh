cd /root/repo
timeout 1200 python -m pytest tests/test_full_size.py -x -q -k "c4_large" 2>&1 | tail -3
