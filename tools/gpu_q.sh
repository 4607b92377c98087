cd /root/repo
timeout 900 python -m pytest tests/test_refine.py -x -q 2>&1 | tail -3
