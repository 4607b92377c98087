cd /root/repo
timeout 300 python tools/neg_wait_probe.py 2>&1 | tail -2
