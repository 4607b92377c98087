cd /root/repo
timeout 300 python tools/plan_probe.py c3 2>&1 | grep "pbkv plan" | tail -3
