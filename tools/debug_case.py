import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
import known_answers as KA
from test_gpu_parity import run_gpu
for c in KA.cases():
    if c.error:
        continue
    try:
        r = run_gpu(c)
        KA.check(c, r)
        print("ok  ", c.name)
    except AssertionError as e:
        print("FAIL", c.name, e)
