"""GPU probe: exact-chain kernel time vs number of binade passes (run under gpurun)."""
import math
import os
import sys
import time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
import torch
from paper_2605_06472_b200 import shard as SH
from paper_2605_06472_b200.api import Policy


def passes(x):
    t, n, p = 0.0, 0, 0
    e_prev = None
    for v in x.tolist():
        t2 = t + v
        if t == 0.0:
            p += 1
        else:
            e = math.frexp(t)[1]
            if e != e_prev:
                p += 1
                e_prev = e
        t = t2
    return p


class H:
    pass


h = H()
h.pol = Policy(num_agents=4, k=3)
rng = np.random.default_rng(0)
for name, x in [("u1e-3", rng.random(23000) * 1e-3), ("half", 0.3 + 0.4 * rng.random(23000)),
                ("92k", 0.3 + 0.4 * rng.random(92000))]:
    xt = torch.from_numpy(x).cuda()
    off = np.array([0, x.size])
    for _ in range(3):
        SH.ShardedPolicy.chain_sums(h, xt, off)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        SH.ShardedPolicy.chain_sums(h, xt, off)
    dt = (time.perf_counter() - t0) / 20
    print(f"{name}: L={x.size} approx binade passes={passes(x)} wall per call={dt * 1e6:.1f} us")
