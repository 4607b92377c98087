"""Timing of Policy.prefetch_round at C3: the C call alone vs the Python wrapper."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np

import bench
from paper_2605_06472_b200 import _abi
from paper_2605_06472_b200._abi import ptr
from paper_2605_06472_b200.api import Policy

t, soa, wf, P, locked, K, _ = bench.workload("c3", 0)
pol = Policy(num_agents=16, k=K, gamma=0.7, device=0)
pol.mirror(t)
pol.put_forecasts(wf, P)
used = int(soa.len[soa.tier == 0][1:].sum())
plan = pol.plan_conservative_prefetch(max(1, used // 50))
sel = np.ascontiguousarray(plan.selected_ids, dtype=np.int32)
n = sel.size
prom = np.zeros(n, np.int32)
vend = np.zeros(n, np.int64)
vict = np.zeros(soa.n_nodes, np.int32)
nv = C.c_int64()
for rep in range(8):
    t0 = time.perf_counter()
    rc = _abi.lib().pbkv_prefetch_round(pol._h, ptr(sel, C.c_int32), n, 0, ptr(prom, C.c_int32), ptr(vend, C.c_int64),
                                        ptr(vict, C.c_int32), vict.size, C.byref(nv))
    t1 = time.perf_counter()
    pr, vs = pol.prefetch_round(sel, 0)
    t2 = time.perf_counter()
    print(f"rc={rc} C call {1e3*(t1-t0):.3f} ms  wrapper {1e3*(t2-t1):.3f} ms  promoted {int(prom.sum())} victims {nv.value}",
          flush=True)
