"""GPU debug: seed-0 random tree, LRU take-all with node 1 locked (run under gpurun)."""
import sys, os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "oracle"]
import numpy as np
import test_gpu_parity as T
import workloads as WL
from oracle import Oracle
from paper_2605_06472_b200._abi import POLICY_LRU
from paper_2605_06472_b200.api import Policy
rng, t, live, P, K, agents = T._instance(0)
gamma = float(rng.uniform(0.1, 0.95))
wf = np.array(live, dtype=np.int64)
soa = t.export()
pol = Policy(num_agents=agents, k=K, gamma=gamma)
soa.score[:] = Oracle.score_nodes(soa, wf, P, K, gamma)
pol.mirror(soa)
for lk in ([], [1]):
    used = int(soa.len[soa.tier == 0].sum())
    for needed in (used, used + 1, 28):
        o = Oracle.select(soa, POLICY_LRU, needed, lk)
        g = pol.select_victims(POLICY_LRU, needed, locked=lk)
        print(lk, needed, used, "ok" if g.victims == o.victims else "DIFF", "\n gpu", g.victims, g.freed, g.shortfall,
              "\n ref", o.victims, o.freed, o.shortfall)
