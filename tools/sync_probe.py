"""Per-call breakdown of the incremental mirror sync at C3 (PBKV_PROFILE_SYNC)."""
import os, sys, time
os.environ["PBKV_PROFILE_SYNC"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np
import bench
from paper_2605_06472_b200.api import Policy

t, soa, wf, P, locked, K, _ = bench.workload("c3", 0)
pol = Policy(num_agents=16, k=K, gamma=0.7, device=0)
pol.mirror(t)
pol.put_forecasts(wf, P)
pol.sync(t)
rng = np.random.default_rng(1)
live = [int(w) for w in wf.tolist() if w >= int(0.3 * 4096)]
last = np.zeros(0, np.int32)
for it in range(8):
    ops, _ = bench.churn_batch(rng, t, live, last, 4096)
    t.apply_ops(ops.words)
    t0 = time.perf_counter()
    pol.sync(t)
    t1 = time.perf_counter()
    print(f"sync wall {1e3*(t1-t0):.3f} ms", file=sys.stderr, flush=True)
    sel = pol.select_victims_hierarchical(25000, locked=locked)
    last = sel.victim_ids
