"""Stage-4 plan phases at C3 (PBKV_DEBUG_PLAN)."""
import os, sys
os.environ["PBKV_DEBUG_PLAN"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import bench
from paper_2605_06472_b200.api import Policy

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
t, soa, wf, P, locked, K, _ = bench.workload(cfg, 0)
pol = Policy(num_agents=16, k=K, gamma=0.7, device=0)
pol.mirror(t)
pol.put_forecasts(wf, P)
used = int(soa.len[soa.tier == 0][1:].sum())
for bw in (used // 50, used // 50, used // 5, 100, 10**12):
    p = pol.plan_conservative_prefetch(bw)
    print("bw", bw, "cand", len(p.candidate_ids), "sel", len(p.selected_ids), file=sys.stderr, flush=True)
