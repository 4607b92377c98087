"""Decision fast path: heavy nodes (thousands of workflows on the shared
prefix) are placed from an interval of their Eq. 2 score instead of waiting
for the exact serial chain.  Victim order, freed tokens and
shortfall must be identical to the exact path and to the CPU oracle, for cuts
that never reach a heavy node (fast path) and for ones that do (exact path)."""
import numpy as np
import pytest

import workloads as WL
from oracle import Oracle
from paper_2605_06472_b200._abi import POLICY_HE, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2])
def test_deferred_decisions_equal_exact(gpu, seed):
    t = HostTree()
    t.synth(n_nodes=30000, n_workflows=512, seed=seed)
    soa = t.export()
    rng = np.random.default_rng(seed)
    K = 4
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, K, 17)
    soa.score[:] = Oracle.score_nodes(soa, wf, P, K, 0.7)
    locked = WL.pinned_paths(soa, rng, 0.01)
    used = int(soa.len[soa.tier == 0][1:].sum())
    fast = Policy(num_agents=16, k=K)
    exact = Policy(num_agents=16, k=K)
    exact.set_defer(False)
    for p in (fast, exact):
        p.mirror(t)
        p.put_forecasts(wf, P)
    for frac in (0.001, 0.01, 0.2, 0.6, 0.999, 1.5):
        needed = max(1, int(frac * used))
        a = fast.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        b = exact.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        o = Oracle.select(soa, POLICY_HE, needed, locked)
        assert (a.victims, a.freed, a.shortfall) == (b.victims, b.freed, b.shortfall), frac
        assert (a.victims, a.freed, a.shortfall) == (o.victims, o.freed, o.shortfall), frac
    f, s = fast.defer_stats()
    assert f >= 3 and s >= 1  # small cuts take the fast path; the take-all cut the exact one
    assert exact.defer_stats() == (0, 0)
