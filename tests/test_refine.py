"""Large cuts on mid-size trees (select.cu
refine_buckets): buckets of the selected heads beyond one CTA's sort
(> 4096 heads sharing their top key digits -- e.g. every retired head at
score 0, or coarse forecasts tying thousands of scores) are split on the
device round after round.  Victim order, freed and shortfall must equal the
oracle for every policy, with and without locks, including take-all cuts
(need above every evictable token), and no library kernel may run."""
import numpy as np
import pytest

import workloads as WL
from oracle import Oracle
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(6))
def test_large_cuts_equal_oracle(gpu, seed):
    rng = np.random.default_rng(7700 + seed)
    t = HostTree()
    t.synth(n_nodes=int(rng.integers(40_000, 90_000)), n_workflows=int(rng.integers(256, 1024)), agents=8,
            retired_frac=float(rng.choice([0.3, 0.6, 0.9])), seed=int(rng.integers(1 << 30)))
    soa = t.export()
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    K = 4
    P = WL.random_forecasts(rng, wf.size, K, 9, coarse=bool(seed % 2))
    pol = Policy(num_agents=8, k=K, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    s = soa.copy()
    s.score[:] = Oracle.score_nodes(soa, wf, P, K, 0.7)
    used = int(soa.len[soa.tier == 0][1:].sum())
    locked = WL.random_locked(soa, rng, 0.02)
    lib0 = pol.launches()[1]
    for frac in (0.6, 0.97, 3.0):
        needed = max(1, int(frac * used))
        for lk in ([], locked):
            o = Oracle.select(s, POLICY_HE, needed, lk)
            g = pol.select_victims_hierarchical(needed, locked=lk, score_mode=SCORE_RECOMPUTE)
            assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), ("he", frac)
            for pid in (POLICY_LRU, POLICY_LAE):
                o = Oracle.select(s, pid, needed, lk)
                g = pol.select_victims(pid, needed, locked=lk)
                assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), (pid, frac)
    # KVFlow (steps-to-execution keys, policies.hpp kvflow): remaining agent
    # sequences for every live workflow
    remaining = {int(w): [int(a) for a in rng.integers(0, 8, size=int(rng.integers(0, 6)))] for w in wf.tolist()}
    for frac in (0.6, 3.0):
        needed = max(1, int(frac * used))
        o = Oracle.select(s, POLICY_KVFLOW, needed, locked, remaining=remaining)
        g = pol.select_victims(POLICY_KVFLOW, needed, remaining=remaining, locked=locked)
        assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), ("kvflow", frac)
    assert pol.launches()[1] == lib0, "library kernels on the selection path"


@pytest.mark.parametrize("seed", range(3))
def test_sharded_large_cuts_equal_single(gpu, seed):
    """Node-set shards (logical ranks on one GPU, shard.py) at large cuts:
    every shard's local selection refines its own oversized buckets; the
    merged decision equals the single-context one and the oracle."""
    from paper_2605_06472_b200 import shard as S

    rng = np.random.default_rng(7900 + seed)
    t = HostTree()
    t.synth(n_nodes=int(rng.integers(60_000, 120_000)), n_workflows=512, agents=8, seed=int(rng.integers(1 << 30)))
    soa = t.export()
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 4, 9)
    locked = WL.pinned_paths(soa, rng, 0.01)
    sps = []
    for s in S.partition(soa, 4):
        sp = S.ShardedPolicy(s, num_agents=8, k=4, gamma=0.7)
        mine = (wf >= s.wf_lo) & (wf < s.wf_hi)
        sp.pol.put_forecasts(wf[mine], P[mine])
        sps.append(sp)
    single = Policy(num_agents=8, k=4, gamma=0.7)
    single.mirror(t)
    single.put_forecasts(wf, P)
    s2 = soa.copy()
    s2.score[:] = Oracle.score_nodes(soa, wf, P, 4, 0.7)
    used = int(soa.len[soa.tier == 0][1:].sum())
    for frac in (0.5, 0.95):
        needed = max(1, int(frac * used))
        got = S.global_select(sps, POLICY_HE, SCORE_RECOMPUTE, needed, locked)
        want = single.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        assert (got[0].tolist(), got[1], got[2]) == (want.victims, want.freed, want.shortfall), frac
        o = Oracle.select(s2, POLICY_HE, needed, locked)
        assert (o.victims, o.freed, o.shortfall) == (want.victims, want.freed, want.shortfall), frac


@pytest.mark.parametrize("seed", range(2))
def test_device_sort_fallback_equals_oracle(gpu, seed, monkeypatch):
    """The last resort of the full radix path (a refinement round with more
    buckets than a CTA caches: the CUB device sort of S driven from the
    host), forced: same victims as the oracle, take-all included."""
    monkeypatch.setenv("PBKV_SELECT_NO_REFINE", "1")
    rng = np.random.default_rng(7800 + seed)
    t = HostTree()
    t.synth(n_nodes=50_000, n_workflows=512, agents=8, retired_frac=0.6, seed=int(rng.integers(1 << 30)))
    soa = t.export()
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 4, 9)
    pol = Policy(num_agents=8, k=4, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    s = soa.copy()
    s.score[:] = Oracle.score_nodes(soa, wf, P, 4, 0.7)
    used = int(soa.len[soa.tier == 0][1:].sum())
    locked = WL.random_locked(soa, rng, 0.02)
    lib0 = pol.launches()[1]
    for frac in (0.7, 3.0):
        needed = max(1, int(frac * used))
        o = Oracle.select(s, POLICY_HE, needed, locked)
        g = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), frac
    assert pol.launches()[1] > lib0, "the fallback did not run"
