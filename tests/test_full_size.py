"""Parity at the benchmark's full size (BASELINE config 3: 1 M-node tree x
4096 workflows x K = 8, 30% retired, 1% of leaves pinned).

The CPU oracle (oracle/pbkv_oracle.c: the reference's greedy frontier itself,
not the closed form) runs at this size in about a second per call, so the
decisions are compared directly, bit for bit, rather than through properties
alone:
  - Eq. 2 for every one of the 1 M nodes (scores bit-identical);
  - HE victim order / freed / shortfall at 0.1%, 1%, 10% and 50% of the
    device tokens (recomputed scores on the GPU, cached scores in the oracle:
    SURVEY.md §0 fact 2), through both the deferred-heavy fast path and the
    exact path;
  - the conservative prefetch plan over the ~40 K host-tier nodes;
plus size-independent properties of the cut: victims distinct, eligible,
freed = sum of their lengths, and minimal (dropping the last victim falls
short of `needed`).
"""
import numpy as np
import pytest

import workloads as WL
from oracle import Oracle
from paper_2605_06472_b200._abi import POLICY_HE, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3(gpu):
    t = HostTree()
    t.synth(n_nodes=1_000_000, n_workflows=4096, agents=16, seed=12345)
    soa = t.export()
    rng = np.random.default_rng(12345)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 8, 17)
    locked = WL.pinned_paths(soa, rng, 0.01)
    pol = Policy(num_agents=16, k=8, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    return t, soa, wf, P, locked, pol


def test_c3_scores_bit_exact(c3):
    t, soa, wf, P, locked, pol = c3
    got = pol.score_all()
    ref = Oracle.score_nodes(soa, wf, P, 8, 0.7)
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))


# 0.5 / 0.9: buckets of S beyond one CTA's sort (the MSD refinement, select.cu
# refine_buckets); 2.0: every head taken (take_all) with a shortfall
@pytest.mark.parametrize("frac", [0.001, 0.01, 0.1, 0.5, 0.9, 2.0])
def test_c3_victims_equal_oracle(c3, frac):
    t, soa, wf, P, locked, pol = c3
    s = soa.copy()
    s.score[:] = Oracle.score_nodes(soa, wf, P, 8, 0.7)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = max(1, int(frac * used))
    o = Oracle.select(s, POLICY_HE, needed, locked)
    lib0 = pol.launches()[1]
    g = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    assert pol.launches()[1] == lib0, "library kernels on the selection path"
    assert (g.freed, g.shortfall) == (o.freed, o.shortfall)
    assert g.victims == o.victims
    # properties of the cut
    v = np.array(g.victims, dtype=np.int64)
    assert np.unique(v).size == v.size
    assert np.all(soa.tier[v] == 0) and np.all(v != 0)
    assert int(soa.len[v].sum()) == g.freed
    if not g.shortfall:
        assert g.freed >= needed and int(soa.len[v[:-1]].sum()) < needed


@pytest.mark.parametrize("frac", [0.5, 2.0])
def test_c3_lru_large_cuts_equal_oracle(c3, frac):
    from paper_2605_06472_b200._abi import POLICY_LRU

    t, soa, wf, P, locked, pol = c3
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = max(1, int(frac * used))
    o = Oracle.select(soa, POLICY_LRU, needed, locked)
    g = pol.select_victims(POLICY_LRU, needed, locked=locked)
    assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall)


def test_c3_exact_path_equals_fast_path(c3):
    t, soa, wf, P, locked, pol = c3
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = max(1, used // 100)
    fast = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    pol.set_defer(False)
    try:
        exact = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    finally:
        pol.set_defer(True)
    assert (fast.victims, fast.freed, fast.shortfall) == (exact.victims, exact.freed, exact.shortfall)


def test_c3_prefetch_plan_equals_oracle(c3):
    t, soa, wf, P, locked, pol = c3
    g = pol.plan_conservative_prefetch(4096)
    o = Oracle.plan(soa, wf, P, 4096)
    assert len(g.candidates) == len(o.candidates) > 1000
    assert [c[0] for c in g.candidates] == [c[0] for c in o.candidates]
    assert np.array_equal(np.array([c[1] for c in g.candidates]).view(np.uint64),
                          np.array([c[1] for c in o.candidates]).view(np.uint64))
    assert g.selected == o.selected and g.selected_tokens == o.selected_tokens


def test_c4_sharded_8_ways_equals_single_and_oracle(gpu):
    """BASELINE config 4 shape (8 M nodes x 16 K workflows x K = 8), split
    into 8 node-set shards (logical ranks on one B200): the sharded decision
    (local cuts, spine records, merge + cut) equals the single-context
    decision on the whole tree and the CPU oracle."""
    from paper_2605_06472_b200 import shard as S

    t = HostTree()
    t.synth(n_nodes=8_000_000, n_workflows=16384, agents=16, seed=4)
    soa = t.export()
    rng = np.random.default_rng(4)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 8, 17)
    locked = WL.pinned_paths(soa, rng, 0.01)
    shards = S.partition(soa, 8)
    sps = []
    for s in shards:
        sp = S.ShardedPolicy(s, num_agents=16, k=8, gamma=0.7)
        mine = (wf >= s.wf_lo) & (wf < s.wf_hi)
        sp.pol.put_forecasts(wf[mine], P[mine])
        sps.append(sp)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = used // 100
    got = S.global_select(sps, POLICY_HE, SCORE_RECOMPUTE, needed, locked)
    del sps
    single = Policy(num_agents=16, k=8, gamma=0.7)
    single.mirror(t)
    single.put_forecasts(wf, P)
    want = single.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    assert (got[0].tolist(), got[1], got[2]) == (want.victims, want.freed, want.shortfall)
    s2 = soa.copy()
    s2.score[:] = Oracle.score_nodes(soa, wf, P, 8, 0.7)
    o = Oracle.select(s2, POLICY_HE, needed, locked)
    assert (o.victims, o.freed, o.shortfall) == (want.victims, want.freed, want.shortfall)


def test_c4_large_cut_equals_oracle(gpu):
    """BASELINE config 4 on one context at 90% of the device tokens: the
    refinement's rounds exceed one window of bucket descriptors (select.cu
    refine_buckets), no library kernel runs, and the victims equal the
    oracle's."""
    t = HostTree()
    t.synth(n_nodes=8_000_000, n_workflows=16384, agents=16, seed=4)
    soa = t.export()
    rng = np.random.default_rng(4)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 8, 17)
    locked = WL.pinned_paths(soa, rng, 0.01)
    pol = Policy(num_agents=16, k=8, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = int(0.9 * used)
    lib0 = pol.launches()[1]
    g = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    assert pol.launches()[1] == lib0, "library kernels on the selection path"
    s2 = soa.copy()
    s2.score[:] = Oracle.score_nodes(soa, wf, P, 8, 0.7)
    o = Oracle.select(s2, POLICY_HE, needed, locked)
    assert (g.freed, g.shortfall) == (o.freed, o.shortfall)
    assert np.array_equal(g.victim_ids, np.asarray(o.victims, dtype=np.int32))
