"""The fused prefetch round (pbkv_prefetch_round) against the
reference's own per-candidate loop (simulator.hpp:632-681) replayed on the
reference CacheTree (oracle/_ref): for every selected candidate in plan
order, select_victims_hierarchical(need) under the ancestry locks of the
remaining candidates plus pinned paths, the retired prefix of that order as
victims (conservative round), skip when short, else demote them and promote
the candidate.  Promotion flags and victim lists must be identical."""
import numpy as np
import pytest

import workloads as WL
from oracle import RefTree, have_ref
from paper_2605_06472_b200._abi import POLICY_HE
from paper_2605_06472_b200.api import HostTree, Policy
from paper_2605_06472_b200.ops import OpStream

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="reference library not built")]

BIG = 1 << 40


def ancestors(parent, v):
    out = []
    v = int(parent[v])
    while v > 0:
        out.append(v)
        v = int(parent[v])
    return out


def reference_round(ops_words, dev_cap, wf, P, selected, pinned):
    """simulator.hpp:640-681 (conservative mode) on the reference tree."""
    t = RefTree(dev_cap, BIG)
    t.apply_ops(ops_words)
    promoted, victims = [], []
    for i, cid in enumerate(selected):
        soa = t.export()
        par = soa.parent
        vic = []
        ok = int(soa.tier[cid]) == 1 and int(soa.tier[par[cid]]) == 0
        if ok:
            free = soa.scalars["device_capacity"] - soa.scalars["device_used"]
            need = int(soa.len[cid]) - free
            if need > 0:
                locked = set(pinned)
                for s in selected[i:]:
                    locked.add(int(par[s]))
                    locked.update(ancestors(par, s))
                sel = t.select(POLICY_HE, need, sorted(locked))
                freed = 0
                for v in sel.victims:
                    if not soa.retired[v]:
                        break
                    vic.append(v)
                    freed += int(soa.len[v])
                    if freed >= need:
                        break
                if freed < need:
                    ok, vic = False, []
                else:
                    o = OpStream()
                    for v in vic:
                        o.demote(v)
                    t.apply_ops(o.words)
            if ok:
                t.apply_ops(OpStream().promote(cid).words)
        promoted.append(1 if ok else 0)
        victims.append(vic if ok else [])
    return promoted, victims


def _active_pinned(soa, rng, k):
    """ancestors + leaf of k random device leaves carrying access (decoding paths)"""
    n = soa.n_nodes
    ent = soa.acc_off[1:] - soa.acc_off[:-1]
    dev = soa.tier == 0
    cand = [i for i in range(1, n) if dev[i] and ent[i] > 0]
    if not cand:
        return []
    out = set()
    for v in rng.choice(cand, size=min(k, len(cand)), replace=False):
        out.add(int(v))
        out.update(ancestors(soa.parent, int(v)))
    return sorted(out)


def _case(seed, n_ops=(20, 90), n_wf=(3, 10)):
    """A random tree whose device is nearly full: capacity = the peak use of the
    random op stream (+ slack), then the space freed by its demotions is
    refilled by a filler workflow that terminates (retired victims)."""
    rng = np.random.default_rng(1000 + seed)
    nw = int(rng.integers(*n_wf))
    agents = int(rng.integers(2, 6))
    ops, live = WL.random_tree_ops(rng, n_ops=int(rng.integers(*n_ops)), n_wf=nw, agents=agents, alphabet=3,
                                   max_len=7, term_frac=0.4 if seed % 3 else 0.1)
    t = HostTree()
    t.apply_ops(ops.words)
    dev_cap = int(t.export().scalars["device_used"]) + int(rng.integers(0, 12))
    for d in WL.legal_demotions(t.export(), rng, 0.3):
        ops.demote(d)
    probe = HostTree(dev_cap, BIG)
    probe.apply_ops(ops.words)
    free = dev_cap - int(probe.export().scalars["device_used"])
    fill = free - int(rng.integers(0, 10))
    filler = nw + 100
    parts = int(rng.integers(1, 5))
    for j in range(parts):
        L = fill // parts + (1 if j < fill % parts else 0)
        if L > 0:
            ops.insert([(1 << 40) + 1000 * j + q for q in range(L)], filler, 0)
    if rng.random() < 0.6:  # else the filler stays active: only the tree's own retired nodes can go
        ops.terminate(filler)
    P = WL.random_forecasts(rng, len(live), 3, agents + 1)
    return rng, ops, dev_cap, live, P, agents


@pytest.mark.parametrize("seed", range(60))
def test_prefetch_round_equals_reference_loop(gpu, seed):
    rng, ops, dev_cap, live, P, agents = _case(seed)
    t = HostTree(dev_cap, BIG)
    t.apply_ops(ops.words)
    soa = t.export()
    wf = np.array(live, dtype=np.int64)
    pol = Policy(num_agents=agents, k=3, gamma=0.7)
    pol.mirror(t)
    if live:
        pol.put_forecasts(wf, P)
    plan = pol.plan_conservative_prefetch(int(rng.integers(5, 200)))
    selected = plan.selected
    if not selected:
        pytest.skip("empty plan")
    pinned = _active_pinned(soa, rng, 2)
    free = soa.scalars["device_capacity"] - soa.scalars["device_used"]
    want_p, want_v = reference_round(ops.words, dev_cap, wf, P, selected, pinned)
    got_p, got_v = pol.prefetch_round(selected, free)
    assert got_p == want_p
    assert got_v == want_v
    # every candidate of the ranking (more demand than the conservative budget
    # admits): the round must skip exactly where the reference does
    every = [c[0] for c in plan.candidates]
    want_p, want_v = reference_round(ops.words, dev_cap, wf, P, every, pinned)
    got_p, got_v = pol.prefetch_round(every, free)
    assert got_p == want_p
    assert got_v == want_v


@pytest.mark.parametrize("seed", range(6))
def test_prefetch_round_larger_trees(gpu, seed):
    """Larger random trees (up to ~60 workflows, 600 ops): many candidates."""
    rng, ops, dev_cap, live, P, agents = _case(500 + seed, n_ops=(300, 600), n_wf=(30, 60))
    t = HostTree(dev_cap, BIG)
    t.apply_ops(ops.words)
    soa = t.export()
    wf = np.array(live, dtype=np.int64)
    pol = Policy(num_agents=agents, k=3, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    plan = pol.plan_conservative_prefetch(10 ** 6)
    assert len(plan.selected) > 5
    pinned = _active_pinned(soa, rng, 4)
    want_p, want_v = reference_round(ops.words, dev_cap, wf, P, plan.selected, pinned)
    got_p, got_v = pol.prefetch_round(plan.selected, soa.scalars["device_capacity"] - soa.scalars["device_used"])
    assert got_p == want_p
    assert got_v == want_v
