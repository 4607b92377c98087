"""CPU check of the victim-order closed form the GPU kernels implement
(SURVEY.md fact 1 / App. B.2):

    order = eligible device nodes sorted by (eff(n), d(n))
    eff(n) = max key over n's device subtree, d(n) = depth(argmax) - depth(n)
    eligible = device, not root, no locked device node in the subtree
    victims = shortest prefix with sum(len) >= needed

compared against the oracle's greedy frontier (itself pinned to the reference
in test_oracle.py) on random trees, for every policy and many cuts.
"""
import math

import numpy as np
import pytest

import workloads as WL
from oracle import Oracle, RefTree, have_oracle, have_ref
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU

pytestmark = pytest.mark.skipif(not (have_oracle() and have_ref()), reason="oracle not built")


def py_key(soa, policy, n, remaining):
    retired = bool(soa.retired[n])
    last = int(soa.last_access[n])
    if policy == POLICY_LRU:
        return (0, 0.0, last, n)
    if policy == POLICY_LAE:
        return (0, float(soa.ever_tagged[n]), last, n) if retired else (1, 0.0, last, n)
    if policy == POLICY_HE:
        return (0, float(soa.ever_tagged[n]), last, n) if retired else (1, float(soa.score[n]), last, n)
    d = math.inf
    if not retired:
        for w, bits in soa.entries_of(n):
            seq = remaining[w]
            for k, a in enumerate(seq):
                if (bits >> a) & 1:
                    d = min(d, float(k + 1))
                    break
    return (0, 0.0, last, n) if math.isinf(d) else (1, -d, last, n)


def closed_form(soa, policy, needed, locked, remaining=None):
    n = soa.n_nodes
    dev = [soa.tier[i] == 0 for i in range(n)]
    depth = soa.depth
    children = [[] for _ in range(n)]
    for i in range(1, n):
        if dev[i]:
            children[soa.parent[i]].append(i)
    lk = set(locked)
    sub_locked = [False] * n
    eff = list(range(n))
    key = {i: py_key(soa, policy, i, remaining) for i in range(1, n) if dev[i]}
    # post-order over the device tree
    order, stack = [], [0]
    while stack:
        v = stack.pop()
        order.append(v)
        stack.extend(children[v])
    for v in reversed(order):
        if v == 0:
            continue
        sub_locked[v] = (v in lk) or any(sub_locked[c] for c in children[v])
        best = v
        for c in children[v]:
            if key[eff[c]] > key[best]:
                best = eff[c]
        eff[v] = best
    elig = [v for v in range(1, n) if dev[v] and not sub_locked[v]]
    elig.sort(key=lambda v: (key[eff[v]], depth[eff[v]] - depth[v]))
    victims, freed = [], 0
    for v in elig:
        if freed >= needed:
            break
        victims.append(v)
        freed += int(soa.len[v])
    return victims, freed, freed < needed


@pytest.mark.parametrize("seed", range(120))
def test_closed_form_equals_greedy_frontier(seed):
    rng = np.random.default_rng(1000 + seed)
    n_wf = int(rng.integers(2, 9))
    agents = int(rng.integers(2, 5))
    K = int(rng.integers(1, 4))
    ops, live = WL.random_tree_ops(rng, n_ops=int(rng.integers(5, 50)), n_wf=n_wf, agents=agents, alphabet=3,
                                   max_len=7)
    t = RefTree()
    t.apply_ops(ops.words)
    for d in WL.legal_demotions(t.export(), rng, 0.15):
        ops.demote(d)
    t = RefTree()
    t.apply_ops(ops.words)
    P = WL.random_forecasts(rng, len(live), K, agents + 1, coarse=bool(rng.random() < 0.5))
    if live:
        t.set_forecasts(live, P)
    t.refresh_nodes(None, K, 0.7)
    soa = t.export()
    remaining = {w: [int(a) for a in rng.integers(0, agents, size=int(rng.integers(0, 5)))] for w in live}
    locked = WL.random_locked(soa, rng, 0.08)
    used = int(soa.len[soa.tier == 0].sum())
    for pol in (POLICY_LRU, POLICY_LAE, POLICY_HE, POLICY_KVFLOW):
        for needed in sorted(set([1, 2, max(1, used // 5), max(1, used // 2), used, used + 3])):
            for lk in ([], locked):
                o = Oracle.select(soa, pol, needed, lk, remaining=remaining)
                cf = closed_form(soa, pol, needed, lk, remaining)
                assert cf == (o.victims, o.freed, o.shortfall), (pol, needed, lk)
