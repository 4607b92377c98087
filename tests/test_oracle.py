"""Pins the CPU oracle (oracle/pbkv_oracle.c) against the reference itself.

* the reference's own Catch2 suite, compiled unmodified (oracle/_ref/flowkv_tests)
* the known-answer vectors of the reference tests (tests/known_answers.py),
  through both the real flowkv::CacheTree + reference policies (RefTree) and
  the C restatement (Oracle)
* random differential: Oracle == reference on random trees, bit-exact
"""
import os
import subprocess

import numpy as np
import pytest

import known_answers as KA
import workloads as WL
from oracle import Oracle, OracleError, RefTree, have_oracle, have_ref
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.skipif(not (have_oracle() and have_ref()), reason="oracle not built (run build())")


def test_reference_catch2_suite_passes():
    exe = os.path.join(ROOT, "oracle", "_ref", "flowkv_tests")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built (make -C oracle ref-tests)")
    r = subprocess.run([exe, "~one cell and one seed gives exactly one metrics row"], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


def run_ref(case: KA.Case):
    t = RefTree(case.dev_cap, case.host_cap)
    t.apply_ops(case.ops.words)
    wf, P = case.forecast_arrays()
    if len(wf):
        t.set_forecasts(wf, P)
    a = case.action
    if a[0] == "score":
        return t.score_nodes(a[1], case.k, case.gamma)
    if a[0] == "value":
        return t.value_nodes(a[1])
    if a[0] == "select":
        return t.select(a[1], a[2], a[3])
    if a[0] == "select_kvflow":
        t.set_remaining(a[3])
        return t.select(POLICY_KVFLOW, a[1], a[2])
    if a[0] == "plan":
        return t.plan(a[1], a[2], a[3])
    raise AssertionError(a)


def run_oracle(case: KA.Case):
    t = RefTree(case.dev_cap, case.host_cap)
    t.apply_ops(case.ops.words)
    soa = t.export()
    wf, P = case.forecast_arrays()
    a = case.action
    if a[0] == "score":
        return Oracle.score_nodes(soa, wf, P, case.k, case.gamma, a[1])
    if a[0] == "value":
        return Oracle.value_nodes(soa, wf, P, a[1])
    if a[0] == "select":
        return Oracle.select(soa, a[1], a[2], a[3])
    if a[0] == "select_kvflow":
        return Oracle.select(soa, POLICY_KVFLOW, a[1], a[2], remaining=a[3])
    if a[0] == "plan":
        return Oracle.plan(soa, wf, P, a[1], a[2], a[3])
    raise AssertionError(a)


@pytest.mark.parametrize("case", KA.cases(), ids=lambda c: c.name)
@pytest.mark.parametrize("impl", ["reference", "oracle"])
def test_known_answers(case, impl):
    run = run_ref if impl == "reference" else run_oracle
    if case.error:
        with pytest.raises(OracleError) as ei:
            run(case)
        assert str(ei.value) == case.error
    else:
        KA.check(case, run(case))


def _random_instance(seed):
    rng = np.random.default_rng(seed)
    n_wf = int(rng.integers(2, 10))
    agents = int(rng.integers(2, 6))
    K = int(rng.integers(1, 5))
    ops, live = WL.random_tree_ops(rng, n_ops=int(rng.integers(5, 60)), n_wf=n_wf, agents=agents,
                                   alphabet=3, max_len=7)
    t = RefTree()
    t.apply_ops(ops.words)
    soa = t.export()
    for d in WL.legal_demotions(soa, rng, 0.15):
        ops.demote(d)
    t = RefTree()
    t.apply_ops(ops.words)
    coarse = bool(rng.random() < 0.5)
    P = WL.random_forecasts(rng, len(live), K, agents + 1, coarse=coarse)
    if live:
        t.set_forecasts(live, P)
    return rng, t, ops, live, P, K, agents


@pytest.mark.parametrize("seed", range(150))
def test_oracle_matches_reference_random(seed):
    rng, t, ops, live, P, K, agents = _random_instance(seed)
    gamma = float(rng.uniform(0.1, 0.95))
    wf = np.array(live, dtype=np.int64)
    # refresh every node's cached score through the reference (scoring.hpp:95)
    t.refresh_nodes(None, K, gamma)
    soa = t.export()
    ids = list(range(soa.n_nodes))
    ref_scores = t.score_nodes(ids, K, gamma)
    orc_scores = Oracle.score_nodes(soa, wf, P, K, gamma)
    assert np.array_equal(ref_scores.view(np.uint64), orc_scores.view(np.uint64))
    locked = WL.random_locked(soa, rng, 0.08)
    used = int(soa.len[(soa.tier == 0)][1:].sum()) if soa.n_nodes > 1 else 0
    cuts = sorted(set([1, max(1, used // 7), max(1, used // 3), max(1, used), used + 5]))
    remaining = {w: [int(a) for a in rng.integers(0, agents, size=int(rng.integers(0, 6)))] for w in live}
    t.set_remaining(remaining)
    for pol in (POLICY_LRU, POLICY_LAE, POLICY_HE, POLICY_KVFLOW):
        for needed in cuts:
            for lk in ([], locked):
                r = t.select(pol, needed, lk)
                o = Oracle.select(soa, pol, needed, lk, remaining=remaining)
                assert (r.victims, r.freed, r.shortfall) == (o.victims, o.freed, o.shortfall), (pol, needed, lk)
    for bw, rho in ((7, -1.0), (50, -1.0), (10 ** 6, -1.0), (40, 0.2), (10 ** 6, 1.0)):
        r = t.plan(bw, 1, rho)
        o = Oracle.plan(soa, wf, P, bw, 1, rho)
        assert r.candidates == o.candidates
        assert (r.selected, r.selected_tokens, r.budget_space, r.budget_bw, r.displacement_budget) == \
               (o.selected, o.selected_tokens, o.budget_space, o.budget_bw, o.displacement_budget)
