"""GPU parity: the CUDA path through the C ABI against the oracle.

Bit-exact for every integer/index result (victim and prefetch sequences,
freed tokens, shortfall, retired classification) and for the FP64 scores
(north_star allows 1e-6 relative; the design is bit-exact, asserted as such).
"""
import numpy as np
import pytest

import known_answers as KA
import workloads as WL
from oracle import Oracle, RefTree, have_oracle
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy, ValidationError

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_oracle(), reason="oracle not built")]


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def run_gpu(case: KA.Case):
    t = HostTree(case.dev_cap, case.host_cap)
    t.apply_ops(case.ops.words)
    pol = Policy(num_agents=case.agents, k=case.k, gamma=case.gamma)
    pol.mirror(t)
    wf, P = case.forecast_arrays()
    if len(wf):
        pol.put_forecasts(wf, P)
    a = case.action
    if a[0] == "score":
        return pol.score_nodes(a[1])
    if a[0] == "value":
        return pol.value_nodes(a[1])
    if a[0] == "select":
        return pol.select_victims(a[1], a[2], locked=a[3])
    if a[0] == "select_kvflow":
        return pol.select_victims_kvflow(a[1], a[3], locked=a[2])
    if a[0] == "plan":
        if a[3] < 0:
            return pol.plan_conservative_prefetch(a[1], a[2])
        return pol.plan_aggressive_prefetch(a[1], a[3], a[2])
    raise AssertionError(a)


@pytest.mark.parametrize("case", KA.cases(), ids=lambda c: c.name)
def test_known_answers_gpu(gpu, case):
    if case.error:
        with pytest.raises(ValidationError) as ei:
            run_gpu(case)
        assert str(ei.value) == case.error
    else:
        KA.check(case, run_gpu(case))


def _instance(seed, coarse=None):
    rng = np.random.default_rng(seed)
    n_wf = int(rng.integers(2, 10))
    agents = int(rng.integers(2, 6))
    K = int(rng.integers(1, 6))
    ops, live = WL.random_tree_ops(rng, n_ops=int(rng.integers(5, 70)), n_wf=n_wf, agents=agents, alphabet=3,
                                   max_len=7)
    t = HostTree()
    t.apply_ops(ops.words)
    for d in WL.legal_demotions(t.export(), rng, 0.15):
        ops.demote(d)
    t = HostTree()
    t.apply_ops(ops.words)
    if coarse is None:
        coarse = bool(rng.random() < 0.5)
    P = WL.random_forecasts(rng, len(live), K, agents + 1, coarse=coarse)
    return rng, t, live, P, K, agents


@pytest.mark.parametrize("seed", range(80))
def test_random_trees_gpu_equals_oracle(gpu, seed):
    rng, t, live, P, K, agents = _instance(seed)
    gamma = float(rng.uniform(0.1, 0.95))
    wf = np.array(live, dtype=np.int64)
    soa = t.export()
    pol = Policy(num_agents=agents, k=K, gamma=gamma)
    pol.mirror(t)
    if live:
        pol.put_forecasts(wf, P)
    # stage 2: every node, bit-exact
    ref_scores = Oracle.score_nodes(soa, wf, P, K, gamma)
    got = pol.score_all()
    assert np.array_equal(bits(got), bits(ref_scores))
    # refreshed cached scores -> mirror again (the simulator's state at a decision)
    soa.score[:] = ref_scores
    pol.mirror(soa)
    remaining = {w: [int(a) for a in rng.integers(0, agents, size=int(rng.integers(0, 6)))] for w in live}
    locked = WL.random_locked(soa, rng, 0.08)
    used = int(soa.len[soa.tier == 0].sum())
    cuts = sorted(set([1, 2, max(1, used // 7), max(1, used // 3), max(1, used), used + 5]))
    for pol_id in (POLICY_LRU, POLICY_LAE, POLICY_HE, POLICY_KVFLOW):
        for needed in cuts:
            for lk in ([], locked):
                o = Oracle.select(soa, pol_id, needed, lk, remaining=remaining)
                g = pol.select_victims(pol_id, needed, remaining=remaining, locked=lk)
                assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), (pol_id, needed, lk)
                if pol_id == POLICY_HE:
                    g2 = pol.select_victims_hierarchical(needed, locked=lk, score_mode=SCORE_RECOMPUTE)
                    assert (g2.victims, g2.freed, g2.shortfall) == (o.victims, o.freed, o.shortfall)
    for bw, rho in ((7, -1.0), (50, -1.0), (10 ** 6, -1.0), (40, 0.2), (10 ** 6, 1.0)):
        o = Oracle.plan(soa, wf, P, bw, 1, rho)
        g = pol.plan_conservative_prefetch(bw) if rho < 0 else pol.plan_aggressive_prefetch(bw, rho)
        assert [c[0] for c in g.candidates] == [c[0] for c in o.candidates]
        assert np.array_equal(bits([c[1] for c in g.candidates]), bits([c[1] for c in o.candidates]))
        assert (g.selected, g.selected_tokens, g.budget_space, g.budget_bw, g.displacement_budget) == \
               (o.selected, o.selected_tokens, o.budget_space, o.budget_bw, o.displacement_budget)


def _heavy_node_tree(n_wf, agents, rng):
    """one node tagged by n_wf workflows (the shared-prefix shape) plus a few leaves"""
    from paper_2605_06472_b200.ops import OpStream

    ops = OpStream()
    for w in range(n_wf):
        ops.insert([1, 2, 3, 4, 100 + (w % 7)], w, int(rng.integers(agents)))
        if rng.random() < 0.3:
            ops.insert([1, 2, 3, 4], w, int(rng.integers(agents)))
    return ops


@pytest.mark.parametrize("n_wf,K,coarse", [(40, 3, False), (700, 8, False), (3000, 8, False), (2500, 4, True),
                                           (5000, 1, False)])
def test_heavy_segment_exact_chain(gpu, n_wf, K, coarse):
    """The parallel-in-binade evaluation of the serial Eq. 2 chain on a node
    with thousands of tagged workflows is bit-identical to the sequential sum."""
    rng = np.random.default_rng(n_wf * 10 + K)
    agents = 9
    ops = _heavy_node_tree(n_wf, agents, rng)
    t = HostTree()
    t.apply_ops(ops.words)
    soa = t.export()
    wf = np.arange(n_wf, dtype=np.int64)
    P = WL.random_forecasts(rng, n_wf, K, agents + 1, coarse=coarse)
    if not coarse:
        # tiny negative probabilities are legal (forecast.hpp:29) and exercise the event path
        P[::17, 0, 1] += P[::17, 0, 0] + 1e-13
        P[::17, 0, 0] = -1e-13
    pol = Policy(num_agents=agents, k=K, gamma=0.5 if coarse else 0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    got = pol.score_all()
    ref = Oracle.score_nodes(soa, wf, P, K, 0.5 if coarse else 0.7)
    assert np.array_equal(bits(got), bits(ref))
    heavy = [i for i in range(soa.n_nodes) if soa.acc_off[i + 1] - soa.acc_off[i] > 32]
    assert heavy, "no heavy node generated"
    v = pol.value_nodes(heavy)
    assert np.array_equal(bits(v), bits(Oracle.value_nodes(soa, wf, P, heavy)))


@pytest.mark.parametrize("n_nodes,n_wf,K", [(10_000, 256, 4), (200_000, 2048, 8)])
def test_synthetic_config_parity(gpu, n_nodes, n_wf, K):
    """Config 2 shape (and a 200K intermediate): the full pipeline -- Eq. 2 over
    every node, HE victim order at 0.1%..50% need with a pinned locked set, in
    cached and recompute modes, and the conservative prefetch plan."""
    t = HostTree()
    t.synth(n_nodes=n_nodes, n_workflows=n_wf)
    soa = t.export()
    rng = np.random.default_rng(12345)
    live = WL.workflows_of(soa)
    wf = np.array(live, dtype=np.int64)
    P = WL.random_forecasts(rng, len(live), K, 17)
    pol = Policy(num_agents=16, k=K, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    scores = pol.score_all()
    ref = Oracle.score_nodes(soa, wf, P, K, 0.7)
    assert np.array_equal(bits(scores), bits(ref))
    soa.score[:] = ref
    pol.mirror(soa)
    locked = WL.pinned_paths(soa, rng, 0.01)
    used = int(soa.len[soa.tier == 0][1:].sum())
    for frac in (0.001, 0.01, 0.1, 0.5, 1.5):  # 1.5: shortfall, every eligible node (take-all path)
        needed = max(1, int(frac * used))
        o = Oracle.select(soa, POLICY_HE, needed, locked)
        g = pol.select_victims_hierarchical(needed, locked=locked)
        assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall), frac
        g2 = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        assert (g2.victims, g2.freed, g2.shortfall) == (o.victims, o.freed, o.shortfall), frac
        # retired classification of the victims
        assert all(soa.retired[v] in (0, 1) for v in g.victims)
    for bw in (512, 10 ** 9):
        o = Oracle.plan(soa, wf, P, bw)
        g = pol.plan_conservative_prefetch(bw)
        assert [c[0] for c in g.candidates] == [c[0] for c in o.candidates]
        assert g.selected == o.selected and g.selected_tokens == o.selected_tokens


def test_async_forecast_put_and_drop(gpu):
    """put_forecasts(validate_now=False) (the shim's pbkv_forecast_put_async):
    the validation error surfaces at the next call that reads the status word,
    with the reference's message; a drop is stream-ordered (no sync) and the
    next decision sees the forecast missing."""
    from paper_2605_06472_b200.ops import OpStream

    t = HostTree()
    t.apply_ops(OpStream().insert([1, 2], 7, 0).insert([3], 8, 1).words)
    pol = Policy(num_agents=2, k=1, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts([7, 8], np.array([[[0.5, 0.3, 0.2]], [[0.5, 0.3, 0.2]]]))
    ok = pol.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)
    pol.put_forecasts([7], np.array([[[1.1, -0.1, 0.0]]]), validate_now=False)  # returns without the check
    with pytest.raises(ValidationError, match="negative forecast probability"):
        pol.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)
    pol.put_forecasts([7], np.array([[[0.5, 0.3, 0.2]]]), validate_now=False)
    again = pol.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)
    assert (again.victims, again.freed) == (ok.victims, ok.freed)
    pol.drop_forecasts([8])
    with pytest.raises(ValidationError, match="missing forecast for active workflow 8"):
        pol.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)


def test_errors_match_reference(gpu):
    t = HostTree()
    from paper_2605_06472_b200.ops import OpStream

    t.apply_ops(OpStream().insert([1, 2], 7, 0).insert([3], 8, 1).words)
    pol = Policy(num_agents=2, k=3, gamma=0.7)
    pol.mirror(t)
    with pytest.raises(ValidationError, match="^missing forecast for active workflow 7$"):
        pol.score_all()
    with pytest.raises(ValidationError, match="eviction request must free a positive amount"):
        pol.select_victims_lru(0)
    with pytest.raises(ValidationError, match="negative forecast probability"):
        pol.put_forecasts([7], np.array([[[1.1, -0.1, 0.0]]]))
    with pytest.raises(ValidationError, match="does not sum to 1"):
        pol.put_forecasts([7], np.array([[[0.5, 0.2, 0.2]]]))
    pol.put_forecasts([7, 8], np.array([[[0.5, 0.3, 0.2]], [[0.5, 0.3, 0.2]]]))
    with pytest.raises(ValidationError, match="forecast horizon shorter than the scoring horizon"):
        pol.score_all()
    with pytest.raises(ValidationError, match="rho must be in"):
        pol.plan_aggressive_prefetch(100, 1.5)
    # HE recompute with a missing forecast on an eligible active node
    pol2 = Policy(num_agents=2, k=1, gamma=0.7)
    pol2.mirror(t)
    pol2.put_forecasts([8], np.array([[[0.5, 0.3, 0.2]]]))
    with pytest.raises(ValidationError, match="missing forecast for active workflow 7"):
        pol2.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)
    # an entry whose agent bits all fall outside [0, A) reads no forecast row:
    # the missing forecast must still raise (scoring.hpp:70-71)
    t3 = HostTree()
    t3.apply_ops(OpStream().insert([5, 6], 9, 3).insert([5, 7], 10, 0).words)
    for K in (1, 3, 8):
        pol3 = Policy(num_agents=2, k=K, gamma=0.7)
        pol3.mirror(t3)
        pol3.put_forecasts([10], np.full((1, K, 3), 1.0 / 3.0))
        with pytest.raises(ValidationError, match="^missing forecast for active workflow 9$"):
            pol3.score_all()
        with pytest.raises(ValidationError, match="missing forecast for active workflow 9"):
            pol3.select_victims_hierarchical(1, score_mode=SCORE_RECOMPUTE)


def test_ctx_wait_stream_orders_device_inputs(gpu):
    """pbkv_ctx_wait_stream: a locked list written late on a torch stream
    (behind a 50 ms spin) is seen by a device-input decision enqueued after
    the wait -- no host synchronisation, same victims as the host-input call."""
    import ctypes as C

    import torch

    from paper_2605_06472_b200 import _abi

    t = HostTree()
    t.synth(n_nodes=20000, n_workflows=128, agents=8, seed=5)
    soa = t.export()
    rng = np.random.default_rng(5)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, 4, 9)
    pol = Policy(num_agents=8, k=4, gamma=0.7)
    pol.mirror(t)
    pol.put_forecasts(wf, P)
    locked = np.asarray(WL.pinned_paths(soa, rng, 0.05), dtype=np.int32)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = used // 3
    want = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    dev = torch.device("cuda", 0)
    src = torch.from_numpy(locked).to(dev)
    torch.cuda.synchronize()
    s = torch.cuda.Stream(device=dev)
    locked_d = torch.zeros_like(src)
    victims = torch.zeros(soa.n_nodes, dtype=torch.int32, device=dev)
    res = torch.zeros(3, dtype=torch.int64, device=dev)
    with torch.cuda.stream(s):
        torch.cuda._sleep(100_000_000)  # ~50 ms of spinning before the write
        locked_d.copy_(src)
    pol._c(_abi.lib().pbkv_ctx_wait_stream(pol.handle, C.c_void_p(s.cuda_stream)))
    pol.select_dev(POLICY_HE, SCORE_RECOMPUTE, needed, locked_d.data_ptr(), int(locked.size), victims.data_ptr(),
                   soa.n_nodes, res.data_ptr())
    torch.cuda.synchronize()
    nv, freed, sf = (int(x) for x in res.cpu().tolist())
    assert (victims[:nv].cpu().tolist(), freed, bool(sf)) == (want.victims, want.freed, want.shortfall)
