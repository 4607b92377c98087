"""Incremental device mirror (pbkv_mirror_delta).

CPU: the change log of the host tree (TrackedCacheTree over the reference
CacheTree) covers every node whose mirrored fields changed, through every
CacheTree mutator (insert / match with splits, termination, demote, promote,
drop, set_score), so a delta built from it is complete.

GPU: a context kept up to date with pbkv_mirror_sync after every batch equals
a fresh full mirror field by field (pbkv_mirror_verify), including pool
relocation, repacking and appended nodes, and its decisions equal the oracle
on the same snapshot.
"""
import numpy as np
import pytest

import workloads as WL
from oracle import Oracle
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_LRU, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy


def _grow(rng, t, n_wf=8, n_ops=60):
    ops, live = WL.random_tree_ops(rng, n_ops=n_ops, n_wf=n_wf, agents=4, alphabet=3, max_len=8)
    t.apply_ops(ops.words)
    return live, [n_wf]


@pytest.mark.parametrize("seed", range(40))
def test_change_log_covers_every_changed_node(seed):
    rng = np.random.default_rng(9100 + seed)
    t = HostTree(1 << 20, int(rng.integers(5, 60)) if seed % 4 == 0 else 1 << 20)
    live, nxt = _grow(rng, t)
    pos, _ = t.log(0)
    prev = t.export()
    for _ in range(10):
        ops = WL.churn_ops(rng, prev, live, nxt)
        t.apply_ops(ops.words)
        cur = t.export()
        end, ids = t.log(pos)
        assert ids is not None
        missing = WL.changed_nodes(prev, cur) - set(ids)
        assert not missing, sorted(missing)[:10]
        assert ids == sorted(ids)
        prev, pos = cur, end


def test_change_log_truncation_forces_full_sync():
    t = HostTree()
    t.synth(n_nodes=2000, n_workflows=32)
    end, _ = t.log(0)
    # a long burst of score writes overflows the bounded log
    from paper_2605_06472_b200.ops import OpStream

    ops = OpStream()
    for i in range(70000):
        ops.set_score(1 + i % 1999, float(i))
    t.apply_ops(ops.words)
    _, ids = t.log(end)
    assert ids is None


# ---------------------------------------------------------------------------- GPU
def _decision_matches_oracle(pol, soa, rng):
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    K = pol.k
    if wf.size:
        P = WL.random_forecasts(rng, wf.size, K, pol.num_agents + 1)
        pol.put_forecasts(wf, P)
        ref = Oracle.score_nodes(soa, wf, P, K, pol.gamma)
        soa = soa.copy()
        soa.score[:] = ref
    used = int(soa.len[1:][soa.tier[1:] == 0].sum())
    if used == 0:
        return
    needed = max(1, int(used * rng.uniform(0.05, 0.6)))
    locked = WL.random_locked(soa, rng, 0.05)
    mode = SCORE_RECOMPUTE if wf.size else 0
    g = pol.select_victims_hierarchical(needed, locked=locked, score_mode=mode)
    o = Oracle.select(soa, POLICY_HE, needed, locked)
    assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall)
    g = pol.select_victims(POLICY_LRU, needed, locked=locked)
    o = Oracle.select(soa, POLICY_LRU, needed, locked)
    assert (g.victims, g.freed, g.shortfall) == (o.victims, o.freed, o.shortfall)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_sync_equals_full_mirror(seed):
    rng = np.random.default_rng(9300 + seed)
    t = HostTree(1 << 20, int(rng.integers(5, 60)) if seed % 4 == 0 else 1 << 20)
    live, nxt = _grow(rng, t)
    pol = Policy(num_agents=4, k=3, gamma=0.7, device=0)
    pol.sync(t)  # first sync: full upload
    assert pol.verify(t) == -1
    for b in range(12):
        t.apply_ops(WL.churn_ops(rng, t.export(), live, nxt).words)
        pol.sync(t)
        assert pol.verify(t) == -1, f"batch {b}"
        if b % 4 == 3:
            _decision_matches_oracle(pol, t.export(), rng)


@pytest.mark.gpu
def test_sync_repacks_and_relocates():
    """Nodes that gain entries outgrow their pool segments and move to the
    pool top; enough moves trigger a repack -- the mirror stays exact."""
    rng = np.random.default_rng(5)
    t = HostTree()
    t.synth(n_nodes=3000, n_workflows=16, agents=4)
    pol = Policy(num_agents=4, k=3, device=0)
    pol.sync(t)
    live, nxt = list(range(5, 16)), [16]
    for b in range(40):
        # many new workflows matching the shared prefix: its entry list grows every batch
        from paper_2605_06472_b200.ops import OpStream

        ops = OpStream()
        for _ in range(20):
            w = nxt[0]
            nxt[0] += 1
            ops.match([(1 << 60) | i for i in range(32)], w, int(rng.integers(4)))
            if rng.random() < 0.5:
                ops.terminate(w)
        t.apply_ops(ops.words)
        pol.sync(t)
        assert pol.verify(t) == -1, f"batch {b}"
    _decision_matches_oracle(pol, t.export(), rng)


@pytest.mark.gpu
def test_plain_mirror_then_sync_is_full():
    """A context that last mirrored a snapshot (pbkv_mirror_full) re-mirrors
    in full on its first sync of a tree."""
    t = HostTree()
    t.synth(n_nodes=1500, n_workflows=16, agents=4)
    pol = Policy(num_agents=4, k=3, device=0)
    pol.mirror(t.export())
    pol.sync(t)
    assert pol.verify(t) == -1


def _records(soa, ids):
    """caller-built pbkv_node_delta records of `ids` from a snapshot"""
    from paper_2605_06472_b200._abi import NODE_DELTA_DTYPE

    r = np.zeros(len(ids), dtype=NODE_DELTA_DTYPE)
    wf, bits = [], []
    for k, i in enumerate(ids):
        r[k]["id"], r[k]["parent"], r[k]["len"] = i, soa.parent[i], soa.len[i]
        r[k]["ever_tagged"], r[k]["depth"] = soa.ever_tagged[i], soa.depth[i]
        r[k]["tier"], r[k]["retired"] = soa.tier[i], soa.retired[i]
        r[k]["last_access"], r[k]["score"] = soa.last_access[i], soa.score[i]
        a, b = int(soa.acc_off[i]), int(soa.acc_off[i + 1])
        r[k]["acc_begin"] = len(wf)
        wf += soa.acc_wf[a:b].tolist()
        bits += soa.acc_bits[a:b].tolist()
        r[k]["acc_end"] = len(wf)
    return r, np.array(wf, dtype=np.int64), np.array(bits, dtype=np.uint64)


def _totals(soa):
    keys = ("device_capacity", "device_used", "retired_device_tokens", "host_capacity", "host_used")
    return {k: int(soa.scalars[k]) for k in keys}


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_caller_delta_unordered_with_stale_duplicates(seed):
    """pbkv_mirror_delta on caller-built batches in any order, with stale
    records of the same node earlier in the batch: the last record wins."""
    rng = np.random.default_rng(9500 + seed)
    t = HostTree()
    live, nxt = _grow(rng, t)
    pol = Policy(num_agents=4, k=3, gamma=0.7, device=0)
    pol.mirror(t.export())
    pos = t.log_end()
    for b in range(6):
        before = t.export()
        t.apply_ops(WL.churn_ops(rng, before, live, nxt).words)
        cur = t.export()
        end, ids = t.log(pos)
        pos = end
        stale = [i for i in ids if i < before.n_nodes][: max(1, len(ids) // 3)]
        r_old, w_old, b_old = _records(before, stale) if stale else _records(cur, [])
        r_new, w_new, b_new = _records(cur, ids)
        perm = rng.permutation(len(r_new))
        r_new = r_new[perm]
        r_old["acc_begin"] += w_new.size
        r_old["acc_end"] += w_new.size
        recs = np.concatenate([r_old, r_new])  # stale first (they lose), then the current ones shuffled
        wf_all = np.concatenate([w_new, w_old]) if w_old.size else w_new
        bits_all = np.concatenate([b_new, b_old]) if b_old.size else b_new
        pol.apply_delta(recs, wf_all, bits_all, _totals(cur))
        assert pol.verify(cur) == -1, f"batch {b}"
    _decision_matches_oracle(pol, t.export(), rng)


@pytest.mark.gpu
def test_caller_delta_rejects_sparse_append():
    from paper_2605_06472_b200.api import PbkvError

    rng = np.random.default_rng(3)
    t = HostTree()
    _grow(rng, t)
    soa = t.export()
    pol = Policy(num_agents=4, k=3, device=0)
    pol.mirror(soa)
    r, w, b = _records(soa, [1])
    r["id"] = soa.n_nodes + 1  # skips id n_nodes
    with pytest.raises(PbkvError, match="dense"):
        pol.apply_delta(r, w, b, _totals(soa))
