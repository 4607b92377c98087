"""Seeded workload generators shared by the parity tests and bench.py.

Random small trees follow SURVEY.md App. A.3 (random inserts and matches over
a small alphabet, several workflows, terminations, demotions, coarse
forecasts to force exact score ties, random locked sets).  Everything is a
pure function of the seed.
"""
from __future__ import annotations

import numpy as np

from paper_2605_06472_b200.ops import OpStream


def random_forecasts(rng: np.random.Generator, n: int, K: int, V1: int, coarse: bool = False) -> np.ndarray:
    """iid-exponential simplex rows (rng.hpp:58-67 / theory.hpp:225-233 shape).
    coarse=True draws from a handful of one-hot / half-half rows so that many
    nodes tie exactly on score."""
    if not coarse:
        x = -np.log1p(-rng.random((n, K, V1)))
        return x / x.sum(axis=2, keepdims=True)
    P = np.zeros((n, K, V1))
    for i in range(n):
        for k in range(K):
            a = int(rng.integers(V1))
            b = int(rng.integers(V1))
            if a == b:
                P[i, k, a] = 1.0
            else:
                P[i, k, a] = 0.5
                P[i, k, b] = 0.5
    return P


def random_tree_ops(rng: np.random.Generator, n_ops: int = 40, n_wf: int = 6, agents: int = 4, alphabet: int = 3,
                    max_len: int = 7, term_frac: float = 0.3, demote_frac: float = 0.15,
                    host_capacity: int | None = None):
    """Build an op stream by simulating enough of the tree to only emit legal
    demotions.  Returns (ops, live_workflows).  The tree itself is built by the
    caller (HostTree or RefTree) from the op stream."""
    ops = OpStream()
    live = list(range(n_wf))
    for _ in range(n_ops):
        w = int(rng.choice(live)) if live else 0
        L = int(rng.integers(1, max_len + 1))
        toks = [int(t) for t in rng.integers(0, alphabet, size=L)]
        agent = int(rng.integers(agents))
        if rng.random() < 0.7:
            ops.insert(toks, w, agent)
        else:
            ops.match(toks, w, agent)
    n_term = int(round(term_frac * n_wf))
    terminated = [int(w) for w in rng.choice(n_wf, size=n_term, replace=False)] if n_term else []
    for w in terminated:
        ops.terminate(w)
    live = [w for w in range(n_wf) if w not in terminated]
    return ops, live


def legal_demotions(soa, rng: np.random.Generator, frac: float, rounds: int = 2) -> list[int]:
    """Pick device leaves to demote (each must be a leaf at its turn): repeated
    leaf peeling on the exported SoA image."""
    n = soa.n_nodes
    tier = soa.tier.copy()
    parent = soa.parent
    out: list[int] = []
    for _ in range(rounds):
        dc = np.zeros(n, dtype=np.int64)
        dev = (tier == 0)
        dev[0] = False
        np.add.at(dc, parent[1:][dev[1:]], 1)
        leaves = [i for i in range(1, n) if tier[i] == 0 and dc[i] == 0]
        rng.shuffle(leaves)
        k = int(round(frac * len(leaves)))
        for i in leaves[:k]:
            tier[i] = 1
            out.append(i)
    return out


def random_locked(soa, rng: np.random.Generator, frac: float = 0.08) -> list[int]:
    n = soa.n_nodes
    if n <= 1:
        return []
    k = int(rng.binomial(n - 1, frac))
    return sorted(set(int(x) for x in rng.integers(1, n, size=k)))


def pinned_paths(soa, rng: np.random.Generator, frac: float = 0.01) -> list[int]:
    """Ancestors of a fraction of device leaves plus the leaves (the image of
    Simulator::pinned_nodes, simulator.hpp:437-446)."""
    n = soa.n_nodes
    tier, parent = soa.tier, soa.parent
    dev = tier == 0
    dc = np.zeros(n, dtype=np.int64)
    m = dev.copy()
    m[0] = False
    np.add.at(dc, parent[1:][m[1:]], 1)
    leaves = np.nonzero(m & (dc == 0))[0]
    if leaves.size == 0:
        return []
    k = max(1, int(frac * leaves.size))
    pick = rng.choice(leaves, size=min(k, leaves.size), replace=False)
    locked = set()
    for v in pick.tolist():
        while v > 0:
            if v in locked:
                break
            locked.add(v)
            v = int(parent[v])
    return sorted(locked)


def workflows_of(soa) -> list[int]:
    return sorted(set(soa.acc_wf[: soa.n_entries].tolist()))


def churn_ops(rng: np.random.Generator, soa, live: list[int], next_wf: list[int], *, n_insert: int = 6,
              n_match: int = 3, p_term: float = 0.3, n_demote: int = 4, n_promote: int = 2, n_drop: int = 1,
              n_score: int = 3, alphabet: int = 3, max_len: int = 7, agents: int = 4) -> OpStream:
    """One batch of tree mutations between two decisions, legal against the
    current snapshot `soa` (every CacheTree mutator: inserts / matches that
    split nodes, a termination, demotions of device leaves, promotions and
    drops of host nodes, cached-score writes).  `live` / `next_wf` are
    updated in place (terminated workflows leave, fresh ones join)."""
    ops = OpStream()
    n = soa.n_nodes
    # demotions of current device leaves, promotions / drops of host nodes
    # under device parents: legal against the snapshot, so they come first
    tier, parent = soa.tier, soa.parent
    dev = tier == 0
    dc = np.zeros(n, dtype=np.int64)
    m = dev.copy()
    m[0] = False
    np.add.at(dc, parent[1:][m[1:]], 1)
    leaves = np.nonzero(m & (dc == 0))[0]
    hosts = [i for i in range(1, n) if tier[i] == 1 and tier[parent[i]] == 0]
    rng.shuffle(hosts)
    promote = hosts[:n_promote]
    keep = {int(parent[i]) for i in promote}  # parents of promoted nodes stay on the device
    leaves = np.array([i for i in leaves.tolist() if i not in keep], dtype=np.int64)
    if leaves.size:
        for i in rng.choice(leaves, size=min(n_demote, leaves.size), replace=False).tolist():
            ops.demote(int(i))
    for i in promote:
        ops.promote(int(i))
    for i in hosts[n_promote:n_promote + n_drop]:
        ops.drop(int(i))
    for _ in range(n_insert + n_match):
        if not live:
            live.append(next_wf[0])
            next_wf[0] += 1
        w = int(rng.choice(live))
        toks = [int(t) for t in rng.integers(0, alphabet, size=int(rng.integers(1, max_len + 1)))]
        agent = int(rng.integers(agents))
        if rng.random() < n_insert / max(1, n_insert + n_match):
            ops.insert(toks, w, agent, int(rng.integers(1, 6)) if rng.random() < 0.2 else -1)
        else:
            ops.match(toks, w, agent)
    if live and rng.random() < p_term:
        w = int(rng.choice(live))
        live.remove(w)
        ops.terminate(w)
        live.append(next_wf[0])
        next_wf[0] += 1
    for i in rng.integers(1, max(n, 2), size=n_score if n > 1 else 0).tolist():
        ops.set_score(int(i), float(rng.random()))
    return ops


def changed_nodes(prev, cur) -> set[int]:
    """Ids whose mirrored fields (cache.hpp:54-69 read side, depth) or access
    entries differ between two snapshots, plus every new id."""
    out = set(range(prev.n_nodes, cur.n_nodes))
    n = prev.n_nodes
    for f in ("parent", "len", "tier", "retired", "last_access", "ever_tagged", "depth"):
        a, b = getattr(prev, f)[:n], getattr(cur, f)[:n]
        out.update(np.nonzero(a != b)[0].tolist())
    out.update(np.nonzero(prev.score[:n].view(np.uint64) != cur.score[:n].view(np.uint64))[0].tolist())
    for i in range(n):
        if prev.entries_of(i) != cur.entries_of(i):
            out.add(i)
    return out
