"""Node-set sharding (BASELINE config 4).

CPU (gloo, world_size 2): partition invariants, the variable-length
all-gather, and that every rank derives identical spine records from the
exchanged reports.  GPU: P logical shards on one B200 -- the sharded decision
(local cuts + spine records + merge + cut) must equal the single-context
selection on the whole tree and the CPU oracle, bit for bit.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as WL
from paper_2605_06472_b200 import shard as S
from paper_2605_06472_b200._abi import POLICY_HE, POLICY_LAE, POLICY_LRU, SCORE_CACHED, SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree


def synth(n=6000, w=192, seed=5):
    t = HostTree()
    t.synth(n_nodes=n, n_workflows=w, seed=seed)
    return t.export()


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_partition_invariants(P):
    soa = synth()
    shards = S.partition(soa, P)
    sp = shards[0].spine
    owned = np.concatenate([s.gids[~np.isin(s.gids, sp.gid)] for s in shards])
    # every non-spine node in exactly one shard
    assert np.array_equal(np.sort(owned), np.setdiff1d(np.arange(soa.n_nodes), sp.gid))
    for s in shards:
        assert np.all(np.diff(s.gids) > 0)  # local ids increase with global ids
        assert np.array_equal(s.gids[s.spine_local], sp.gid)
        loc = s.soa
        # parents map to the same global parent
        for i in range(1, loc.n_nodes):
            assert s.gids[loc.parent[i]] == soa.parent[s.gids[i]]
        # access entries stay inside the rank's WorkflowId block
        w = loc.acc_wf[: loc.n_entries]
        assert np.all((w >= s.wf_lo) & (w < s.wf_hi))
    # spine entries are split across ranks without loss, in rank (= id) order
    for j, g in enumerate(sp.gid.tolist()):
        parts = []
        for s in shards:
            li = s.spine_local[j]
            parts.extend(s.soa.acc_wf[s.soa.acc_off[li]:s.soa.acc_off[li + 1]].tolist())
        a, b = soa.acc_off[g], soa.acc_off[g + 1]
        assert parts == soa.acc_wf[a:b].tolist()


def test_key_packing_matches_order():
    ks = [S.make_key(0, 0.0, 5), S.make_key(0, 3.0, 1), S.make_key(1, 0.0, 0), S.make_key(1, 0.25, 9),
          S.make_key(1, 0.5, 0), S.make_key(1, 1e300, 0)]
    assert ks == sorted(ks)
    assert S.make_key(1, -0.0, 3) == S.make_key(1, 0.0, 3)


def _spine_fixture():
    sp = S.Spine(gid=np.array([0, 1]), parent=np.array([-1, 0]), depth=np.array([0, 1]), len=np.array([0, 32]),
                 tier=np.array([0, 0]), retired=np.array([0, 0]), ever=np.array([0, 9]),
                 last=np.array([0, 100], dtype=np.uint64), score=np.array([0.0, 2.5]))
    return sp


def test_spine_records_eligibility_and_eff():
    sp = _spine_fixture()
    rep = np.zeros((2, 2), dtype=S.SPINE_DTYPE)
    hi = S.make_key(1, 7.0, 3)
    rep[1, 1] = (hi[0], hi[1], 77, 5, 1, 0)
    lo = S.make_key(1, 0.1, 3)
    rep[0, 1] = (lo[0], lo[1], 12, 4, 1, 0)
    rec = S.spine_records(sp, rep, sp.score, POLICY_HE, set())
    assert rec.size == 1 and int(rec[0]["gid"]) == 1
    assert int(rec[0]["eff_gid"]) == 77 and int(rec[0]["d"]) == 4
    # own key wins when it is the maximum
    rep[1, 1]["has_eff"] = 0
    rec = S.spine_records(sp, rep, np.array([0.0, 9.0]), POLICY_HE, set())
    assert int(rec[0]["eff_gid"]) == 1 and int(rec[0]["d"]) == 0
    # a locked node below on any rank makes it ineligible
    rep[0, 1]["sublock"] = 1
    assert S.spine_records(sp, rep, sp.score, POLICY_HE, set()).size == 0
    rep[0, 1]["sublock"] = 0
    assert S.spine_records(sp, rep, sp.score, POLICY_HE, {1}).size == 0


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # variable-length all-gather of candidate records
        n = 3 + 4 * rank
        recs = np.zeros(n, dtype=S.CAND_DTYPE)
        recs["gid"] = np.arange(n) + 100 * rank
        t = torch.from_numpy(recs.view(np.uint8).copy())
        g, lens = S.allgather_var(dist, t, world)
        got = [np.frombuffer(g[r, :lens[r]].numpy().tobytes(), dtype=S.CAND_DTYPE)["gid"].tolist()
               for r in range(world)]
        # spine records from exchanged reports are identical on every rank
        sp = _spine_fixture()
        rep = np.zeros(2, dtype=S.SPINE_DTYPE)
        k = S.make_key(1, 5.0 + rank, 2 + rank)  # above the spine's own score (2.5)
        rep[1] = (k[0], k[1], 50 + rank, 3, 1, 0)
        rg, _ = S.allgather_var(dist, torch.from_numpy(rep.view(np.uint8).copy()), world)
        allrep = np.stack([np.frombuffer(rg[r].numpy().tobytes(), dtype=S.SPINE_DTYPE) for r in range(world)])
        srec = S.spine_records(sp, allrep, sp.score, POLICY_HE, set())
        q.put((rank, got, srec.tobytes()))
    finally:
        dist.destroy_process_group()


def test_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    want = [list(range(3)), [100 + i for i in range(7)]]
    assert res[0][1] == want and res[1][1] == want
    assert res[0][2] == res[1][2]  # identical spine records on both ranks
    rec = np.frombuffer(res[0][2], dtype=S.CAND_DTYPE)
    assert rec.size == 1 and int(rec[0]["eff_gid"]) == 51  # rank 1 reported the larger key


# ---- GPU: logical shards on one device ----------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("policy,mode", [(POLICY_HE, SCORE_RECOMPUTE), (POLICY_HE, SCORE_CACHED),
                                         (POLICY_LRU, SCORE_CACHED), (POLICY_LAE, SCORE_CACHED)])
def test_sharded_equals_single(gpu, P, policy, mode):
    from oracle import Oracle
    from paper_2605_06472_b200.api import Policy

    soa = synth(n=8000, w=256, seed=P)
    rng = np.random.default_rng(P)
    K, A = 4, 16
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    Pf = WL.random_forecasts(rng, wf.size, K, A + 1)
    ref_scores = Oracle.score_nodes(soa, wf, Pf, K, 0.7)
    soa.score[:] = ref_scores  # cached mode: the tree's scores are current
    single = Policy(num_agents=A, k=K, gamma=0.7)
    single.mirror(soa)
    single.put_forecasts(wf, Pf)
    shards = S.partition(soa, P)
    sps = []
    for s in shards:
        sp = S.ShardedPolicy(s, num_agents=A, k=K, gamma=0.7)
        mine = (wf >= s.wf_lo) & (wf < s.wf_hi)
        if mine.any():
            sp.pol.put_forecasts(wf[mine], Pf[mine])
        sps.append(sp)
    used = int(soa.len[soa.tier == 0][1:].sum())
    locked = WL.pinned_paths(soa, rng, 0.02) + [1] * (P == 3)  # P=3 also locks the shared prefix
    for frac in (0.001, 0.01, 0.1, 0.5, 2.0):
        needed = max(1, int(frac * used))
        got = S.global_select(sps, policy, mode, needed, locked)
        want = single.select_victims(policy, needed, locked=locked, score_mode=mode)
        assert got[0].tolist() == want.victims, f"P={P} frac={frac}: order differs"
        assert got[1] == want.freed and got[2] == want.shortfall
        if frac in (0.01, 0.5):
            o = Oracle.select(soa, policy, needed, locked)
            assert got[0].tolist() == o.victims and got[1] == o.freed


@pytest.mark.gpu
def test_chain_sum_bit_exact(gpu):
    """pbkv_chain_sum (the exact parallel rounding chain) against the serial
    IEEE loop, including ties, zeros, binade-edge values and long inputs."""
    from paper_2605_06472_b200.api import Policy

    rng = np.random.default_rng(3)
    segs = [rng.random(23000) * 1e-3,
            np.r_[0.0, 0.0, rng.random(100)],
            np.full(5000, 0.5) * 2.0 ** -rng.integers(0, 40, 5000),           # short mantissas: many ties
            rng.random(40000) * 2.0 ** rng.integers(-30, 3, 40000),
            np.array([1.0, 2.0 ** -53, 2.0 ** -53, 2.0 ** -52, 3 * 2.0 ** -53]),
            np.r_[rng.random(7) * 1e-300, rng.random(9000)],
            np.array([], dtype=np.float64)]
    x = np.concatenate(segs)
    off = np.cumsum([0] + [s.size for s in segs])
    pol = Policy(num_agents=4, k=3)
    from paper_2605_06472_b200 import shard as SH

    class _P:  # minimal holder to reuse ShardedPolicy.chain_sums
        pass

    h = _P()
    h.pol = pol
    h.dev = torch.device("cuda", 0)
    h.order_after_torch = lambda: SH.ShardedPolicy.order_after_torch(h)
    xt = torch.from_numpy(x).cuda()
    got = SH.ShardedPolicy.chain_sums(h, xt, off)
    for i, s in enumerate(segs):
        t = 0.0
        for v in s.tolist():
            t += v
        assert got[i] == t, f"segment {i}: {got[i]!r} != {t!r}"


def _dist_gpu_worker(rank, world, port, q):
    """world ranks on cuda:0 (gloo exchange): the per-rank decision path of
    global_select(dist=...) against the single-context selection."""
    import sys

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_06472_b200.api import Policy

        soa = synth(n=12000, w=256, seed=11)
        rng = np.random.default_rng(11)
        K, A = 4, 16
        wf = np.array(WL.workflows_of(soa), dtype=np.int64)
        Pf = WL.random_forecasts(rng, wf.size, K, A + 1)
        shards = S.partition(soa, world)
        me = S.ShardedPolicy(shards[rank], num_agents=A, k=K, gamma=0.7)
        mine = (wf >= shards[rank].wf_lo) & (wf < shards[rank].wf_hi)
        me.pol.put_forecasts(wf[mine], Pf[mine])
        used = int(soa.len[soa.tier == 0][1:].sum())
        locked = WL.pinned_paths(soa, rng, 0.02)
        out = []
        for frac in (0.01, 0.3, 2.0):
            needed = max(1, int(frac * used))
            v, fr, sf = S.global_select(me, POLICY_HE, SCORE_RECOMPUTE, needed, locked, dist=dist, world=world)
            out.append((v.tolist(), fr, sf))
        want = None
        if rank == 0:
            single = Policy(num_agents=A, k=K, gamma=0.7)
            single.mirror(soa)
            single.put_forecasts(wf, Pf)
            want = []
            for frac in (0.01, 0.3, 2.0):
                needed = max(1, int(frac * used))
                r = single.select_victims(POLICY_HE, needed, locked=locked, score_mode=SCORE_RECOMPUTE)
                want.append((r.victims, r.freed, r.shortfall))
        q.put((rank, out, want))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, "ERR " + traceback.format_exc(), None))
        sys.stderr.write(str(e))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_dist_exchange_two_ranks_equals_single(gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_dist_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert not isinstance(r[1], str), r[1]
    want = res[0][2]
    for rank, out, _ in res:
        assert [tuple(o) for o in out] == [tuple(w) for w in want], f"rank {rank} differs from single"


@pytest.mark.gpu
def test_interval_sums_bound(gpu):
    """pbkv_interval_sums (the sharded fast path's any-order spine sums):
    every output within its interval bound L * ulp(sum|x|) of the exact sum,
    over pieces scattered in the array (empty pieces and outputs included)."""
    import math

    import torch

    from paper_2605_06472_b200 import shard as SH

    from paper_2605_06472_b200.api import Policy

    rng = np.random.default_rng(3)
    x = np.r_[rng.random(50000) * 2.0 ** rng.integers(-20, 4, 50000), rng.random(3000) * 1e-200]
    pol = Policy(num_agents=4, k=3)

    class _P:
        pass

    h = _P()
    h.pol = pol
    h.dev = torch.device("cuda", 0)
    h.order_after_torch = lambda: SH.ShardedPolicy.order_after_torch(h)
    xt = torch.from_numpy(x).cuda()
    n_out = 7
    pieces, out_off = [], [0]
    for j in range(n_out):
        for _ in range(int(rng.integers(0, 4))):
            a = int(rng.integers(0, x.size))
            b = min(x.size, a + int(rng.integers(0, 20000)))
            pieces.append((a, b))
        out_off.append(len(pieces))
    got = SH.ShardedPolicy.interval_sums(h, xt.data_ptr(), np.array(pieces, dtype=np.int64).reshape(-1, 2),
                                         np.array(out_off, dtype=np.int64))
    for j in range(n_out):
        vals = np.concatenate([x[a:b] for a, b in pieces[out_off[j]:out_off[j + 1]]] or [np.zeros(0)])
        exact, mag = math.fsum(vals.tolist()), math.fsum(np.abs(vals).tolist())
        L = max(vals.size, 1)
        bound = 2.0 * L * (np.spacing(mag) if mag > 0 else 0.0)
        assert abs(got[j, 0] - exact) <= bound, (j, got[j, 0], exact, bound)
        assert abs(got[j, 1] - mag) <= bound, (j, got[j, 1], mag, bound)
