"""Node-set sharding of stages 2-3 across GPUs (BASELINE config 4).

One process per GPU.  Each rank keeps its shard of the radix tree resident
(the subtrees it owns plus a copy of the spine: the ancestors whose subtrees
span ranks) in its own pbkv context, and per decision:

  1. runs the local selection (pbkv_shard_select): spine excluded, records of
     its local cut (shortest local prefix with sum(len) >= needed -- an upper
     bound on its share of the global prefix) and one report per spine node;
  2. HE with recomputed scores: the Eq. 2 products of its workflows' entries
     on the spine nodes (pbkv_shard_spine_products) are all-gathered; ranks
     own contiguous WorkflowId blocks, so rank order IS the reference's
     summation order (std::map, cache.hpp:64) and every rank evaluates the
     spine scores' exact chains (pbkv_chain_sum) bit-identically;
  3. all-gathers counts, records and spine reports (torch.distributed: NCCL
     over NVLink on GPUs, gloo in the CPU tests);
  4. turns the reports into the spine's own records (host, a handful of
     nodes) and merges every run + the spine run with the global cut on the
     device (pbkv_merge_cut).

No data-path work is duplicated across ranks except the spine (O(#spine)).
The result equals the single-GPU selection on the whole tree (and hence the
reference's greedy frontier, policies.hpp:50-83): tests/test_shard.py.
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU, SCORE_RECOMPUTE, SoAArrays, ptr

CAND_DTYPE = np.dtype([("w0", "<u8"), ("w1", "<u8"), ("eff_gid", "<i4"), ("gid", "<i4"), ("d", "<i4"),
                       ("len", "<i4")])
SPINE_DTYPE = np.dtype([("w0", "<u8"), ("w1", "<u8"), ("eff_gid", "<i4"), ("eff_depth", "<i4"),
                        ("has_eff", "<i4"), ("sublock", "<i4")])


class CandC(C.Structure):
    _fields_ = [("w0", C.c_uint64), ("w1", C.c_uint64), ("eff_gid", C.c_int32), ("gid", C.c_int32),
                ("d", C.c_int32), ("len", C.c_int32)]


class SpineInfoC(C.Structure):
    _fields_ = [("w0", C.c_uint64), ("w1", C.c_uint64), ("eff_gid", C.c_int32), ("eff_depth", C.c_int32),
                ("has_eff", C.c_int32), ("sublock", C.c_int32)]


# ---- CandidateKey packing (policies.hpp:40-48; common.cuh make_key) -----------------
def enc_rank(r: float) -> int:
    if r == 0.0:
        r = 0.0  # -0.0 == +0.0 under std::tie
    b = struct.unpack("<Q", struct.pack("<d", r))[0]
    return (~b) & 0xFFFFFFFFFFFFFFFF if b >> 63 else b | (1 << 63)


def make_key(cls: int, rank: float, last: int) -> tuple[int, int]:
    e = enc_rank(rank)
    return (cls << 63) | (e >> 1), ((e & 1) << 63) | int(last)


def node_key(policy: int, retired: bool, ever: int, last: int, score: float) -> tuple[int, int]:
    if policy == POLICY_LRU:
        return make_key(0, 0.0, last)
    if policy == POLICY_LAE:
        return make_key(0, float(ever), last) if retired else make_key(1, 0.0, last)
    if policy == POLICY_HE:
        return make_key(0, float(ever), last) if retired else make_key(1, score, last)
    raise ValueError("kvflow is not supported on a sharded tree")


# ---- the spine -----------------------------------------------------------------------
@dataclass
class Spine:
    """Global fields of the spine nodes, identical on every rank; index j order
    is the order of pbkv_shard_set / the reports."""
    gid: np.ndarray        # int64
    parent: np.ndarray     # spine index of the parent, -1 for the root
    depth: np.ndarray
    len: np.ndarray
    tier: np.ndarray
    retired: np.ndarray
    ever: np.ndarray
    last: np.ndarray
    score: np.ndarray      # cached (CacheTree) score

    @property
    def n(self) -> int:
        return int(self.gid.size)


def spine_records(sp: Spine, reports: np.ndarray, scores: np.ndarray, policy: int,
                  locked_gids: set[int]) -> np.ndarray:
    """Records of the eligible spine nodes from the ranks' reports
    ([P, n_spine] SPINE_DTYPE).  eff(s) = max over s's own key, its spine
    children's eff and every rank's maximum below s; eligible iff device, not
    the root, and no locked node below it on any rank (App. B.2)."""
    n = sp.n
    eff: list[tuple] = [None] * n  # (w0, w1, gid, depth)
    sub = [False] * n
    order = sorted(range(n), key=lambda j: -int(sp.depth[j]))  # children before parents
    for j in order:
        k = node_key(policy, bool(sp.retired[j]), int(sp.ever[j]), int(sp.last[j]), float(scores[j]))
        best = None
        if int(sp.tier[j]) == 0:
            best = (k[0], k[1], int(sp.gid[j]), int(sp.depth[j]))
        for r in range(reports.shape[0]):
            rep = reports[r, j]
            if int(rep["has_eff"]):
                c = (int(rep["w0"]), int(rep["w1"]), int(rep["eff_gid"]), int(rep["eff_depth"]))
                best = c if best is None or c[:3] > best[:3] else best
            sub[j] = sub[j] or bool(int(rep["sublock"]))
        for c_ in range(n):
            if int(sp.parent[c_]) == j:
                if eff[c_] is not None and (best is None or eff[c_][:3] > best[:3]):
                    best = eff[c_]
                sub[j] = sub[j] or sub[c_]
        sub[j] = sub[j] or int(sp.gid[j]) in locked_gids
        eff[j] = best
    recs = []
    for j in range(n):
        if int(sp.parent[j]) < 0 or int(sp.tier[j]) != 0 or sub[j] or eff[j] is None:
            continue
        w0, w1, eg, ed = eff[j]
        recs.append((w0, w1, eg, int(sp.gid[j]), ed - int(sp.depth[j]), int(sp.len[j])))
    out = np.array(recs, dtype=CAND_DTYPE) if recs else np.zeros(0, dtype=CAND_DTYPE)
    return np.sort(out, order=["w0", "w1", "eff_gid", "d"])


# ---- partition of a global tree ----------------------------------------------------------
@dataclass
class Shard:
    rank: int
    soa: SoAArrays              # local tree (local ids, increasing in global id)
    gids: np.ndarray            # int32 [n_local] global id of each local node
    spine_local: np.ndarray     # int32 local ids of the spine copies, in Spine order
    wf_lo: int                  # owned WorkflowId block [wf_lo, wf_hi)
    wf_hi: int
    spine: Spine = field(repr=False, default=None)


def _depths(parent: np.ndarray) -> np.ndarray:
    """Depth of every node (root 0), by pointer doubling over the parent array."""
    n = parent.size
    par = parent.astype(np.int64).copy()
    par[0] = 0
    depth = (np.arange(n) != 0).astype(np.int64)  # one hop to the parent
    anc = par.copy()
    while True:
        more = anc != 0
        if not more.any():
            return depth
        depth = np.where(more, depth + depth[anc], depth)
        anc = np.where(more, anc[anc], 0)


def partition(soa: SoAArrays, n_ranks: int, spine_depth: int = 1, only: int | None = None) -> list[Shard]:
    """Splits a global tree into n_ranks shards.  Spine = nodes of depth <=
    spine_depth; the subtrees below it go to ranks in contiguous global-id
    blocks of roughly equal size.  Requires that every non-spine node is
    tagged only by workflows of its rank's WorkflowId block (workflows are
    co-located with their subtrees; true of the synthetic generator, whose
    group subtrees hold only that group's workflows).  Vectorised (8 M-node
    trees partition in seconds)."""
    n = soa.n_nodes
    parent = soa.parent.astype(np.int64)
    depth = soa.depth.astype(np.int64) if np.any(soa.depth[1:]) else _depths(parent)
    is_spine = depth <= spine_depth
    # subtree root (at spine_depth + 1) of every non-spine node, by doubling
    top = np.arange(n)
    up = parent.copy()
    up[0] = 0
    lift = np.where(depth > spine_depth + 1, depth - (spine_depth + 1), 0)
    bit = 0
    while np.any(lift >> bit):
        sel = ((lift >> bit) & 1).astype(bool)
        top = np.where(sel, up[top], top)
        up = up[up]
        bit += 1
    nz = np.nonzero(~is_spine)[0]
    roots, inv = np.unique(top[nz], return_inverse=True)
    sizes = np.bincount(inv, minlength=roots.size)
    cum = np.cumsum(sizes)
    total = int(cum[-1]) if cum.size else 0
    owner_of_root = np.minimum((cum - 1) * n_ranks // max(total, 1), n_ranks - 1)
    owner = np.full(n, -1, dtype=np.int64)
    owner[nz] = owner_of_root[inv]
    off = soa.acc_off.astype(np.int64)
    cnt = np.diff(off)
    E = int(off[-1])
    wfv = soa.acc_wf[:E].astype(np.int64)
    # WorkflowId range of each rank's non-spine entries
    tagged = nz[cnt[nz] > 0]
    first = wfv[off[tagged]] if tagged.size else np.zeros(0, np.int64)
    last = wfv[off[tagged + 1] - 1] if tagged.size else np.zeros(0, np.int64)
    INF = 1 << 62
    lo_r = np.full(n_ranks, INF, dtype=np.int64)
    hi_r = np.full(n_ranks, -INF, dtype=np.int64)
    np.minimum.at(lo_r, owner[tagged], first)
    np.maximum.at(hi_r, owner[tagged], last + 1)
    # block boundaries: rank r owns WorkflowIds in [bound[r], bound[r+1]) (the
    # whole id line is covered, so workflows tagged only on spine nodes count too)
    bound = [-INF] + [0] * (n_ranks - 1) + [INF]
    prev_hi = -INF
    for r in range(n_ranks):
        if r > 0:
            bound[r] = int(lo_r[r]) if lo_r[r] != INF else max(prev_hi, bound[r - 1])
            if bound[r] < prev_hi:
                raise ValueError("tree is not shardable by WorkflowId blocks (workflows span ranks)")
        if hi_r[r] != -INF:
            prev_hi = max(prev_hi, int(hi_r[r]))
    lo = np.array(bound[:-1], dtype=np.int64)
    hi = np.array(bound[1:], dtype=np.int64)
    node_of_entry = np.repeat(np.arange(n), cnt)
    spine_ids = np.nonzero(is_spine)[0]
    sp_index = np.full(n, -1, dtype=np.int64)
    sp_index[spine_ids] = np.arange(spine_ids.size)
    sp_par = np.where(parent[spine_ids] >= 0, sp_index[np.maximum(parent[spine_ids], 0)], -1)
    sp_par[spine_ids == 0] = -1
    spine = Spine(gid=spine_ids.astype(np.int64), parent=sp_par.astype(np.int64), depth=depth[spine_ids],
                  len=soa.len[spine_ids].astype(np.int64), tier=soa.tier[spine_ids].astype(np.int64),
                  retired=soa.retired[spine_ids].astype(np.int64), ever=soa.ever_tagged[spine_ids].astype(np.int64),
                  last=soa.last_access[spine_ids].astype(np.uint64), score=soa.score[spine_ids].astype(np.float64))
    shards = []
    for r in range(n_ranks):
        if only is not None and r != only:  # one rank's shard (every rank partitions the same tree)
            continue
        keep = np.nonzero(is_spine | (owner == r))[0]  # sorted global ids
        loc = np.full(n, -1, dtype=np.int64)
        loc[keep] = np.arange(keep.size)
        m = keep.size
        in_block = (wfv >= lo[r]) & (wfv < hi[r])
        en = node_of_entry
        bad = (owner[en] == r) & ~in_block
        if bad.any():
            raise ValueError("non-spine node tagged by another rank's workflow")
        ekeep = ((owner[en] == r) | (is_spine[en] & in_block))
        kcnt = np.bincount(en[ekeep], minlength=n)[keep]
        loc_soa = SoAArrays(m, int(kcnt.sum()), dict(soa.scalars))
        for f in SoAArrays.FIELDS:
            setattr(loc_soa, f, getattr(soa, f)[keep].copy())
        loc_soa.parent = np.where(keep == 0, -1, loc[np.maximum(parent[keep], 0)]).astype(np.int32)
        loc_soa.depth = depth[keep].astype(np.int32)
        loc_soa.acc_off = np.concatenate([[0], np.cumsum(kcnt)]).astype(np.int64)
        if loc_soa.n_entries:
            loc_soa.acc_wf = wfv[ekeep].astype(np.int64)
            loc_soa.acc_bits = soa.acc_bits[:E][ekeep].astype(np.uint64)
        shards.append(Shard(r, loc_soa, keep.astype(np.int32), loc[spine_ids].astype(np.int32), int(lo[r]),
                            int(hi[r]), spine))
    return shards


# ---- collectives -----------------------------------------------------------------------
def allgather_var(dist, t, world: int):
    """all_gather of a 1-D tensor whose length differs per rank: returns the
    padded [world, max_len] gather and the per-rank lengths."""
    import torch

    dev = t.device if dist.get_backend() == "nccl" else torch.device("cpu")
    n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    lens = [int(x.item()) for x in ns]
    mx = max(lens) if lens else 0
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    if t.numel():
        pad[: t.numel()] = t
    out = torch.zeros(world * mx, dtype=t.dtype, device=t.device)
    if mx:
        if t.is_cuda and dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(out, pad)
        else:  # gloo: host staging
            host = [torch.zeros(mx, dtype=t.dtype) for _ in range(world)]
            dist.all_gather(host, pad.cpu())
            out.copy_(torch.cat(host))
    return out.view(world, mx), lens


# per-step host wall of the distributed decision's stages (ms), when set to a
# dict (bench.py --sharded / PBKV_PROFILE_SHARD)
PROFILE = None


# ---- per-rank driver ------------------------------------------------------------------------
class ShardedPolicy:
    """A rank's view of a sharded tree: its pbkv context plus the collective
    exchange.  `dist` is torch.distributed (initialised by the caller) or None
    for a single process driving every shard itself (tests: logical shards on
    one GPU, exchange = concatenation)."""

    def __init__(self, shard: Shard, num_agents: int, k: int, gamma: float, device: int = 0):
        import torch

        from .api import Policy

        self.shard = shard
        self.pol = Policy(num_agents=num_agents, k=k, gamma=gamma, device=device)
        self.pol.mirror(shard.soa)
        g = np.ascontiguousarray(shard.gids, dtype=np.int32)
        sl = np.ascontiguousarray(shard.spine_local, dtype=np.int32)
        self.pol._c(_abi.lib().pbkv_shard_set(self.pol.handle, ptr(g, C.c_int32), ptr(sl if sl.size else None,
                                                                                     C.c_int32), int(sl.size)))
        self.dev = torch.device("cuda", device)
        n = shard.soa.n_nodes
        self.cand = torch.zeros(n * CAND_DTYPE.itemsize, dtype=torch.uint8, device=self.dev)
        self.spine_out = torch.zeros(max(1, shard.spine.n) * SPINE_DTYPE.itemsize, dtype=torch.uint8,
                                     device=self.dev)
        self.result = torch.zeros(3, dtype=torch.int64, device=self.dev)
        self.pmax = None  # max spine-product count over ranks (refreshed every decision)

    def order_after_torch(self) -> None:
        """The pbkv stream waits for torch's current stream (inputs built and
        outputs zero-filled there), with no host synchronisation."""
        import torch

        self.pol._c(_abi.lib().pbkv_ctx_wait_stream(self.pol.handle,
                                                      C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)))

    def locked_view(self, locked_gids):
        """(device tensor of this shard's local ids among `locked_gids`, their
        count, the locked spine gids) -- vectorised (sorted global ids,
        searchsorted), and cached for the same array object (a serving loop
        passing one locked array per decision pays this once per change)."""
        import torch

        c = getattr(self, "_lk_cache", None)
        if c is not None and c[0] is locked_gids:
            return c[1], c[2], c[3]
        g = np.asarray(locked_gids, dtype=np.int64).ravel()
        gids = self.shard.gids.astype(np.int64)
        pos = np.searchsorted(gids, g)
        ok = pos < gids.size
        ok[ok] = gids[pos[ok]] == g[ok]
        loc = np.unique(pos[ok]).astype(np.int32)
        ld = torch.from_numpy(loc if loc.size else np.zeros(1, np.int32)).to(self.dev)
        sp_gid = self.shard.spine.gid.astype(np.int64)
        sp_locked = set(int(x) for x in sp_gid[np.isin(sp_gid, g)]) if sp_gid.size else set()
        if isinstance(locked_gids, np.ndarray):
            self._lk_cache = (locked_gids, ld, int(loc.size), sp_locked)
        return ld, int(loc.size), sp_locked

    def local_ids(self, gids) -> np.ndarray:
        """Local ids of the given global ids that this shard holds."""
        g = np.asarray(sorted(set(int(x) for x in gids)), dtype=np.int64)
        pos = np.searchsorted(self.shard.gids, g)
        ok = (pos < self.shard.gids.size) & (self.shard.gids[np.minimum(pos, self.shard.gids.size - 1)] == g)
        return pos[ok].astype(np.int32)

    # -- step 1: local selection -----------------------------------------------------------
    def local_select(self, policy: int, score_mode: int, needed: int, locked_local_dev, n_locked: int,
                     want_count: bool = True):
        L = _abi.lib()
        self.order_after_torch()
        rc = L.pbkv_shard_select(self.pol.handle, int(policy), int(score_mode), int(needed),
                                 C.cast(C.c_void_p(locked_local_dev or None), C.POINTER(C.c_int32)), int(n_locked),
                                 C.cast(C.c_void_p(self.cand.data_ptr()), C.POINTER(CandC)),
                                 int(self.shard.soa.n_nodes),
                                 C.cast(C.c_void_p(self.spine_out.data_ptr()), C.POINTER(SpineInfoC)),
                                 C.cast(C.c_void_p(self.result.data_ptr()), C.POINTER(C.c_int64)))
        self.pol._c(rc)
        if not want_count:
            return None, self.spine_out[: self.shard.spine.n * SPINE_DTYPE.itemsize]
        n_cand = int(self.result[0].item())
        return self.cand[: n_cand * CAND_DTYPE.itemsize], self.spine_out[: self.shard.spine.n * SPINE_DTYPE.itemsize]

    # -- step 2: spine products (HE recompute) ------------------------------------------------
    def spine_products(self):
        import torch

        ns = self.shard.spine.n
        counts = np.zeros(max(ns, 1), dtype=np.int64)
        total = int(sum(int(self.shard.soa.acc_off[s + 1] - self.shard.soa.acc_off[s])
                        for s in self.shard.spine_local.tolist())) * self.pol.k
        out = torch.zeros(max(total, 1), dtype=torch.float64, device=self.dev)
        self.order_after_torch()
        self.pol._c(_abi.lib().pbkv_shard_spine_products(self.pol.handle, C.cast(C.c_void_p(out.data_ptr()),
                                                                                 C.POINTER(C.c_double)),
                                                         ptr(counts, C.c_int64)))
        return out[:total], counts[:ns]

    def chain_sums(self, x_dev, offsets: np.ndarray) -> np.ndarray:
        out = np.zeros(max(offsets.size - 1, 1), dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        self.order_after_torch()
        self.pol._c(_abi.lib().pbkv_chain_sum(self.pol.handle, C.cast(C.c_void_p(x_dev.data_ptr()),
                                                                      C.POINTER(C.c_double)),
                                              ptr(off, C.c_int64), int(off.size - 1), ptr(out, C.c_double)))
        return out[: offsets.size - 1]

    def interval_sums(self, x_ptr: int, pieces: np.ndarray, out_off: np.ndarray) -> np.ndarray:
        """pbkv_interval_sums: [n_out, 2] (sum, sum of magnitudes) of the
        double array at device address x_ptr over each output's pieces."""
        pc = np.ascontiguousarray(pieces, dtype=np.int64).reshape(-1)
        oo = np.ascontiguousarray(out_off, dtype=np.int64)
        n_out = int(oo.size - 1)
        out = np.zeros(max(2 * n_out, 1), dtype=np.float64)
        self.order_after_torch()
        self.pol._c(_abi.lib().pbkv_interval_sums(self.pol.handle, C.c_void_p(x_ptr), ptr(pc if pc.size else np.zeros(2, np.int64), C.c_int64),
                                                  ptr(oo, C.c_int64), n_out, ptr(out, C.c_double)))
        return out[: 2 * n_out].reshape(n_out, 2)

    def merge_cut(self, runs_dev, starts: list[int], lens: list[int], needed: int):
        import torch

        victims = torch.zeros(max(1, sum(lens)), dtype=torch.int32, device=self.dev)
        res = torch.zeros(3, dtype=torch.int64, device=self.dev)
        st = np.array(starts, dtype=np.int64)
        ln = np.array(lens, dtype=np.int64)
        self.order_after_torch()
        self.pol._c(_abi.lib().pbkv_merge_cut(self.pol.handle,
                                              C.cast(C.c_void_p(runs_dev.data_ptr()), C.POINTER(CandC)),
                                              ptr(st, C.c_int64), ptr(ln, C.c_int64), int(st.size), int(needed),
                                              C.cast(C.c_void_p(victims.data_ptr()), C.POINTER(C.c_int32)),
                                              C.cast(C.c_void_p(res.data_ptr()), C.POINTER(C.c_int64))))
        nv, freed, sf = (int(x) for x in res.tolist())
        return victims[:nv], freed, bool(sf)


def global_select(ranks: list[ShardedPolicy] | ShardedPolicy, policy: int, score_mode: int, needed: int,
                  locked_gids, dist=None, world: int = 1):
    """One sharded eviction decision: (victim global ids as an int32 array in
    eviction order, freed tokens, shortfall).  With dist=None, `ranks` is the list of
    every shard's ShardedPolicy in one process (logical shards); otherwise it
    is this rank's ShardedPolicy and the exchange goes through `dist`."""
    import torch

    if policy == POLICY_KVFLOW:
        raise ValueError("kvflow is not supported on a sharded tree")
    if dist is not None:
        return _global_select_dist(ranks if not isinstance(ranks, list) else ranks[0], policy, score_mode, needed,
                                   locked_gids, dist, world)
    local = ranks if isinstance(ranks, list) else [ranks]
    sp = local[0].shard.spine
    locked_set = set(int(x) for x in locked_gids)
    cands, reps, prods, pcounts = [], [], [], []
    for rp in local:
        g2l = {int(g): i for i, g in enumerate(rp.shard.gids.tolist())}
        loc = np.array([g2l[g] for g in locked_set if g in g2l], dtype=np.int32)
        ld = torch.from_numpy(loc if loc.size else np.zeros(1, np.int32)).to(rp.dev)
        c, r = rp.local_select(policy, score_mode, needed, ld.data_ptr(), loc.size)
        cands.append(c)
        reps.append(r)
        if policy == POLICY_HE and score_mode == SCORE_RECOMPUTE and sp.n:
            x, cnt = rp.spine_products()
            prods.append(x)
            pcounts.append(cnt)
    me = local[0]
    if dist is None:
        runs = cands
        rep_all = np.stack([np.frombuffer(r.cpu().numpy().tobytes(), dtype=SPINE_DTYPE) for r in reps]) \
            if sp.n else np.zeros((len(reps), 0), SPINE_DTYPE)
        prod_runs = prods
        cnt_all = pcounts
    else:
        g, lens = allgather_var(dist, cands[0], world)
        runs = [g[r, : lens[r]] for r in range(world)]
        rg, _ = allgather_var(dist, reps[0], world)
        rep_all = np.stack([np.frombuffer(rg[r].cpu().numpy().tobytes(), dtype=SPINE_DTYPE)[: sp.n]
                            for r in range(world)]) if sp.n else np.zeros((world, 0), SPINE_DTYPE)
        prod_runs, cnt_all = [], []
        if prods:
            pg, plens = allgather_var(dist, prods[0], world)
            cg, _ = allgather_var(dist, torch.from_numpy(pcounts[0]).to(me.dev), world)
            prod_runs = [pg[r, : plens[r]] for r in range(world)]
            cnt_all = [cg[r].cpu().numpy()[: sp.n] for r in range(world)]
    # spine scores: exact chains over all ranks' products in rank (= WorkflowId) order
    if prod_runs:
        pieces, offs = [], [0]
        for j in range(sp.n):
            for r in range(len(prod_runs)):
                base = int(np.sum(cnt_all[r][:j]))
                pieces.append(prod_runs[r][base: base + int(cnt_all[r][j])])
            offs.append(offs[-1] + sum(int(cnt_all[r][j]) for r in range(len(prod_runs))))
        x = torch.cat(pieces) if pieces else torch.zeros(1, dtype=torch.float64, device=me.dev)
        scores = me.chain_sums(x, np.array(offs, dtype=np.int64))
    else:
        scores = sp.score
    srec = spine_records(sp, rep_all, scores, policy, locked_set)
    allruns = [r for r in runs] + [torch.from_numpy(srec.view(np.uint8).copy()).to(me.dev)]
    lens = [int(r.numel() // CAND_DTYPE.itemsize) for r in allruns]
    starts = list(np.cumsum([0] + lens[:-1]))
    buf = torch.cat([r.reshape(-1) for r in allruns]) if sum(lens) else torch.zeros(CAND_DTYPE.itemsize,
                                                                                     dtype=torch.uint8,
                                                                                     device=me.dev)
    v, freed, sf = me.merge_cut(buf, [int(s) for s in starts], lens, needed)
    return v.cpu().numpy(), freed, sf


def _global_select_dist(rp: ShardedPolicy, policy: int, score_mode: int, needed: int, locked_gids, dist,
                        world: int):
    """The per-rank decision with two collectives: (1) one all-gather of a
    fixed-size header [candidate count | spine reports | spine product counts
    | spine products padded to the largest rank's], (2) one all-gather of the
    candidate records padded to the largest count.  Everything else is local."""
    import time

    import torch

    prof = PROFILE is not None
    t0 = time.perf_counter()
    marks = []

    def mark(what):
        if prof:
            marks.append((what, time.perf_counter()))

    sp = rp.shard.spine
    dev = rp.dev
    ld, n_loc, locked_set = rp.locked_view(locked_gids)  # spine gids among the locked: all spine_records needs
    _, rep = rp.local_select(policy, score_mode, needed, ld.data_ptr(), n_loc, want_count=False)
    mark("local_select")
    he_rc = policy == POLICY_HE and score_mode == SCORE_RECOMPUTE and sp.n > 0
    if he_rc:
        prod, pcnt = rp.spine_products()
        # the largest rank's product count, every decision (it moves with the
        # workflows tagging the spine; a stale maximum would desynchronise the
        # header sizes across ranks)
        t = torch.tensor([prod.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rp.pmax = int(t.item())
        pad = torch.zeros(rp.pmax, dtype=torch.float64, device=dev)
        pad[: prod.numel()] = prod
        pcnt_t = torch.from_numpy(np.ascontiguousarray(pcnt, dtype=np.int64)).to(dev)
    else:
        pad = torch.zeros(0, dtype=torch.float64, device=dev)
        pcnt_t = torch.zeros(sp.n, dtype=torch.int64, device=dev)
    head = torch.cat([rp.result[:1].view(torch.uint8), rep.reshape(-1), pcnt_t.view(torch.uint8),
                      pad.view(torch.uint8)])
    hdr = torch.empty(world * head.numel(), dtype=torch.uint8, device=dev)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(hdr, head)
    else:
        parts = [torch.zeros(head.numel(), dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, head.cpu())
        hdr.copy_(torch.cat(parts))
    mark("spine products + header all-gather")
    hdr = hdr.view(world, head.numel())
    nrep = sp.n * SPINE_DTYPE.itemsize
    meta = hdr[:, : 8 + nrep + 8 * sp.n].cpu().numpy()  # counts + reports + product counts (small)
    counts = meta[:, :8].copy().view(np.int64)[:, 0]
    rep_all = np.stack([np.frombuffer(meta[r, 8: 8 + nrep].tobytes(), dtype=SPINE_DTYPE) for r in range(world)]) \
        if sp.n else np.zeros((world, 0), SPINE_DTYPE)
    cnt_all = meta[:, 8 + nrep:].copy().view(np.int64) if sp.n else np.zeros((world, 0), np.int64)
    # (2) candidate records, padded to the largest count
    mx = int(counts.max()) if counts.size else 0
    rec = CAND_DTYPE.itemsize
    if mx:
        mine = torch.zeros(mx * rec, dtype=torch.uint8, device=dev)
        n_me = int(counts[rp.shard.rank])
        mine[: n_me * rec] = rp.cand[: n_me * rec]
        allc = torch.empty(world * mx * rec, dtype=torch.uint8, device=dev)
        if dist.get_backend() == "nccl":
            dist.all_gather_into_tensor(allc, mine)
        else:
            parts = [torch.zeros(mx * rec, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, mine.cpu())
            allc.copy_(torch.cat(parts))
    else:
        allc = torch.zeros(rec, dtype=torch.uint8, device=dev)
    mark("header readback + records all-gather")
    starts = [r * mx for r in range(world)] + [world * mx]
    n_cand = int(counts.sum())

    def cut_with(srec):
        lens = [int(c) for c in counts] + [int(srec.size)]
        buf = torch.cat([allc[: world * mx * rec] if mx else allc[:0],
                         torch.from_numpy(srec.view(np.uint8).copy()).to(dev)])
        if buf.numel() == 0:
            buf = torch.zeros(rec, dtype=torch.uint8, device=dev)
        return rp.merge_cut(buf, starts, lens, needed)

    if not he_rc:
        v, freed, sf = cut_with(spine_records(sp, rep_all, sp.score, policy, locked_set))
        return v.cpu().numpy(), freed, sf
    # spine scores over every rank's products, rank (= WorkflowId) order:
    # spine node j's products are rank r's piece [b_rj, b_rj + cnt_all[r, j])
    # of its header row (in doubles from the header's base address)
    row = head.numel()
    pstart = 8 + nrep + 8 * sp.n
    assert row % 8 == 0 and pstart % 8 == 0
    bj = np.concatenate([np.zeros((world, 1), np.int64), np.cumsum(cnt_all, axis=1)], axis=1) if sp.n else None
    pieces = np.array([[(r * row + pstart) // 8 + int(bj[r, j]), (r * row + pstart) // 8 + int(bj[r, j + 1])]
                       for j in range(sp.n) for r in range(world)], dtype=np.int64).reshape(-1, 2)
    offs = [0]
    for j in range(sp.n):
        offs.append(offs[-1] + int(cnt_all[:, j].sum()))
    mark("spine products gathered")
    # fast path: the exact serial chain E and any-order sum A
    # both lie within L * ulp(sum|x|) / 2 of the real sum.  If the spine
    # records are after every candidate record for both ends of the interval,
    # and the cut ends inside the candidates, the exact chains are not needed.
    # any-order sums per spine node on the device (pbkv_interval_sums), one
    # synchronisation
    sums = rp.interval_sums(hdr.data_ptr(), pieces, np.arange(0, world * sp.n + 1, world, dtype=np.int64)) \
        if sp.n else np.zeros((0, 2))
    A = sums[:, 0].copy()
    Sa = sums[:, 1].copy()
    mark("spine interval sums")
    L = np.diff(offs).astype(np.float64)
    B = np.array([2.0 * L[j] * np.ldexp(1.0, np.frexp(Sa[j])[1] - 53) if Sa[j] > 0 else 0.0 for j in range(sp.n)])
    lo = spine_records(sp, rep_all, A - B, policy, locked_set)
    hi = spine_records(sp, rep_all, A + B, policy, locked_set)
    fast = np.isfinite(A).all() and lo.size == hi.size and np.array_equal(lo["gid"], hi["gid"])
    mark("spine records (interval ends)")
    if fast and n_cand and lo.size:
        # the last record of every rank's run (only those come to the host)
        rr = [r for r in range(world) if counts[r] > 0]
        idx = torch.tensor([(r * mx + int(counts[r]) - 1) * rec + b for r in rr for b in range(rec)],
                           dtype=torch.int64, device=dev)
        last = np.frombuffer(allc[idx].cpu().numpy().tobytes(), dtype=CAND_DTYPE)
        maxrec = max(tuple(q[f] for f in ("w0", "w1", "eff_gid", "d")) for q in last)
        fast = all(tuple(int(v) for v in (q["w0"], q["w1"], q["eff_gid"], q["d"])) > maxrec for q in lo)
    mark("spine interval check")
    if fast:
        v, freed, sf = cut_with(lo)
        if int(v.numel()) <= n_cand and not sf:
            out = v.cpu().numpy()
            mark("merge + cut")
            if prof:
                prev = t0
                for what, t in marks:
                    PROFILE.setdefault(what, []).append(1e3 * (t - prev))
                    prev = t
            return out, freed, sf
    # exact chains (the interval could not place the spine): the products in
    # rank order, then one serial chain per spine node
    prods = hdr[:, pstart:].reshape(world, -1).view(torch.float64)
    parts = [prods[r, int(bj[r, j]): int(bj[r, j + 1])] for j in range(sp.n) for r in range(world)]
    x = torch.cat(parts) if parts else torch.zeros(1, dtype=torch.float64, device=dev)
    scores = rp.chain_sums(x, np.array(offs, dtype=np.int64))
    v, freed, sf = cut_with(spine_records(sp, rep_all, scores, policy, locked_set))
    return v.cpu().numpy(), freed, sf
