#!/usr/bin/env python
"""Benchmark of the PBKV decision hot path on B200 (BASELINE.json metric:
"cache nodes scored+ranked/sec and p99 eviction-decision latency").

One step = one eviction decision over the whole tree, resident in HBM:
Eq. 2 recomputed for every node from the resident forecasts (stage 2), the
hierarchical candidate keys, locked-subtree marks and subtree-max reduction,
and the token-weighted cut + victim order (stage 3) -- pbkv_select_dev in
PBKV_SCORE_RECOMPUTE mode.  Workload (configs[2]): 1M-node radix tree x 4096
workflows x K=8, 30% retired, A=16, need = 1% of device tokens, 1% of leaves
pinned.  `value` = nodes scored+ranked per second (all
ranks); `e2e` = the same through the host C ABI (forecast upload from pinned
host memory + pbkv_select with host locked list and host victim output).

--impl reference times the reference's own CPU policy code (oracle/_ref,
compiled from /root/reference) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

import numpy as np  # noqa: E402

METRIC = "cache nodes scored+ranked/sec and p99 eviction-decision latency"
CONFIGS = {
    # name: (n_nodes, n_workflows, K)
    "c2": (10_000, 256, 4),
    "c3": (1_000_000, 4096, 8),
    "c4": (8_000_000, 16384, 8),  # config 4: one GPU, or strong-scaled over N ranks (run_sharded)
}
AGENTS = 16
GAMMA = 0.7


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--needed-frac", type=float, default=0.01)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-decisions", type=int, default=2)
    ap.add_argument("--no-pipeline", action="store_true", help="skip the config-2 predictor pipeline line")
    ap.add_argument("--no-sweep", action="store_true", help="skip the need sweep (0.1/1/10/50%%) and --no-defer line")
    ap.add_argument("--no-prefetch", action="store_true", help="skip the stage-4 prefetch plan object")
    ap.add_argument("--sharded", action="store_true",
                    help="the sharded config-4 path even with one rank (measures its exchange overhead)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload(cfg: str, rank: int):
    """Synthetic tree + forecasts + pinned set, deterministic per (config, rank)."""
    import workloads as WL
    from paper_2605_06472_b200.api import HostTree

    n_nodes, n_wf, K = CONFIGS[cfg]
    t = HostTree()
    t0 = time.perf_counter()
    t.synth(n_nodes=n_nodes, n_workflows=n_wf, agents=AGENTS, seed=12345 + rank)
    build_s = time.perf_counter() - t0
    soa = t.export()
    rng = np.random.default_rng(12345 + rank)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, K, AGENTS + 1)
    locked = np.array(WL.pinned_paths(soa, rng, 0.01), dtype=np.int32)
    return t, soa, wf, P, locked, K, build_s


def churn_batch(rng, t, live: list[int], victims: np.ndarray, n_wf: int, n_insert: int = 16, n_match: int = 8,
                n_demote: int = 64):
    """One serving-loop batch of tree mutations between two decisions, in the
    synthetic generator's token namespaces (csrc/host/ops.hpp): the previous
    decision's first victims demoted (in eviction order each is a device
    leaf), then inserts and matches of live workflows along their own
    shared + group + private paths, then one termination.  Returns the op
    stream and the workflows whose state changed (the ones the simulator's
    refresh_workflow re-forecasts, simulator.hpp:430-435)."""
    from paper_2605_06472_b200.ops import OpStream

    ops = OpStream()
    touched = []
    for v in victims[:n_demote].tolist():
        ops.demote(int(v))
    for j in range(n_insert + n_match):
        w = int(live[int(rng.integers(len(live)))])
        touched.append(w)
        toks = [(1 << 60) | i for i in range(32)] + [(2 << 60) | ((w // 16) << 20) | i for i in range(8)]
        toks.append((3 << 60) | w)
        toks += [int(x) for x in rng.integers(0, 4, size=int(rng.integers(1, 11)))]
        agent = int(rng.integers(AGENTS))
        if j < n_insert:
            ops.insert(toks, w, agent)
        else:
            ops.match(toks, w, agent)
    if len(live) > 1:
        w = live.pop(int(rng.integers(len(live))))
        ops.terminate(w)
        touched.append(w)
    return ops, sorted(set(touched))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        self.result = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                       "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_decisions(cfg: str, needed_frac: float, decisions: int, rank: int = 0,
                            plan_bandwidth: int | None = None, round_probe=None):
    """The reference policy code (oracle/_ref) on the same workload: per
    decision, refresh every node's score (refresh_nodes, scoring.hpp:95) and
    select_victims_hierarchical (policies.hpp:108)."""
    import workloads as WL
    from oracle import RefTree, have_ref
    from paper_2605_06472_b200._abi import POLICY_HE

    if not have_ref():
        return None
    n_nodes, n_wf, K = CONFIGS[cfg]
    t = RefTree()
    t0 = time.perf_counter()
    t.synth(n_nodes=n_nodes, n_workflows=n_wf, agents=AGENTS, seed=12345 + rank)
    build_s = time.perf_counter() - t0
    soa = t.export()
    rng = np.random.default_rng(12345 + rank)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, K, AGENTS + 1)
    locked = WL.pinned_paths(soa, rng, 0.01)
    t.set_forecasts(wf, P)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = max(1, int(needed_frac * used))
    times = []
    for _ in range(decisions):
        t0 = time.perf_counter()
        t.refresh_nodes(None, K, GAMMA)
        sel = t.select(POLICY_HE, needed, locked)
        times.append(time.perf_counter() - t0)
    out = {"n_nodes": soa.n_nodes, "times": times, "build_s": build_s, "n_victims": len(sel.victims)}
    if plan_bandwidth is not None:  # plan_conservative_prefetch (policies.hpp:220) on the same tree
        pt = []
        for _ in range(max(1, decisions)):
            t0 = time.perf_counter()
            pl = t.plan(plan_bandwidth)
            pt.append(time.perf_counter() - t0)
        out["plan_times"] = pt
        out["plan_selected"] = list(pl.selected)
        out["plan_candidates"] = [c[0] for c in pl.candidates]
    if round_probe is not None and round_probe[0] is not None:
        # one candidate step of the reference prefetch round: HE selection of
        # the candidate's length under the ancestry locks of every candidate
        first, sel_ids = round_probe
        par = soa.parent
        locked = set()
        for s in sel_ids.tolist():
            v = int(par[s])
            while v > 0:
                locked.add(v)
                v = int(par[v])
        t0 = time.perf_counter()
        t.select(POLICY_HE, max(1, int(soa.len[first])), sorted(locked))
        out["round_candidate_s"] = time.perf_counter() - t0
    return out


def reference_threads() -> int:
    """Host threads for the reference arm: every core, capped so that one
    C3 tree per thread (~0.5 GB resident) fits comfortably."""
    n = os.cpu_count() or 1
    try:
        import psutil

        n = min(n, max(1, int(psutil.virtual_memory().available // (1 << 30)) // 2))
    except Exception:
        pass
    return max(1, min(n, int(os.environ.get("PBKV_REF_THREADS", "32"))))


def run_reference(args, rank, world):
    """The reference's own CPU policy code (oracle/_ref, the unmodified
    headers) on the same workload.  The reference is single-threaded per
    decision; its scenario runner parallelises independent
    simulations over a thread pool (scenario.hpp:291-301), so the arm runs
    one independent decision stream per host thread, each on its own tree,
    and reports the aggregate nodes/s."""
    if rank != 0:
        return
    import threading

    n_nodes, n_wf, K = CONFIGS[args.config]
    steps = max(1, args.steps)
    warm = max(0, min(args.warmup, 1))
    T = reference_threads()
    results = [None] * T

    def worker(i):
        results[i] = cpu_reference_decisions(args.config, args.needed_frac, warm + steps)

    # one stream alone first, then T concurrent streams; the arm reports the
    # better aggregate (the reference's allocator-heavy maps can scale badly)
    single = cpu_reference_decisions(args.config, args.needed_frac, warm + steps)
    if single is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libflowkv_ref.so not built"}))
        return
    th = [threading.Thread(target=worker, args=(i,)) for i in range(T)] if T > 1 else []
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    one = single["n_nodes"] / statistics.mean(single["times"][warm:])
    many = 0.0
    if T > 1 and all(r is not None for r in results):
        many = sum(rr["n_nodes"] / statistics.mean(rr["times"][warm:]) for rr in results)
    if many > one:
        val, times = many, [x for rr in results for x in rr["times"][warm:]]
    else:
        val, times, T = one, single["times"][warm:], 1
    r = single
    ms = 1000.0 * statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "nodes/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n_nodes} nodes x {n_wf} workflows x K={K}, 30% retired, "
                               f"HE select at {args.needed_frac:.2%} need",
                   "parallelism": f"cpu x{T} threads (independent decision streams)"},
        "p99_decision_ms": 1000.0 * float(np.percentile(times, 99)),
        "cpu_baseline": {"value": val, "unit": "nodes/s", "cores": T, "kind": "reference",
                         "sample": f"{T} threads x {steps} decisions (refresh_nodes over all nodes + "
                                   f"select_victims_hierarchical), one tree per thread; single-thread mean "
                                   f"{ms:.1f} ms/decision; wall {wall:.1f} s"},
        "e2e": {"value": val, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def pipeline_c2(torch, dev, reps: int = 20):
    """configs[1]: 10K-node tree x 256 workflows x K=4 -- stage 1 (the
    predictor forward from prefill hidden states resident in HBM, H = 5120)
    + stage 2 + stage 3 end to end, one decision per step; also the stage-1
    forward alone at the config-3 batch (4096 workflows, K = 8)."""
    import workloads as WL
    from paper_2605_06472_b200._abi import POLICY_HE, SCORE_RECOMPUTE
    from paper_2605_06472_b200.api import HostTree, Policy
    from paper_2605_06472_b200.predictor import PredictorWeights, random_inputs

    out = {}
    for name, (n_nodes, n_wf, K) in (("c2", CONFIGS["c2"]), ("c3_predict", CONFIGS["c3"])):
        t = HostTree()
        t.synth(n_nodes=n_nodes, n_workflows=n_wf, agents=AGENTS, seed=777)
        soa = t.export()
        wf = np.array(WL.workflows_of(soa), dtype=np.int64)
        H = 5120
        w = PredictorWeights.random(num_agents=AGENTS, horizon=K, text_dim=H)
        off, pre, x = random_inputs(wf.size, AGENTS, H, max_prefix=64)
        pol = Policy(num_agents=AGENTS, k=K, gamma=GAMMA)
        pol.mirror(t)
        pol.load_predictor(w, max_prefix=64)
        xd = torch.from_numpy(x.view(np.int16)).to(dev)
        used = int(soa.len[soa.tier == 0][1:].sum())
        needed = max(1, used // 100)
        locked_d = torch.zeros(1, dtype=torch.int32, device=dev)
        victims_d = torch.empty(soa.n_nodes, dtype=torch.int32, device=dev)
        res_d = torch.zeros(3, dtype=torch.int64, device=dev)
        stream = torch.cuda.ExternalStream(pol.stream_handle(), device=dev)

        def run(decide):
            pol.predict(wf, off, pre, None, x_device_ptr=xd.data_ptr(), want_probs=False)
            if decide:
                pol.select_dev(POLICY_HE, SCORE_RECOMPUTE, needed, locked_d.data_ptr(), 0, victims_d.data_ptr(),
                               soa.n_nodes, res_d.data_ptr())

        decide = name == "c2"
        for _ in range(3):
            run(decide)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(decide)
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name] = {"nodes": soa.n_nodes, "workflows": int(wf.size), "K": K, "H": H,
                     "ms_mean": statistics.mean(ts), "ms_p99": float(np.percentile(ts, 99)),
                     "what": "predict + score + select (device-resident x)" if decide else "predict only"}
    return out


def shard_workload(cfg: str, rank: int, world: int):
    """Strong scaling of config 4: every rank generates the same global
    8 M-node x 16 K-workflow tree (deterministic synthetic generator), the
    tree is partitioned by subtree into `world` node-set shards (spine = the
    root and the shared prefix, replicated; workflows co-located with their
    group subtrees: contiguous WorkflowId blocks), and the rank keeps its own
    shard resident.  Forecasts: the rank's own workflows."""
    import workloads as WL
    from paper_2605_06472_b200 import shard as SH
    from paper_2605_06472_b200.api import HostTree

    n_nodes, n_wf, K = CONFIGS[cfg]
    t = HostTree()
    t0 = time.perf_counter()
    t.synth(n_nodes=n_nodes, n_workflows=n_wf, agents=AGENTS, seed=4)
    soa = t.export()
    del t
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(4)
    wf = np.array(WL.workflows_of(soa), dtype=np.int64)
    P = WL.random_forecasts(rng, wf.size, K, AGENTS + 1)
    locked = np.array(WL.pinned_paths(soa, rng, 0.01), dtype=np.int64)
    used = int(soa.len[soa.tier == 0][1:].sum())
    shard = SH.partition(soa, world, only=rank)[0]
    mine = (wf >= shard.wf_lo) & (wf < shard.wf_hi)
    return shard, wf[mine], P[mine], locked, K, used, soa.n_nodes, build_s


def run_sharded(args, rank, world, local, dist, torch):
    """config 4, strong scaling: one eviction decision over the whole 8 M-node
    tree per step, its node set sharded over the ranks (local score + select,
    spine products and records exchanged with two NCCL all-gathers, exact
    spine chains or their interval placement, merge + cut); max over ranks of
    the device-event time.  e2e: the same decision through the public sharded
    API with every rank's forecasts uploaded from host memory and the victim
    list returned to the host."""
    from paper_2605_06472_b200 import shard as SH
    from paper_2605_06472_b200._abi import POLICY_HE, SCORE_RECOMPUTE

    cfg = "c4" if args.config == "c3" else args.config
    dev = torch.device("cuda", local)
    shard, wf, P, locked, K, used, n_global, build_s = shard_workload(cfg, rank, world)
    sp = SH.ShardedPolicy(shard, num_agents=AGENTS, k=K, gamma=GAMMA, device=local)
    sp.pol.put_forecasts(wf, P)
    needed = max(1, int(args.needed_frac * used))
    lk = np.ascontiguousarray(locked, dtype=np.int64)  # the decision's locked set (global ids)

    def step():
        return SH.global_select(sp, POLICY_HE, SCORE_RECOMPUTE, needed, lk, dist=dist, world=world)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if os.environ.get("PBKV_PROFILE_SHARD"):
        SH.PROFILE = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    k0, _ = sp.pol.launches()
    times = []
    dist.barrier()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            res = step()
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    dist.barrier()
    k1, _ = sp.pol.launches()
    stage_ms = {k: statistics.mean(v) for k, v in SH.PROFILE.items()} if SH.PROFILE else None
    SH.PROFILE = None
    # e2e: forecasts from (pageable) host memory + the decision, host wall
    e2e = []
    for _ in range(max(3, min(10, args.steps))):
        flush.fill_(1)
        torch.cuda.synchronize()
        dist.barrier()
        w0 = time.perf_counter()
        sp.pol.put_forecasts(wf, P)
        res = step()
        e2e.append(1e3 * (time.perf_counter() - w0))
    dist.barrier()
    tt = torch.tensor([statistics.mean(times), float(np.percentile(times, 99)), statistics.mean(e2e)],
                      dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms, p99, e2e_ms = tt.tolist()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the reference on one host core: C3 per-node rate (a C4 decision is ~8 s)
        r = cpu_reference_decisions("c3", args.needed_frac, 1)
        if r:
            cpu = {"value": r["n_nodes"] / statistics.mean(r["times"]), "unit": "nodes/s", "cores": 1,
                   "kind": "reference",
                   "sample": f"1 decision on the c3 tree (refresh_nodes all + select_victims_hierarchical), "
                             f"{statistics.mean(r['times']):.3f} s; the reference is single-threaded per decision"}
    if rank == 0:
        n_nodes, n_wf, _ = CONFIGS[cfg]
        line = {
            "metric": METRIC, "value": n_global / (ms * 1e-3), "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config 4: {n_nodes} nodes x {n_wf} workflows x K={K} sharded by subtree over "
                                   f"{world} GPUs, HE select at {args.needed_frac:.2%} of global need",
                       "n_nodes": n_global, "needed_tokens": needed, "n_victims": len(res[0]),
                       "l2": "flushed between steps (256 MiB write)", "parallelism": f"node-set shards x{world}"},
            "p99_decision_ms": p99, "gpu_launches": int(k1 - k0), "clocks": clk.result,
            "cpu_baseline": cpu,
            "e2e": {"value": n_global / (e2e_ms * 1e-3), "unit": "nodes/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(P.nbytes + 8 * wf.size), "d2h_bytes_per_step": int(4 * len(res[0]) + 24),
                    "what": "per rank: forecasts from host memory + the sharded decision (victims to the host); "
                            "max over ranks of the host wall"},
            "tree_build_s": build_s,
            "stage_host_ms": stage_ms,
            "defer": dict(zip(("fast", "exact"), sp.pol.defer_stats())),
        }
        print(json.dumps(line))
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if "PBKV_FORCE_DEVICE" in os.environ:  # testing: several ranks sharing one GPU (with PBKV_DIST_BACKEND=gloo)
        local = int(os.environ["PBKV_FORCE_DEVICE"])
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch

    from paper_2605_06472_b200._abi import POLICY_HE, SCORE_RECOMPUTE
    from paper_2605_06472_b200.api import Policy

    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.sharded:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        backend = os.environ.get("PBKV_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU (testing)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        run_sharded(args, rank, world, local, dist, torch)
        return

    n_nodes, n_wf, K = CONFIGS[args.config]
    t, soa, wf, P, locked, K, build_s = workload(args.config, rank)
    used = int(soa.len[soa.tier == 0][1:].sum())
    needed = max(1, int(args.needed_frac * used))

    pol = Policy(num_agents=AGENTS, k=K, gamma=GAMMA, device=local)
    pol.mirror(t)
    pol.put_forecasts(wf, P)

    dev = torch.device("cuda", local)
    locked_d = torch.from_numpy(locked if locked.size else np.zeros(1, np.int32)).to(dev)
    victims_d = torch.empty(soa.n_nodes, dtype=torch.int32, device=dev)
    result_d = torch.zeros(3, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.ExternalStream(pol.stream_handle(), device=dev)

    def step():
        pol.select_dev(POLICY_HE, SCORE_RECOMPUTE, needed, locked_d.data_ptr(), locked.size, victims_d.data_ptr(),
                       soa.n_nodes, result_d.data_ptr())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region ---------------------------------------------
    k0, l0 = pol.launches()
    per_step = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # evict the working set from L2 between decisions
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            per_step.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    k1, l1 = pol.launches()
    ms_local = statistics.mean(per_step)
    p99_local = float(np.percentile(per_step, 99))
    res = result_d.cpu().tolist()

    # ---- per-stage split (separate pass: events between stages) ---------------------
    pol.set_timing(True)
    stage = np.zeros(5)
    kern = np.zeros(2)
    n_stage = max(3, min(10, args.steps))
    for _ in range(n_stage):
        flush.fill_(1)
        torch.cuda.synchronize()
        step()
        stage += np.array(pol.timings())
        kern += np.array(pol.kernel_timings())
    stage /= n_stage
    kern /= n_stage
    select_phases = [round(x, 2) for x in pol.phase_times_us()]
    pol.set_timing(False)

    # ---- need sweep (0.1 / 1 / 10 / 50% of device tokens) -----------
    # 50% reaches deep into the active-by-score region; lib_calls counts any
    # library (CUB) fallback sort inside those decisions.  --no-defer: the same
    # 1% decision with every heavy node's exact Eq. 2 chain computed inside
    # the timed step (no interval placement).
    sweep = {}
    reps = max(3, min(10, args.steps))

    def timed(fn, n):
        out = []
        for _ in range(n):
            flush.fill_(1)
            torch.cuda.synchronize()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            fn()
            a1.record(stream)
            a1.synchronize()
            out.append(a0.elapsed_time(a1))
        return out

    if not args.no_sweep:
        for frac in (0.001, 0.01, 0.1, 0.5):
            nd = max(1, int(frac * used))

            def dec(nd=nd):
                pol.select_dev(POLICY_HE, SCORE_RECOMPUTE, nd, locked_d.data_ptr(), locked.size,
                               victims_d.data_ptr(), soa.n_nodes, result_d.data_ptr())

            dec()
            q0, ql0 = pol.launches()
            f0 = pol.defer_stats()
            ts = timed(dec, reps)
            q1, ql1 = pol.launches()
            f1 = pol.defer_stats()
            rr = result_d.cpu().tolist()
            sweep[f"{frac:.3%}"] = {"needed_tokens": nd, "n_victims": rr[0], "ms_mean": statistics.mean(ts),
                                    "ms_p99": float(np.percentile(ts, 99)),
                                    "nodes_per_s": soa.n_nodes / (statistics.mean(ts) * 1e-3),
                                    "gpu_launches_per_step": (q1 - q0) / reps, "lib_calls": int(ql1 - ql0),
                                    "defer_fast_exact": [f1[0] - f0[0], f1[1] - f0[1]]}
        pol.set_defer(False)
        step()
        ts = timed(step, reps)
        pol.set_defer(True)
        sweep["1.000%_no_defer"] = {"needed_tokens": needed, "ms_mean": statistics.mean(ts),
                                    "ms_p99": float(np.percentile(ts, 99)),
                                    "what": "every heavy node's exact Eq. 2 chain inside the step"}

    # ---- stage 4: conservative prefetch plan (policies.hpp:220) ----------------------
    prefetch = None
    if not args.no_prefetch:
        host = (soa.tier == 1)
        host[0] = False
        par_dev = np.zeros_like(host)
        par_dev[1:] = soa.tier[soa.parent[1:]] == 0
        hc = host & par_dev
        n_host_c = int(hc.sum())
        e_host = int((soa.acc_off[1:] - soa.acc_off[:-1])[hc].sum())
        bw = max(1, used // 50)
        pol.plan_conservative_prefetch(bw)
        pol.set_timing(True)
        pk, pw = [], []
        for _ in range(reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            plan = pol.plan_conservative_prefetch(bw)
            pw.append(1e3 * (time.perf_counter() - w0))
            pk.append(pol.kernel_timings()[1])
        pol.set_timing(False)
        # algorithmic bytes of one plan (SURVEY.md §8(d) stage 4): the tier
        # byte of every node; per host candidate node its parent id + parent
        # tier, entry range and len; 12 B per entry; its forecast rows' step-0
        # column; the sorted candidates written (id 4 + value 8)
        alg_pf = soa.n_nodes + n_host_c * (4 + 1 + 8 + 4) + 12 * e_host + wf.size * (AGENTS + 1) * 8 \
            + 12 * len(plan.candidates)
        pk_ms = statistics.mean(pk)
        prefetch = {
            "what": f"plan_conservative_prefetch, bandwidth {bw} tokens (2% of device tokens), {args.config} tree "
                    f"({n_host_c} host nodes under device parents)",
            "n_candidates": len(plan.candidates), "n_selected": len(plan.selected),
            "selected_tokens": plan.selected_tokens,
            "kernel_ms": pk_ms, "kernel_p99_ms": float(np.percentile(pk, 99)),
            "e2e": {"ms_mean": statistics.mean(pw), "ms_p99": float(np.percentile(pw, 99)),
                    "what": "host wall of the public call: kernel + one synchronisation + the plan copied from "
                            "pinned memory into the caller's arrays", "h2d_bytes": 48,
                    "d2h_bytes": 12 * len(plan.candidates) + 4 * len(plan.selected) + 32},
            "roofline": {"bound": "hbm", "kernel": "prefetch_plan_kernel", "achieved": alg_pf / (pk_ms * 1e-3) / 1e9,
                         "peak": float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0))
                         if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0,
                         "unit": "GB/s", "alg_bytes_per_launch": alg_pf},
            "lib_calls": 0,
        }
        prefetch["roofline"]["frac"] = prefetch["roofline"]["achieved"] / prefetch["roofline"]["peak"]
        prefetch["_plan"] = plan
        # the round that applies the plan (simulator.hpp:632-681) with the
        # device full (device_free = 0: every candidate needs victims), fused
        # into one hierarchical decision + the retired-prefix scan
        sel_ids = plan.selected_ids
        pol.prefetch_round(sel_ids, 0)
        rw = []
        for _ in range(reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            prom, vics = pol.prefetch_round(sel_ids, 0)
            rw.append(1e3 * (time.perf_counter() - w0))
        prefetch["round"] = {
            "what": "pbkv_prefetch_round over the plan's selected candidates with device_free = 0 (host wall of "
                    "the public call: one hierarchical decision + the per-candidate retired-prefix scan)",
            "candidates": int(sel_ids.size), "promoted": int(sum(prom)), "victims": int(vics.flat.size),
            "ms_mean": statistics.mean(rw), "ms_p99": float(np.percentile(rw, 99))}
        prefetch["_round_first"] = (int(sel_ids[0]) if sel_ids.size else None, sel_ids)

    # ---- e2e through the host C ABI, with the tree changing between decisions ----------
    # Before every decision the host tree (the reference CacheTree, tracked)
    # takes a serving-loop batch of mutations (churn_batch: inserts of live
    # workflows, a termination, the previous decision's first victims
    # demoted); the timed call then uploads only the changed nodes
    # (pbkv_mirror_sync -> pbkv_mirror_delta), re-puts the forecasts of the
    # workflows the batch touched (the simulator's refresh_workflow,
    # simulator.hpp:430-435, fresh rows from ordinary pageable host memory)
    # and drops the terminated one's (simulator.hpp:617), and takes the
    # decision with a host locked list and host victim output.
    import workloads as WL

    rng_e2e = np.random.default_rng(4242)
    live = [int(w) for w in wf.tolist() if w >= int(0.3 * n_wf)]
    row_of = {int(w): i for i, w in enumerate(wf.tolist())}
    P = P.copy()  # refreshed rows are written into the host forecast table
    pol.sync(t)  # the tracked tree's first sync is a full upload
    e2e_ms = []
    e2e_wall = []
    delta_nodes = []
    delta_fc = []
    n_victims_e2e = 0
    last_victims = np.zeros(0, dtype=np.int32)
    dropped = []
    for it in range(args.warmup + max(1, args.steps)):
        ops, touched = churn_batch(rng_e2e, t, live, last_victims, n_wf)
        t.apply_ops(ops.words)
        ids = t.log(pos_prev)[1] if it else None
        live_set = set(live)
        gone = [w for w in touched if w not in live_set]
        fresh = [w for w in touched if w in live_set]
        rows = np.array([row_of[w] for w in fresh], dtype=np.int64)
        P[rows] = WL.random_forecasts(rng_e2e, rows.size, K, AGENTS + 1)
        wf_d = wf[rows]
        P_d = np.ascontiguousarray(P[rows])
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        tw0 = time.perf_counter()
        e0.record(stream)
        pol.sync(t)
        tw1 = time.perf_counter()
        if gone:
            pol.drop_forecasts(gone)
        pol.put_forecasts(wf_d, P_d, validate_now=False)  # validated on the device, raised by the select
        tw2 = time.perf_counter()
        sel = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
        e1.record(stream)
        e1.synchronize()
        tw3 = time.perf_counter()
        pos_prev = t.log_end()
        last_victims = sel.victim_ids
        if it >= args.warmup:
            e2e_wall.append((tw1 - tw0, tw2 - tw1, tw3 - tw2))
            e2e_ms.append(max(e0.elapsed_time(e1), 1e3 * (tw3 - tw0)))
            delta_nodes.append(len(ids) if ids is not None else 0)
            delta_fc.append(int(P_d.nbytes + wf_d.nbytes + 8 * len(gone)))
        dropped += gone
        n_victims_e2e = len(sel)
    # the same decision when every forecast is re-put (host wall of the upload alone)
    keep = np.array([i for i, w in enumerate(wf.tolist()) if w not in set(dropped)], dtype=np.int64)
    wf_all, P_all = wf[keep], np.ascontiguousarray(P[keep])
    put_all = []
    for _ in range(5):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        pol.put_forecasts(wf_all, P_all)
        torch.cuda.synchronize()
        put_all.append(1e3 * (time.perf_counter() - w0))
    # the last e2e decision, checked against a fresh device-resident decision
    # on a full re-mirror of the same tree (victim ids in order)
    pol_chk = Policy(num_agents=AGENTS, k=K, gamma=GAMMA, device=local)
    pol_chk.mirror(t.export())
    pol_chk.put_forecasts(wf_all, P_all)
    chk = pol_chk.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    assert np.array_equal(chk.victim_ids, sel.victim_ids) and chk.freed == sel.freed, \
        "e2e decision (incremental mirror) differs from a full re-mirror"
    mirror_ok = pol.verify(t) == -1
    pol_chk.close()

    # ---- aggregate over ranks (max time) --------------------------------------------
    ms = ms_local
    p99 = p99_local
    e2e = statistics.mean(e2e_ms)
    if dist:
        tt = torch.tensor([ms_local, p99_local, e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, p99, e2e = tt.tolist()
    total_nodes = soa.n_nodes * world
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    N, E = soa.n_nodes, soa.n_entries
    F = wf.size * K * (AGENTS + 2) * 8
    # light Eq. 2 + key pass: per node acc_off 4 + flags 1 +
    # last 8 + ever 4 read, score 8 + key 16 + eff 4 + sublock 4 + missing 1
    # written; 12 B per access entry; the forecast rows + gs table once
    alg_light = 50 * N + 12 * E + F
    light_ms = float(kern[0])
    achieved = alg_light / (light_ms * 1e-3) / 1e9 if light_ms > 0 else None
    # selection: rank inputs 29 B + eff key 21 B per node
    alg_sel = 50 * N
    sel_ms = float(kern[1])
    achieved_sel = alg_sel / (sel_ms * 1e-3) / 1e9 if sel_ms > 0 else None
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        pass

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        r = cpu_reference_decisions(args.config, args.needed_frac, args.cpu_decisions,
                                    plan_bandwidth=max(1, used // 50) if prefetch else None,
                                    round_probe=prefetch["_round_first"] if prefetch else None)
        if r and prefetch and "round_candidate_s" in r:
            prefetch["round"]["cpu_reference"] = {
                "per_candidate_ms": 1e3 * r["round_candidate_s"], "cores": 1, "kind": "reference",
                "round_estimate_s": r["round_candidate_s"] * len(prefetch["_round_first"][1]),
                "sample": "one select_victims_hierarchical under the round's ancestry locks (simulator.hpp:652-657), "
                          "the per-candidate step of the reference loop; the round estimate multiplies it by the "
                          "candidate count"}
        if r and prefetch and "plan_times" in r:
            plan = prefetch["_plan"]
            prefetch["cpu_baseline"] = {"value": 1e3 * statistics.mean(r["plan_times"]), "unit": "ms/plan",
                                        "cores": 1, "kind": "reference",
                                        "sample": f"{len(r['plan_times'])} plan_conservative_prefetch calls on the "
                                                  f"same {args.config} tree"}
            prefetch["parity_vs_reference"] = (r["plan_selected"] == list(plan.selected)
                                               and r["plan_candidates"] == [c[0] for c in plan.candidates])
        if r:
            cpu = {"value": r["n_nodes"] / statistics.mean(r["times"]), "unit": "nodes/s", "cores": 1,
                   "kind": "reference",
                   "sample": f"{len(r['times'])} decisions on the same {args.config} tree "
                             f"(refresh_nodes all + select_victims_hierarchical), "
                             f"{statistics.mean(r['times']):.3f} s each; tree build {r['build_s']:.1f} s untimed"}
    line = {
        "metric": METRIC, "value": total_nodes / (ms * 1e-3), "unit": "nodes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n_nodes} nodes x {n_wf} workflows x K={K}, 30% retired, "
                               f"A={AGENTS}, HE select at {args.needed_frac:.2%} need, 1% leaves pinned",
                   "n_nodes": N, "n_entries": E, "needed_tokens": needed, "n_victims": res[0],
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single"},
        "p99_decision_ms": p99,
        "p50_decision_ms": float(np.percentile(per_step, 50)),
        "stage_ms": {"score_keys": float(stage[0]), "select": float(stage[1]), "total": float(stage[4])},
        "kernel_ms": {"score_light": float(kern[0]), "select_persistent": float(kern[1])},
        "select_phases_us": {"note": "lock, eff, chains, [hist, pick+compact] x passes, cut-head, "
                                     "sort, chain-starts, scatter, cut", "us": select_phases},
        "roofline": {"bound": "hbm", "kernel": "score_light_kernel (Eq. 2 of every light node + stage-3 keys)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None,
                     "traffic": traffic.get("score_light_kernel"), "alg_bytes_per_launch": alg_light,
                     "launch_ms": light_ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
        "roofline_select": {"bound": "hbm", "kernel": "select_persistent_kernel (latency-bound: grid phases)",
                            "achieved": achieved_sel, "peak": hbm_peak, "unit": "GB/s",
                            "frac": (achieved_sel / hbm_peak) if achieved_sel else None,
                            "traffic": traffic.get("select_persistent_kernel"), "alg_bytes_per_launch": alg_sel,
                            "launch_ms": sel_ms},
        "defer": dict(zip(("fast", "exact"), pol.defer_stats())),
        "need_sweep": sweep or None,
        "prefetch": {k: v for k, v in prefetch.items() if not k.startswith("_")} if prefetch else None,
        "pipeline_c2": pipeline_c2(torch, dev) if not args.no_pipeline else None,
        "cpu_baseline": cpu,
        "e2e": {"value": total_nodes / (e2e * 1e-3), "unit": "nodes/s",
                "h2d_bytes_per_step": int(statistics.mean(delta_fc) + 4 * locked.size
                                          + statistics.mean(delta_nodes) * (56 + 16 * E / N)),
                "d2h_bytes_per_step": int(4 * n_victims_e2e + 24), "ms_per_step": e2e,
                "p99_ms": float(np.percentile(e2e_ms, 99)),
                "what": "per decision: tree delta sync (pbkv_mirror_sync of the nodes changed by a churn batch: "
                        "16 inserts + 8 matches of live workflows, 1 termination, the previous decision's first 64 "
                        "victims demoted) + the touched workflows' forecasts re-put from pageable host memory "
                        "(refresh_workflow) and the terminated one's dropped + select with host locked list / "
                        "host victims; max(device events, host wall)",
                "delta_nodes_mean": statistics.mean(delta_nodes),
                "forecast_bytes_mean": statistics.mean(delta_fc),
                "put_all_forecasts_ms": statistics.median(put_all),
                "ms_per_step_all_forecasts_est": e2e - 1e3 * statistics.median(w[1] for w in e2e_wall)
                                             + statistics.median(put_all),
                "mirror_verified": mirror_ok,
                "host_wall_ms": {"sync": 1e3 * statistics.median(w[0] for w in e2e_wall),
                                 "put_forecasts": 1e3 * statistics.median(w[1] for w in e2e_wall),
                                 "select": 1e3 * statistics.median(w[2] for w in e2e_wall)}},
        "gpu_launches": int(k1 - k0),
        "lib_calls": int(l1 - l0),
        "clocks": clk.result,
        "tree_build_s": build_s,
    }
    print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
