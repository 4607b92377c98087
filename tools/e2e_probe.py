"""GPU probe: where the e2e (host C ABI) decision time goes (run under gpurun)."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "oracle"]
import numpy as np
import torch
import workloads as WL
from paper_2605_06472_b200._abi import SCORE_RECOMPUTE
from paper_2605_06472_b200.api import HostTree, Policy
t = HostTree(); t.synth(n_nodes=1_000_000, n_workflows=4096, agents=16, seed=12345); soa = t.export()
rng = np.random.default_rng(12345)
wf = np.array(WL.workflows_of(soa), dtype=np.int64)
P = WL.random_forecasts(rng, wf.size, 8, 17)
locked = np.array(WL.pinned_paths(soa, rng, 0.01), dtype=np.int32)
pol = Policy(num_agents=16, k=8); pol.mirror(t); pol.put_forecasts(wf, P)
Pp = torch.from_numpy(np.ascontiguousarray(P)).pin_memory().numpy()
used = int(soa.len[soa.tier == 0][1:].sum()); needed = used // 100
for _ in range(5):
    pol.put_forecasts(wf, Pp); pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
tp, ts = [], []
for _ in range(20):
    t0 = time.perf_counter(); pol.put_forecasts(wf, Pp); t1 = time.perf_counter()
    pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE); t2 = time.perf_counter()
    tp.append(t1 - t0); ts.append(t2 - t1)
print(f"locked={locked.size} put_forecasts {np.median(tp)*1e6:.0f} us  select(host) {np.median(ts)*1e6:.0f} us  P bytes {P.nbytes}")
# raw C ABI call (no Python list conversion) for the same decision
import ctypes as C
from paper_2605_06472_b200 import _abi
from paper_2605_06472_b200._abi import POLICY_HE
L = _abi.lib()
lk = np.ascontiguousarray(locked, dtype=np.int32)
vb = np.empty(soa.n_nodes, dtype=np.int32)
nv, fr, sf = C.c_int64(), C.c_int64(), C.c_int()
tc = []
for _ in range(20):
    t0 = time.perf_counter()
    L.pbkv_select(pol._h, POLICY_HE, SCORE_RECOMPUTE, int(needed), lk.ctypes.data_as(C.POINTER(C.c_int32)), int(lk.size),
                  vb.ctypes.data_as(C.POINTER(C.c_int32)), int(vb.size), C.byref(nv), C.byref(fr), C.byref(sf))
    tc.append(time.perf_counter() - t0)
print(f"raw pbkv_select {np.median(tc)*1e6:.0f} us (victims {nv.value})")
# the bench's e2e loop shape: L2 flush + synchronize before each timed call pair
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.ExternalStream(pol.stream_handle())
tw, te = [], []
for _ in range(20):
    flush.fill_(1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    pol.put_forecasts(wf, Pp)
    sel = pol.select_victims_hierarchical(needed, locked=locked, score_mode=SCORE_RECOMPUTE)
    e1.record(stream)
    e1.synchronize()
    tw.append(time.perf_counter() - t0)
    te.append(e0.elapsed_time(e1))
print(f"flushed e2e: wall {np.median(tw)*1e6:.0f} us, events {np.median(te)*1e3:.0f} us")
