"""GPU probe: host vs device time of one pbkv_predict call at the C3 batch (run under gpurun)."""
import os, sys, time
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
import numpy as np
import torch
from paper_2605_06472_b200.api import Policy
from paper_2605_06472_b200.predictor import PredictorWeights, random_inputs
n, A, K, H = 2868, 16, 8, 5120
w = PredictorWeights.random(num_agents=A, horizon=K, text_dim=H)
off, pre, x = random_inputs(n, A, H, max_prefix=64)
pol = Policy(num_agents=A, k=K, gamma=0.7)
pol.load_predictor(w, max_prefix=64)
wf = np.arange(n)
xd = torch.from_numpy(x.view(np.int16)).cuda()
for _ in range(5):
    pol.predict(wf, off, pre, None, x_device_ptr=xd.data_ptr(), want_probs=False)
torch.cuda.synchronize()
ts, td = [], []
pol.set_timing(True)
for _ in range(30):
    t0 = time.perf_counter()
    pol.predict(wf, off, pre, None, x_device_ptr=xd.data_ptr(), want_probs=False)
    ts.append(time.perf_counter() - t0)
    td.append(pol.timings()[0])
pol.set_timing(False)
print(f"predict wall {np.median(ts)*1e6:.0f} us, device (events) {np.median(td)*1e3:.0f} us, prefix elems {pre.size}")
