"""GPU probe: predictor error vs the FP64 restatement and device time (run under gpurun)."""
import sys
import os
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "tests"]
import numpy as np
import torch
import predictor_ref as PR
from paper_2605_06472_b200.api import Policy
from paper_2605_06472_b200.predictor import PredictorWeights, random_inputs

for n, A, K, H in [(256, 16, 4, 5120), (4096, 16, 8, 5120)]:
    w = PredictorWeights.random(num_agents=A, horizon=K, text_dim=H)
    off, pre, x = random_inputs(n, A, H, max_prefix=64)
    pol = Policy(num_agents=A, k=K, gamma=0.7)
    pol.load_predictor(w, max_prefix=64)
    wf = np.arange(n)
    P = pol.predict(wf, off, pre, x)
    R = PR.forward(w, off, pre, x)
    # ablation: zero x must change the result (h_txt really flows through the GEMM)
    P0 = pol.predict(wf, off, pre, np.zeros_like(x))
    xd = torch.from_numpy(x.view(np.int16)).cuda()
    for _ in range(3):
        pol.predict(wf, off, pre, None, x_device_ptr=xd.data_ptr(), want_probs=False)
    torch.cuda.synchronize()
    pol.set_timing(True)
    ts = []
    for _ in range(20):
        pol.predict(wf, off, pre, None, x_device_ptr=xd.data_ptr(), want_probs=False)
        ts.append(pol.timings()[0])
    pol.set_timing(False)
    print(f"n={n} A={A} K={K} H={H}: max|err|={np.max(np.abs(P - R)):.3e} "
          f"mean|err|={np.mean(np.abs(P - R)):.3e} |P-P(x=0)|max={np.max(np.abs(P - P0)):.3f} "
          f"device ms (predict+prepare) median={np.median(ts):.4f} x bytes={x.nbytes}")
