"""Per-call latency of the policy call sites in the unmodified reference
simulator: the reference (oracle/_ref/sim_cpu) vs the GPU drop-in
(oracle/_ref/sim_gpu), same scenario and seed (BASELINE configs 1 and 5).
Writes one JSON object per (scenario, cell) to stdout (and to argv[1] if
given).  Run on the GPU box: python tools/sim_latency.py gpurun_out/sim_latency.json"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCEN = os.path.join(ROOT, "oracle", "_ref", "scenarios")
RUNS = [("codegen_retry.json", "policy_preset-he", 1), ("codegen_retry.json", "policy_preset-full", 1),
        ("loop.json", "policy_preset-he", 1), ("loop.json", "policy_preset-full", 1)]


def run(binary, scen, cell, seeds):
    env = dict(os.environ, PBKV_SIM_TIMING="1")
    r = subprocess.run([os.path.join(ROOT, "oracle", "_ref", binary), os.path.join(SCEN, scen), cell, str(seeds)],
                       capture_output=True, text=True, env=env, timeout=1800)
    assert r.returncode == 0, r.stderr
    line = r.stdout.strip().splitlines()[-1].split()
    ops = {}
    for ln in r.stderr.splitlines():
        f = ln.split()
        if f and f[0] == "timing":
            ops[f[1]] = {"calls": int(f[2]), "p50_us": float(f[3]), "p99_us": float(f[4]), "total_ms": float(f[5])}
    return {"hit_rate": float(line[2]), "events_fnv": line[6], "wall_s": float(line[-1]), "ops": ops}


out = []
for scen, cell, seeds in RUNS:
    c = run("sim_cpu", scen, cell, seeds)
    g = run("sim_gpu", scen, cell, seeds)
    rec = {"scenario": scen, "cell": cell, "seed": 1, "identical": c["events_fnv"] == g["events_fnv"],
           "hit_rate": c["hit_rate"], "wall_s": {"reference_cpu": c["wall_s"], "gpu_dropin": g["wall_s"]},
           "per_call": {op: {"reference_cpu": c["ops"].get(op), "gpu_dropin": g["ops"].get(op)}
                        for op in sorted(set(c["ops"]) | set(g["ops"]))}}
    out.append(rec)
    print(json.dumps(rec))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
