"""Records the CPU reference simulator's outcomes (oracle/_ref/sim_cpu, the
unmodified reference built from /root/reference) for the bundled scenarios
into tests/golden/sim_cpu.txt.  tests/test_sim_interpose.py replays the same
(scenario, cell, seeds) through oracle/_ref/sim_gpu (policy call sites
interposed onto the GPU drop-in) and requires identical lines.

Run here (needs /root/reference): python tools/make_sim_golden.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from sim_cases import CASES, FED_CASES  # noqa: E402

out = []
seen = set()
for scen, cell, seeds in CASES + FED_CASES:
    r = subprocess.run([os.path.join(ROOT, "oracle/_ref/sim_cpu"), os.path.join(ROOT, "oracle/_ref/scenarios", scen),
                        cell, str(seeds)], check=True, capture_output=True, text=True)
    for line in r.stdout.strip().splitlines():
        f = line.split()
        ln = " ".join([scen] + f[:-1])  # drop the wall-clock column
        if ln not in seen:
            seen.add(ln)
            out.append(ln)
path = os.path.join(ROOT, "tests/golden/sim_cpu.txt")
open(path, "w").write("\n".join(out) + "\n")
print(f"{len(out)} runs -> {path}")
