"""The unmodified reference simulator driving the GPU drop-in.

oracle/_ref/sim_gpu is simulator.hpp + scenario.hpp compiled with their
policy call sites (simulator.hpp:434, :464, :618, :636-637, :657) renamed onto
flowkv::gpu::* from include/pbkv/flowkv_gpu.hpp.  Every
score refresh, eviction decision and prefetch plan of the run is computed by
libpbkv.so on the B200.  The run must reproduce the CPU reference exactly:
hit rate, eviction / prefetch counters, and FNV-1a hashes of the full event
log and of the final tree dump (tests/golden/sim_cpu.txt, recorded by
tools/make_sim_golden.py from the reference-only build).
"""
import os
import subprocess

import pytest

from sim_cases import CASES, FED_CASES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SIM_GPU = os.path.join(ROOT, "oracle", "_ref", "sim_gpu")
SIM_CPU = os.path.join(ROOT, "oracle", "_ref", "sim_cpu")
SIM_FED = os.path.join(ROOT, "oracle", "_ref", "sim_gpu_fed")
SCEN = os.path.join(ROOT, "oracle", "_ref", "scenarios")
GOLDEN = os.path.join(ROOT, "tests", "golden", "sim_cpu.txt")


def golden_lines(scen):
    return [ln for ln in open(GOLDEN).read().splitlines() if ln.split()[0] == scen]


def run(binary, scen, cell, seeds):
    r = subprocess.run([binary, os.path.join(SCEN, scen), cell, str(seeds)], capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stderr
    return [" ".join([scen] + ln.split()[:-1]) for ln in r.stdout.strip().splitlines()]


def test_golden_covers_cases():
    lines = open(GOLDEN).read().splitlines()
    assert len(lines) == len(set(lines)) == 72
    # hit-rate means of the reference per preset: he 0.6189 on codegen_retry
    he = [float(ln.split()[3]) for ln in lines if ln.startswith("codegen_retry.json policy_preset-he ")]
    assert len(he) == 5 and abs(sum(he) / 5 - 0.6189) < 5e-5


@pytest.mark.skipif(not os.path.exists(SIM_CPU), reason="reference simulator not built (oracle/Makefile sim)")
def test_cpu_reference_reproduces_golden():
    scen, cell, seeds = CASES[0]
    got = run(SIM_CPU, scen, cell, seeds)
    want = [ln for ln in golden_lines(scen) if cell in ln]
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("scen,cell,seeds", CASES, ids=[f"{c[0]}:{c[1] or 'all'}" for c in CASES])
def test_gpu_simulator_matches_reference(gpu, scen, cell, seeds):
    if not os.path.exists(SIM_GPU):
        pytest.fail("oracle/_ref/sim_gpu missing: build with `make -C oracle sim` where /root/reference exists")
    got = run(SIM_GPU, scen, cell, seeds)
    want = [ln for ln in golden_lines(scen) if cell in ln.split()[1] and int(ln.split()[2]) <= seeds]
    assert len(got) == len(want) > 0
    for g, w in zip(got, want):
        assert g == w, f"GPU-driven simulator diverged from the reference:\n gpu {g}\n ref {w}"


FPARITY = os.path.join(ROOT, "oracle", "_ref", "forecast_parity")


@pytest.mark.gpu
def test_reference_predictors_bit_exact_on_gpu(gpu):
    """CallGraph::true_kstep_marginals, noisy_predict and MarkovModel::predict
    (orders 1-3) vs the batched GPU forecaster (csrc/fmodel.cu), on every
    bundled call graph: all probabilities bit-identical."""
    if not os.path.exists(FPARITY):
        pytest.fail("oracle/_ref/forecast_parity missing: build with `make -C oracle sim` where /root/reference exists")
    r = subprocess.run([FPARITY, os.path.join(SCEN, "graphs")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches=0" in r.stdout.splitlines()[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("scen,cell,seeds", FED_CASES, ids=[f"{c[0]}:{c[1] or 'all'}" for c in FED_CASES])
def test_device_fed_simulator_matches_reference(gpu, scen, cell, seeds):
    """The predictor slot too runs on the GPU (oracle / noisy / Markov
    forecasts, csrc/fmodel.cu): the run is device-fed end to end and must
    still reproduce the CPU reference's hit rate, counters, event log and
    final tree byte for byte."""
    if not os.path.exists(SIM_FED):
        pytest.fail("oracle/_ref/sim_gpu_fed missing: build with `make -C oracle sim` where /root/reference exists")
    got = run(SIM_FED, scen, cell, seeds)
    want = [ln for ln in golden_lines(scen) if cell in ln.split()[1] and int(ln.split()[2]) <= seeds]
    assert len(got) == len(want) > 0
    for g, w in zip(got, want):
        assert g == w, f"device-fed simulator diverged from the reference:\n gpu {g}\n ref {w}"
