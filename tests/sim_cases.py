"""(scenario file, cell filter, number of seeds) replayed by the interposed
simulator parity tests.

CASES run through oracle/_ref/sim_gpu (policy call sites on the GPU drop-in):
BASELINE configs 1 (codegen_retry, every preset) and 5 (loop.json: the mixed
multi-agent scenario with the HiCache host tier, every preset, seeds 1-10 for
the score-driven presets) plus the static pipeline.

FED_CASES run through oracle/_ref/sim_gpu_fed, where the predictor slot
(simulator.hpp:414-421) is device-fed as well (oracle, noisy and Markov
predictors; tests/scenarios/*.json are scenario files over the bundled call
graphs)."""
CASES = [
    ("codegen_retry.json", "", 5),           # config 1: lru / lae / he / full, seeds 1-5
    ("static_pipeline.json", "", 2),         # lru / kvflow / full
    ("loop.json", "policy_preset-he", 10),   # config 5: score-driven eviction
    ("loop.json", "policy_preset-full", 10), # + conservative prefetch under load
    ("loop.json", "policy_preset-lru", 3),
    ("loop.json", "policy_preset-lae", 3),
]
FED_CASES = [
    ("codegen_predictors.json", "", 3),      # oracle / noisy (lambda 0.3) / markov (order 2) x he / full
    ("loop_predictors.json", "", 1),         # noisy / markov on loop.json's graph, full preset
    ("loop.json", "policy_preset-full", 1),  # the oracle predictor on config 5
]
