"""(scenario file, cell filter, number of seeds) replayed by the interposed
simulator parity test (BASELINE configs 1 and 5 plus the static pipeline)."""
CASES = [
    ("codegen_retry.json", "", 5),       # config 1: lru / lae / he / full, seeds 1-5
    ("static_pipeline.json", "", 2),     # lru / kvflow / full
    ("loop.json", "policy_preset-he", 2),    # config 5 (mixed multi-agent, HiCache host tier)
    ("loop.json", "policy_preset-full", 2),  # score-driven eviction + conservative prefetch
]
