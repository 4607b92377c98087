"""Known-answer vectors restated from the reference's own tests.

Each case rebuilds, through the op stream, the tree a reference TEST_CASE
builds through the CacheTree API, and carries the answer that test asserts:

  test_scoring.cpp:67-79    single-step value 0.7 / 0.8
  test_scoring.cpp:92-98    worked three-step score 0.9368
  test_scoring.cpp:318-323  missing forecast is an error
  test_policies.cpp:49-65   LRU evicts the least recently accessed leaf
  test_policies.cpp:67-75   exhausted candidates -> shortfall, 2 victims, 8 tokens
  test_policies.cpp:77-80   needed = 0 throws
  test_policies.cpp:105-117 LAE clears retired cache first
  test_policies.cpp:119-133 less popular retired first (ever_tagged 1 vs 7)
  test_policies.cpp:152-163 HE drains retired before any active score
  test_policies.cpp:165-176 HE ascending score order {b, c, a}
  test_policies.cpp:195-202 locked nodes are never selected
  test_policies.cpp:262-287 kvflow farthest first / never-recurring first
  test_policies.cpp:296-309 kvflow minimises distance across tagged workflows
  test_policies.cpp:311-324 zero space budget -> empty plan
  test_policies.cpp:326-341 bandwidth caps the selected volume (Sbw 60 vs 100)
  test_policies.cpp:343-370 greedy fill {c1, c3} = 60 tokens
  test_policies.cpp:372-409 greedy below the knapsack optimum: {c1}
  test_policies.cpp:411-419 zero-value host nodes are never candidates
  test_policies.cpp:421-434 candidates must hang below device-resident parents
  test_policies.cpp:436-459 aggressive rho = 0.2 -> displacement 200
"""
from __future__ import annotations

import numpy as np

from paper_2605_06472_b200._abi import POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU
from paper_2605_06472_b200.ops import OpStream


def tokens_of(base: int, n: int) -> list[int]:
    return list(range(base, base + n))


def constant_forecast(outcomes: int, hot: int, K: int = 3) -> np.ndarray:
    P = np.zeros((K, outcomes))
    P[:, hot] = 1.0
    return P


class Case:
    def __init__(self, name, ops, dev_cap=1 << 20, host_cap=1 << 20, forecasts=None, agents=None, k=3,
                 gamma=0.7, action=None, expect=None, error=None):
        self.name = name
        self.ops = ops
        self.dev_cap, self.host_cap = dev_cap, host_cap
        self.forecasts = forecasts or {}  # wf -> [K, V1]
        self.k, self.gamma = k, gamma
        self.action = action  # tuple
        self.expect = expect or {}
        self.error = error
        V1s = {np.asarray(p).shape[1] for p in self.forecasts.values()}
        self.agents = agents if agents is not None else (max(V1s) - 1 if V1s else 4)

    def forecast_arrays(self):
        if not self.forecasts:
            return np.zeros(0, dtype=np.int64), np.zeros((0, 1, self.agents + 1))
        wf = sorted(self.forecasts)
        H = max(np.asarray(self.forecasts[w]).shape[0] for w in wf)
        return np.array(wf, dtype=np.int64), np.stack([np.asarray(self.forecasts[w], dtype=np.float64) for w in wf])

    def __repr__(self):
        return self.name


def cases() -> list[Case]:
    out: list[Case] = []

    # --- stage 2 -----------------------------------------------------------------
    ops = OpStream().insert([1, 2, 3], 1, 0)
    f = np.array([[0.5, 0.3, 0.2]] * 3)  # P(a)=0.5, p_end=0.2 at every step
    out.append(Case("worked_three_step_score", ops, forecasts={1: f}, k=3, gamma=0.7,
                    action=("score", [1]), expect={"approx": [0.9368], "tol": 1e-12}))

    ops = OpStream().insert([1, 2], 1, 0).insert([1, 2], 1, 2)  # bits 0b101
    out.append(Case("single_step_value_0.7", ops, forecasts={1: np.array([[0.2, 0.3, 0.5, 0.0]])}, k=1,
                    action=("value", [1]), expect={"approx": [0.7], "tol": 1e-12}))

    ops = OpStream().insert([5], 1, 0).insert([5], 2, 0).insert([5], 2, 2)
    out.append(Case("single_step_value_0.8", ops,
                    forecasts={1: np.array([[0.4, 0.1, 0.2, 0.3]]), 2: np.array([[0.25, 0.3, 0.15, 0.3]])}, k=1,
                    action=("value", [1]), expect={"approx": [0.8], "tol": 1e-12}))

    ops = OpStream().insert([1], 1, 0)
    out.append(Case("missing_forecast_is_error", ops, agents=2, forecasts={}, action=("score", [1]),
                    error="missing forecast for active workflow 1"))

    # --- stage 3 -----------------------------------------------------------------
    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0).insert(tokens_of(300, 4), 3, 0)
    ops.match(tokens_of(100, 4), 1, 0).match(tokens_of(300, 4), 3, 0)
    out.append(Case("lru_oldest_leaf", ops, action=("select", POLICY_LRU, 1, []),
                    expect={"first": 2, "shortfall": False}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0)
    out.append(Case("exhausted_shortfall", ops, action=("select", POLICY_LRU, 100, []),
                    expect={"victims": [1, 2], "freed": 8, "shortfall": True}))
    out.append(Case("needed_zero_throws", ops, action=("select", POLICY_LRU, 0, []),
                    error="eviction request must free a positive amount"))
    out.append(Case("locked_never_selected", ops, action=("select", POLICY_LRU, 8, [1]),
                    expect={"victims": [2], "freed": 4, "shortfall": True}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0).terminate(1)
    ops.match(tokens_of(200, 4), 2, 0)
    out.append(Case("lae_retired_first", ops, action=("select", POLICY_LAE, 1, []), expect={"first": 1}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0)
    for w in range(3, 9):
        ops.match(tokens_of(200, 4), w, 0)
    for w in range(1, 9):
        ops.terminate(w)
    out.append(Case("lae_less_popular_first", ops, action=("select", POLICY_LAE, 8, []),
                    expect={"victims": [1, 2]}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0).terminate(1)
    ops.set_score(1, 10.0).set_score(2, 0.01)
    out.append(Case("he_retired_before_active", ops, action=("select", POLICY_HE, 1, []), expect={"first": 1}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 0).insert(tokens_of(300, 4), 3, 0)
    ops.set_score(1, 0.9).set_score(2, 0.1).set_score(3, 0.5)
    out.append(Case("he_ascending_score", ops, action=("select", POLICY_HE, 12, []),
                    expect={"victims": [2, 3, 1]}))

    ops = OpStream().insert(tokens_of(100, 4), 1, 0).insert(tokens_of(200, 4), 2, 1)
    out.append(Case("kvflow_farthest_first", ops,
                    action=("select_kvflow", 1, [], {1: [0, 2, 2], 2: [2, 2, 2, 2, 1]}), expect={"first": 2}))
    out.append(Case("kvflow_never_recurring_first", ops,
                    action=("select_kvflow", 8, [], {1: [2, 2, 2], 2: [1]}), expect={"victims": [1, 2]}))
    out.append(Case("kvflow_requires_sequences", OpStream().insert(tokens_of(100, 4), 1, 0),
                    action=("select_kvflow", 1, [], {}),
                    error="kvflow needs a static remaining sequence for workflow 1"))
    ops = OpStream().insert(tokens_of(100, 4), 1, 0).match(tokens_of(100, 4), 2, 1).insert(tokens_of(200, 4), 3, 2)
    out.append(Case("kvflow_min_distance", ops,
                    action=("select_kvflow", 1, [], {1: [2, 2, 0], 2: [1], 3: [1, 2]}), expect={"first": 2}))

    # --- stage 4 -----------------------------------------------------------------
    ops = OpStream().insert(tokens_of(500, 100), 9, 0).insert(tokens_of(900, 10), 1, 0, budget=0)
    out.append(Case("prefetch_zero_budget", ops, dev_cap=100,
                    forecasts={1: constant_forecast(3, 0), 9: constant_forecast(3, 1)},
                    action=("plan", 1000, 1, -1.0), expect={"budget_space": 0, "selected": []}))

    ops = OpStream().insert(tokens_of(500, 80), 1, 0).demote(1)
    out.append(Case("prefetch_bw_cap_60", ops, dev_cap=200, forecasts={1: constant_forecast(2, 0)},
                    action=("plan", 60, 1, -1.0), expect={"budget_space": 200, "budget_bw": 60, "selected": []}))
    out.append(Case("prefetch_bw_cap_100", ops, dev_cap=200, forecasts={1: constant_forecast(2, 0)},
                    action=("plan", 100, 1, -1.0), expect={"selected": [1]}))

    def weighted(v):
        return np.array([[v, 1.0 - v, 0.0]])

    ops = OpStream().insert(tokens_of(500, 50), 1, 0).insert(tokens_of(700, 40), 2, 0).insert(tokens_of(900, 10), 3, 0)
    ops.demote(1).demote(2).demote(3).insert(tokens_of(100, 940), 9, 1)
    out.append(Case("prefetch_greedy_c1_c3", ops, dev_cap=1000,
                    forecasts={1: weighted(0.9), 2: weighted(0.8), 3: weighted(0.7), 9: weighted(0.0)}, k=1,
                    action=("plan", 1000, 1, -1.0),
                    expect={"n_candidates": 3, "first_candidate": 1, "selected": [1, 3], "selected_tokens": 60}))

    ops = OpStream().insert(tokens_of(500, 60), 1, 0).insert(tokens_of(700, 30), 2, 0).insert(tokens_of(900, 30), 3, 0)
    ops.demote(1).demote(2).demote(3).insert(tokens_of(100, 940), 9, 1)
    out.append(Case("prefetch_greedy_below_knapsack", ops, dev_cap=1000,
                    forecasts={1: weighted(0.9), 2: weighted(0.85), 3: weighted(0.8), 9: weighted(0.0)}, k=1,
                    action=("plan", 1000, 1, -1.0), expect={"selected": [1]}))

    ops = OpStream().insert(tokens_of(500, 10), 1, 0).demote(1).terminate(1)
    out.append(Case("prefetch_zero_value_excluded", ops, dev_cap=1000, agents=2, forecasts={},
                    action=("plan", 1000, 1, -1.0), expect={"n_candidates": 0}))

    ops = OpStream().insert(tokens_of(500, 10), 1, 0).insert(tokens_of(500, 20), 1, 0).demote(2).demote(1)
    out.append(Case("prefetch_device_parent_required", ops, dev_cap=1000, forecasts={1: constant_forecast(3, 0)},
                    action=("plan", 1000, 1, -1.0), expect={"candidates": [1]}))

    ops = OpStream().insert(tokens_of(500, 100), 1, 0).demote(1).insert(tokens_of(100, 950), 9, 1)
    fc = {1: constant_forecast(3, 0), 9: constant_forecast(3, 1)}
    out.append(Case("prefetch_conservative_cannot_fit", ops, dev_cap=1000, forecasts=fc,
                    action=("plan", 10000, 1, -1.0), expect={"selected": []}))
    out.append(Case("prefetch_aggressive_rho0", ops, dev_cap=1000, forecasts=fc,
                    action=("plan", 10000, 1, 0.0), expect={"selected": [], "displacement_budget": 0}))
    out.append(Case("prefetch_aggressive_rho02", ops, dev_cap=1000, forecasts=fc,
                    action=("plan", 10000, 1, 0.2), expect={"selected": [1], "displacement_budget": 200}))
    out.append(Case("prefetch_aggressive_rho_out_of_range", ops, dev_cap=1000, forecasts=fc,
                    action=("plan", 10000, 1, 1.5), error="rho must be in [0, 1]"))
    return out


def check(case: Case, result) -> None:
    """Assert `result` (Selection / Plan / list of floats) matches the case."""
    e = case.expect
    kind = case.action[0]
    if kind in ("score", "value"):
        vals = list(result)
        for got, want in zip(vals, e["approx"]):
            assert abs(got - want) <= e["tol"], (case.name, got, want)
        return
    if kind.startswith("select"):
        if "first" in e:
            assert result.victims and result.victims[0] == e["first"], (case.name, result)
        if "victims" in e:
            assert result.victims == e["victims"], (case.name, result)
        if "freed" in e:
            assert result.freed == e["freed"], (case.name, result)
        if "shortfall" in e:
            assert result.shortfall == e["shortfall"], (case.name, result)
        return
    if kind == "plan":
        for key in ("budget_space", "budget_bw", "selected_tokens", "displacement_budget"):
            if key in e:
                assert getattr(result, key) == e[key], (case.name, key, result)
        if "selected" in e:
            assert result.selected == e["selected"], (case.name, result)
        if "n_candidates" in e:
            assert len(result.candidates) == e["n_candidates"], (case.name, result)
        if "first_candidate" in e:
            assert result.candidates[0][0] == e["first_candidate"], (case.name, result)
        if "candidates" in e:
            assert [c[0] for c in result.candidates] == e["candidates"], (case.name, result)
        return
    raise AssertionError(kind)
