"""Host-side mirror of the reference policy interface, on top of libpbkv.so.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/flowkv/{policies,scoring}.hpp:

  reference (C++)                                   here (GPU path)
  select_victims(tree, policy, needed, rem, locked)  Policy.select_victims
  select_victims_{lru,lae,hierarchical,kvflow}      Policy.select_victims_*
  plan_conservative_prefetch(tree, fp, bw, step)     Policy.plan_conservative_prefetch
  plan_aggressive_prefetch(tree, fp, bw, rho, step)  Policy.plan_aggressive_prefetch
  multi_step_score(node_terms(...))                  Policy.score_nodes / score_all
  single_step_value(node_terms(...))                 Policy.value_nodes
  flowkv::ValidationError                            ValidationError (same messages)

The tree is mirrored on the device: ``Policy.mirror(tree)`` uploads the whole
struct-of-arrays image (from a HostTree -- the reference flowkv::CacheTree
with a change log -- or from any SoAArrays export), ``Policy.sync(tree)``
uploads only the nodes changed since (pbkv_mirror_delta), and
``Policy.apply_delta`` takes caller-built node records; forecasts are
uploaded with ``put_forecasts``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

from . import _abi
from ._abi import (POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU, SCORE_CACHED, SCORE_RECOMPUTE,
                   SoAArrays, ptr)


class ValidationError(RuntimeError):
    """flowkv::ValidationError (errors.hpp:24-26) raised through the C ABI."""


class PbkvError(RuntimeError):
    """CUDA / allocation / ABI-level failure (PBKV_ECUDA, PBKV_ENOMEM, PBKV_EARG)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[pbkv status {status}] {msg}")
        self.status = status


def _check(rc: int, handle) -> None:
    if rc == _abi.PBKV_OK:
        return
    msg = _abi.lib().pbkv_last_error(handle).decode()
    if rc == _abi.PBKV_EINVAL:
        raise ValidationError(msg)
    raise PbkvError(rc, msg)


class VictimSelection:
    """policies.hpp:30-34 (victims, freed, shortfall).

    `victim_ids` is the int32 array the C ABI filled; `victims` is the same
    order as a Python list, built on first access (a 7 K-victim list costs
    tens of microseconds, more than the copy out of the GPU)."""

    __slots__ = ("victim_ids", "freed", "shortfall", "_list")

    def __init__(self, victims=None, freed: int = 0, shortfall: bool = False):
        self.victim_ids = np.asarray(victims if victims is not None else [], dtype=np.int32)
        self.freed = int(freed)
        self.shortfall = bool(shortfall)
        self._list = victims if isinstance(victims, list) else None

    @property
    def victims(self) -> list[int]:
        if self._list is None:
            self._list = self.victim_ids.tolist()
        return self._list

    def __len__(self) -> int:
        return int(self.victim_ids.size)

    def __bool__(self) -> bool:
        # A selection is a result, not a container: an empty one (shortfall,
        # no victims) stays truthy, as the dataclass it replaces was.
        return True

    def __eq__(self, other) -> bool:
        if not isinstance(other, VictimSelection):
            return NotImplemented
        return (self.victims, self.freed, self.shortfall) == (other.victims, other.freed, other.shortfall)

    def __repr__(self) -> str:
        return f"VictimSelection(victims={self.victims!r}, freed={self.freed}, shortfall={self.shortfall})"


class RoundVictims:
    """The victims demoted before each candidate of a prefetch round, as one
    flat array with per-candidate ends; indexes and compares like the list of
    lists the reference loop produces (simulator.hpp:649-672)."""

    __slots__ = ("flat", "ends")

    def __init__(self, flat: np.ndarray, ends: np.ndarray):
        self.flat = flat
        self.ends = ends

    def __len__(self) -> int:
        return int(self.ends.size)

    def __getitem__(self, i: int) -> list[int]:
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        b = int(self.ends[i - 1]) if i else 0
        return self.flat[b: int(self.ends[i])].tolist()

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    def __eq__(self, other) -> bool:
        if isinstance(other, RoundVictims):
            return np.array_equal(self.flat, other.flat) and np.array_equal(self.ends, other.ends)
        try:
            if len(other) != len(self):
                return False
            lens = np.diff(np.concatenate([[0], self.ends]))
            if any(len(o) != int(l) for o, l in zip(other, lens)):
                return False
            flat = [int(v) for o in other for v in o]
            return np.array_equal(self.flat, np.asarray(flat, dtype=self.flat.dtype))
        except TypeError:
            return NotImplemented

    def __repr__(self) -> str:
        return f"RoundVictims({list(self)!r})"


class PrefetchPlan:
    """policies.hpp:170-177.

    `candidate_ids` / `candidate_values` / `selected_ids` are the arrays the C
    ABI filled; `candidates` (a list of (id, value) pairs, best first) and
    `selected` are built from them on first access."""

    __slots__ = ("candidate_ids", "candidate_values", "selected_ids", "budget_space", "budget_bw",
                 "displacement_budget", "selected_tokens", "_cand", "_sel")

    def __init__(self, candidates=None, budget_space: int = 0, budget_bw: int = 0, displacement_budget: int = 0,
                 selected=None, selected_tokens: int = 0):
        cand = list(candidates) if candidates is not None else []
        self.candidate_ids = np.array([c[0] for c in cand], dtype=np.int32)
        self.candidate_values = np.array([c[1] for c in cand], dtype=np.float64)
        self.selected_ids = np.asarray(selected if selected is not None else [], dtype=np.int32)
        self.budget_space = int(budget_space)
        self.budget_bw = int(budget_bw)
        self.displacement_budget = int(displacement_budget)
        self.selected_tokens = int(selected_tokens)
        self._cand = cand if candidates is not None else None
        self._sel = list(selected) if selected is not None else None

    @classmethod
    def from_arrays(cls, cid, cv, sel, budget_space, budget_bw, displacement_budget, selected_tokens):
        p = cls.__new__(cls)
        p.candidate_ids, p.candidate_values, p.selected_ids = cid, cv, sel
        p.budget_space, p.budget_bw = int(budget_space), int(budget_bw)
        p.displacement_budget, p.selected_tokens = int(displacement_budget), int(selected_tokens)
        p._cand = p._sel = None
        return p

    @property
    def candidates(self) -> list[tuple[int, float]]:
        if self._cand is None:
            self._cand = list(zip(self.candidate_ids.tolist(), self.candidate_values.tolist()))
        return self._cand

    @property
    def selected(self) -> list[int]:
        if self._sel is None:
            self._sel = self.selected_ids.tolist()
        return self._sel

    def __eq__(self, other) -> bool:
        if not isinstance(other, PrefetchPlan):
            return NotImplemented
        return (self.candidates, self.budget_space, self.budget_bw, self.displacement_budget, self.selected,
                self.selected_tokens) == (other.candidates, other.budget_space, other.budget_bw,
                                          other.displacement_budget, other.selected, other.selected_tokens)

    def __repr__(self) -> str:
        return (f"PrefetchPlan(candidates={self.candidates!r}, budget_space={self.budget_space}, "
                f"budget_bw={self.budget_bw}, displacement_budget={self.displacement_budget}, "
                f"selected={self.selected!r}, selected_tokens={self.selected_tokens})")


# ----------------------------------------------------------------------------------
class HostTree:
    """The reference flowkv::CacheTree (cache.hpp) wrapped in TrackedCacheTree
    (include/pbkv/tracked_tree.hpp): the reference mutation semantics, an SoA
    export and a change log for incremental device sync."""

    def __init__(self, device_capacity: int = 1 << 40, host_capacity: int = 1 << 40):
        L = _abi.lib()
        h = C.c_void_p()
        _check(L.pbkv_tree_create(C.byref(h), int(device_capacity), int(host_capacity)), None)
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _abi.lib().pbkv_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def apply_ops(self, words: Sequence[int] | np.ndarray) -> None:
        w = np.ascontiguousarray(np.asarray(words, dtype=np.int64))
        _check(_abi.lib().pbkv_tree_apply_ops(self._h, ptr(w, C.c_int64), int(w.size)), None)

    def synth(self, **params) -> None:
        p = _abi.synth_params(**params)
        _check(_abi.lib().pbkv_tree_synth(self._h, C.byref(p)), None)

    def export(self) -> SoAArrays:
        L = _abi.lib()
        shape = _abi.TreeSoA()
        _check(L.pbkv_tree_shape(self._h, C.byref(shape)), None)
        arr = SoAArrays(shape.n_nodes, shape.n_entries, dict(
            device_capacity=shape.device_capacity, device_used=shape.device_used,
            retired_device_tokens=shape.retired_device_tokens, host_capacity=shape.host_capacity,
            host_used=shape.host_used))
        s = arr.struct()
        _check(L.pbkv_tree_export(self._h, C.byref(s)), None)
        return arr

    def log(self, pos: int = 0) -> tuple[int, list[int] | None]:
        """(change-log end, ascending ids of the nodes changed since pos --
        None when the log no longer reaches back to pos)."""
        L = _abi.lib()
        end, n = C.c_int64(), C.c_int64()
        _check(L.pbkv_tree_log(self._h, int(pos), C.byref(end), None, 0, C.byref(n)), None)
        if n.value < 0:
            return end.value, None
        ids = np.zeros(max(n.value, 1), dtype=np.int32)
        _check(L.pbkv_tree_log(self._h, int(pos), C.byref(end), ptr(ids, C.c_int32), n.value, C.byref(n)), None)
        return end.value, ids[: n.value].tolist()

    def log_end(self) -> int:
        """Current change-log position."""
        end, n = C.c_int64(), C.c_int64()
        _check(_abi.lib().pbkv_tree_log(self._h, 1 << 62, C.byref(end), None, 0, C.byref(n)), None)
        return end.value

    def touched(self, wf: int) -> list[int]:
        L = _abi.lib()
        n = C.c_int64()
        _check(L.pbkv_tree_touched(self._h, int(wf), None, 0, C.byref(n)), None)
        ids = np.zeros(max(n.value, 1), dtype=np.int32)
        _check(L.pbkv_tree_touched(self._h, int(wf), ptr(ids, C.c_int32), n.value, C.byref(n)), None)
        return ids[: n.value].tolist()


# ----------------------------------------------------------------------------------
class Policy:
    """One device context (one CUDA stream, one tree mirror, one forecast store)."""

    def __init__(self, num_agents: int, k: int = 3, gamma: float = 0.7, device: int = 0):
        L = _abi.lib()
        cfg = _abi.Cfg(int(device), int(k), float(gamma), int(num_agents))
        h = C.c_void_p()
        _check(L.pbkv_ctx_create(C.byref(h), C.byref(cfg)), None)
        self._h = h
        self.k, self.gamma, self.num_agents = int(k), float(gamma), int(num_agents)
        self.n_nodes = 0

    def close(self):
        if getattr(self, "_h", None):
            _abi.lib().pbkv_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def _c(self, rc):
        _check(rc, self._h)

    # ---- mirror ------------------------------------------------------------------
    def mirror(self, tree: "HostTree | SoAArrays", with_depth: bool = True) -> None:
        L = _abi.lib()
        if isinstance(tree, HostTree):
            self._c(L.pbkv_mirror_tree(self._h, tree.handle))
        else:
            s = tree.struct(with_depth=with_depth)
            self._c(L.pbkv_mirror_full(self._h, C.byref(s)))
        n = C.c_int64()
        self._c(L.pbkv_mirror_node_count(self._h, C.byref(n), None))
        self.n_nodes = n.value

    def sync(self, tree: "HostTree") -> None:
        """pbkv_mirror_sync: upload only the nodes changed since this context
        last mirrored `tree` (a full upload the first time)."""
        L = _abi.lib()
        self._c(L.pbkv_mirror_sync(self._h, tree.handle))
        n = C.c_int64()
        self._c(L.pbkv_mirror_node_count(self._h, C.byref(n), None))
        self.n_nodes = n.value

    def apply_delta(self, records: np.ndarray, acc_wf: np.ndarray, acc_bits: np.ndarray,
                    totals: Mapping[str, int] | None = None) -> None:
        """pbkv_mirror_delta: records is a NODE_DELTA_DTYPE array."""
        L = _abi.lib()
        r = np.ascontiguousarray(records, dtype=_abi.NODE_DELTA_DTYPE)
        w = np.ascontiguousarray(acc_wf if len(acc_wf) else [0], dtype=np.int64)
        b = np.ascontiguousarray(acc_bits if len(acc_bits) else [0], dtype=np.uint64)
        t = _abi.TreeTotals(**totals) if totals else None
        self._c(L.pbkv_mirror_delta(self._h, C.c_void_p(r.ctypes.data), int(r.size), ptr(w, C.c_int64),
                                    ptr(b, C.c_uint64), C.byref(t) if t is not None else None))
        n = C.c_int64()
        self._c(L.pbkv_mirror_node_count(self._h, C.byref(n), None))
        self.n_nodes = n.value

    def verify(self, tree: "HostTree | SoAArrays") -> int:
        """pbkv_mirror_verify against a full snapshot: -1 when the device
        mirror equals it field by field, else the first differing node id."""
        soa = tree.export() if isinstance(tree, HostTree) else tree
        s = soa.struct(with_depth=isinstance(tree, HostTree))
        m = C.c_int64()
        self._c(_abi.lib().pbkv_mirror_verify(self._h, C.byref(s), C.byref(m)))
        return m.value

    def set_scores(self, ids: Sequence[int], scores: Sequence[float]) -> None:
        i = np.ascontiguousarray(ids, dtype=np.int32)
        s = np.ascontiguousarray(scores, dtype=np.float64)
        self._c(_abi.lib().pbkv_mirror_set_scores(self._h, ptr(i, C.c_int32), ptr(s, C.c_double), int(i.size)))

    # ---- forecasts -----------------------------------------------------------------
    def put_forecasts(self, wf_ids: Sequence[int], probs: np.ndarray, validate_now: bool = True) -> None:
        """probs: [n, horizon, outcomes] float64 (Forecast rows, forecast.hpp:19).
        validate_now=False (pbkv_forecast_put_async, the C++ shim's mode): no
        synchronisation; a validation error (forecast.hpp:25-34) is raised by
        the next call that reads the status word."""
        w = np.ascontiguousarray(wf_ids, dtype=np.int64)
        p = np.ascontiguousarray(probs, dtype=np.float64)
        if p.ndim != 3 or p.shape[0] != w.size:
            raise ValueError("probs must be [n_workflows, horizon, outcomes]")
        fn = _abi.lib().pbkv_forecast_put if validate_now else _abi.lib().pbkv_forecast_put_async
        self._c(fn(self._h, ptr(w, C.c_int64), int(w.size), int(p.shape[1]), int(p.shape[2]), ptr(p, C.c_double)))

    def drop_forecasts(self, wf_ids: Iterable[int]) -> None:
        w = np.ascontiguousarray(list(wf_ids), dtype=np.int64)
        self._c(_abi.lib().pbkv_forecast_drop(self._h, ptr(w, C.c_int64), int(w.size)))

    def set_remaining(self, remaining: Mapping[int, Sequence[int]]) -> None:
        """Static remaining agent sequences for KVFlow (policies.hpp:144-153)."""
        wf = np.array(sorted(remaining), dtype=np.int64)
        off = np.zeros(wf.size + 1, dtype=np.int64)
        flat: list[int] = []
        for i, w in enumerate(wf.tolist()):
            flat.extend(int(a) for a in remaining[w])
            off[i + 1] = len(flat)
        seq = np.array(flat if flat else [0], dtype=np.int32)
        self._c(_abi.lib().pbkv_set_remaining(self._h, ptr(wf, C.c_int64), int(wf.size), ptr(off, C.c_int64),
                                              ptr(seq, C.c_int32)))

    # ---- stage 1 -------------------------------------------------------------------
    def load_predictor(self, w, max_prefix: int = 64) -> None:
        """pbkv_predictor_load: weights of the PAPER.md:1040-1066 model
        (paper_2605_06472_b200.predictor.PredictorWeights)."""
        cfg = _abi.PredictorCfg(w.num_agents, w.horizon, w.dim, w.hidden, w.text_dim, max_prefix)
        keep = {f: np.ascontiguousarray(getattr(w, f)) for f in
                ("embed", "transition", "sage1", "sage2", "query", "mlp1", "mlp1_bias", "mlp2", "mlp2_bias")}
        keep["text"] = np.ascontiguousarray(w.text, dtype=np.uint16)
        pw = _abi.PredictorWeights(**{f: ptr(a, C.c_uint16 if f == "text" else C.c_float) for f, a in keep.items()})
        self._c(_abi.lib().pbkv_predictor_load(self._h, C.byref(cfg), C.byref(pw)))
        self._pred = (w.horizon, w.num_agents + 1, w.text_dim)

    def predict(self, wf_ids: Sequence[int], prefix_off: np.ndarray, prefix: np.ndarray, x, *,
                x_device_ptr: int | None = None, want_probs: bool = True) -> np.ndarray | None:
        """pbkv_predict: one batched forward; the forecasts become resident
        (replacing put_forecasts).  x: [n, H] bf16 bits (host), or pass
        x_device_ptr for hidden states already in HBM.  Returns the stored
        [n, K, A+1] float64 forecasts when want_probs."""
        K, V1, H = self._pred
        w = np.ascontiguousarray(wf_ids, dtype=np.int64)
        off = np.ascontiguousarray(prefix_off, dtype=np.int64)
        pre = np.ascontiguousarray(prefix if len(prefix) else [0], dtype=np.int32)
        out = np.zeros((w.size, K, V1), dtype=np.float64) if want_probs else None
        if x_device_ptr is not None:
            xp, on_dev = C.c_void_p(int(x_device_ptr)), 1
        else:
            xa = np.ascontiguousarray(x, dtype=np.uint16)
            if xa.shape != (w.size, H):
                raise ValueError("x must be [n_workflows, text_dim] bf16 bits")
            xp, on_dev = C.c_void_p(xa.ctypes.data), 0
        self._c(_abi.lib().pbkv_predict(self._h, ptr(w, C.c_int64), int(w.size), ptr(off, C.c_int64),
                                        ptr(pre, C.c_int32), xp, on_dev,
                                        ptr(out, C.c_double) if out is not None else ptr(None, C.c_double)))
        return out

    # ---- stage 2 -------------------------------------------------------------------
    def score_all(self) -> np.ndarray:
        out = np.zeros(self.n_nodes, dtype=np.float64)
        self._c(_abi.lib().pbkv_score_all(self._h, ptr(out, C.c_double)))
        return out

    def score_nodes(self, ids: Sequence[int]) -> np.ndarray:
        i = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(i.size, dtype=np.float64)
        self._c(_abi.lib().pbkv_score_nodes(self._h, ptr(i, C.c_int32), int(i.size), ptr(out, C.c_double)))
        return out

    def value_nodes(self, ids: Sequence[int]) -> np.ndarray:
        i = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(i.size, dtype=np.float64)
        self._c(_abi.lib().pbkv_value_nodes(self._h, ptr(i, C.c_int32), int(i.size), ptr(out, C.c_double)))
        return out

    # ---- stage 3 -------------------------------------------------------------------
    def select_victims(self, policy: int, needed: int, remaining: Mapping[int, Sequence[int]] | None = None,
                       locked: Iterable[int] = (), score_mode: int = SCORE_CACHED) -> VictimSelection:
        """policies.hpp:155-168"""
        if policy == POLICY_KVFLOW:
            if remaining is None:
                raise ValidationError("kvflow selected without static sequences")
            self.set_remaining(remaining)
        if isinstance(locked, np.ndarray):  # fast path: any order, duplicates allowed by the C ABI
            lk = np.ascontiguousarray(locked, dtype=np.int32)
            n_lk = int(lk.size)
            if n_lk == 0:
                lk = np.zeros(1, dtype=np.int32)
        else:
            lk_list = sorted(set(int(x) for x in locked))
            lk = np.ascontiguousarray(lk_list or [0], dtype=np.int32)
            n_lk = len(lk_list)
        cap = max(self.n_nodes, 1)
        victims = getattr(self, "_vbuf", None)
        if victims is None or victims.size < cap:
            victims = self._vbuf = np.empty(cap, dtype=np.int32)
        nv, fr, sf = C.c_int64(), C.c_int64(), C.c_int()
        self._c(_abi.lib().pbkv_select(self._h, int(policy), int(score_mode), int(needed), ptr(lk, C.c_int32), n_lk,
                                       ptr(victims, C.c_int32), cap, C.byref(nv), C.byref(fr), C.byref(sf)))
        return VictimSelection(victims[: nv.value].copy(), int(fr.value), bool(sf.value))

    def select_dev(self, policy: int, score_mode: int, needed: int, locked_ptr: int, n_locked: int,
                   victims_ptr: int, cap: int, result_ptr: int) -> None:
        """pbkv_select_dev: device-resident inputs/outputs (raw device pointers,
        e.g. torch tensor data_ptr()); result_ptr -> int64[3] {n_victims, freed, shortfall}."""
        self._c(_abi.lib().pbkv_select_dev(self._h, int(policy), int(score_mode), int(needed),
                                           C.c_void_p(locked_ptr or None), int(n_locked),
                                           C.c_void_p(victims_ptr or None), int(cap), C.c_void_p(result_ptr)))

    def select_victims_lru(self, needed: int, locked: Iterable[int] = ()) -> VictimSelection:
        return self.select_victims(POLICY_LRU, needed, locked=locked)

    def select_victims_lae(self, needed: int, locked: Iterable[int] = ()) -> VictimSelection:
        return self.select_victims(POLICY_LAE, needed, locked=locked)

    def select_victims_hierarchical(self, needed: int, locked: Iterable[int] = (),
                                    score_mode: int = SCORE_CACHED) -> VictimSelection:
        return self.select_victims(POLICY_HE, needed, locked=locked, score_mode=score_mode)

    def select_victims_kvflow(self, needed: int, remaining: Mapping[int, Sequence[int]],
                              locked: Iterable[int] = ()) -> VictimSelection:
        return self.select_victims(POLICY_KVFLOW, needed, remaining=remaining, locked=locked)

    # ---- stage 4 -------------------------------------------------------------------
    def _plan(self, bandwidth: int, step_duration: int, rho: float) -> PrefetchPlan:
        L = _abi.lib()
        pl = _abi.PrefetchPlanC()
        self._c(L.pbkv_plan_prefetch(self._h, int(bandwidth), int(step_duration), float(rho), None, None, 0, None, 0,
                                     C.byref(pl)))
        nc, ns = pl.n_candidates, pl.n_selected
        cid = np.empty(nc, dtype=np.int32)
        cv = np.empty(nc, dtype=np.float64)
        sel = np.empty(ns, dtype=np.int32)
        self._c(L.pbkv_plan_fetch(self._h, ptr(cid, C.c_int32), ptr(cv, C.c_double), nc, ptr(sel, C.c_int32), ns))
        return PrefetchPlan.from_arrays(cid, cv, sel, pl.budget_space, pl.budget_bw, pl.displacement_budget,
                                        pl.selected_tokens)

    def prefetch_round(self, selected: Sequence[int], device_free: int) -> tuple[list[int], list[list[int]]]:
        """One conservative prefetch round (simulator.hpp:632-681) as one device
        decision: (promoted flags, victims demoted before each candidate)."""
        sel = np.ascontiguousarray(np.asarray(selected, dtype=np.int32))
        n = int(sel.size)
        prom = np.empty(max(n, 1), dtype=np.int32)
        vend = np.empty(max(n, 1), dtype=np.int64)
        cap = max(int(self.n_nodes), 1)
        vict = np.empty(cap, dtype=np.int32)
        nv = C.c_int64()
        self._c(_abi.lib().pbkv_prefetch_round(self._h, ptr(sel, C.c_int32), n, int(device_free), ptr(prom, C.c_int32),
                                                ptr(vend, C.c_int64), ptr(vict, C.c_int32), cap, C.byref(nv)))
        return prom[:n].tolist(), RoundVictims(vict[: nv.value].copy(), vend[:n].copy())

    def plan_conservative_prefetch(self, bandwidth: int, step_duration: int = 1) -> PrefetchPlan:
        """policies.hpp:220-224"""
        return self._plan(bandwidth, step_duration, -1.0)

    def plan_aggressive_prefetch(self, bandwidth: int, rho: float, step_duration: int = 1) -> PrefetchPlan:
        """policies.hpp:228-235"""
        if not (0.0 <= rho <= 1.0):
            raise ValidationError("rho must be in [0, 1]")
        return self._plan(bandwidth, step_duration, rho)

    # ---- timing ------------------------------------------------------------------------
    def set_timing(self, on: bool) -> None:
        self._c(_abi.lib().pbkv_ctx_set_timing(self._h, 1 if on else 0))

    def kernel_timings(self) -> list[float]:
        """[light Eq. 2 pass ms, persistent selection kernel ms] of the last timed call."""
        ms = (C.c_float * 2)()
        self._c(_abi.lib().pbkv_ctx_kernel_timings(self._h, ms))
        return [float(x) for x in ms]

    def set_defer(self, on: bool) -> None:
        """Heavy-node deferral in RECOMPUTE decisions (results identical)."""
        self._c(_abi.lib().pbkv_ctx_set_defer(self._h, 1 if on else 0))

    def defer_stats(self) -> tuple[int, int]:
        f, s = C.c_int64(), C.c_int64()
        self._c(_abi.lib().pbkv_ctx_defer_stats(self._h, C.byref(f), C.byref(s)))
        return f.value, s.value

    def launches(self) -> tuple[int, int]:
        """(pbkv kernels launched, CUB library calls) since the context was created."""
        k, l = C.c_int64(), C.c_int64()
        self._c(_abi.lib().pbkv_ctx_launches(self._h, C.byref(k), C.byref(l)))
        return k.value, l.value

    def phase_times_us(self) -> list[float]:
        """Durations between the selection kernel's phase stamps (microseconds)."""
        buf = (C.c_uint64 * 32)()
        n = C.c_int()
        self._c(_abi.lib().pbkv_ctx_phase_times(self._h, buf, 32, C.byref(n)))
        ts = list(buf)[: min(n.value, 32)]
        return [(b - a) / 1000.0 for a, b in zip(ts, ts[1:])]

    def stream_handle(self) -> int:
        s = C.c_void_p()
        self._c(_abi.lib().pbkv_ctx_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def timings(self) -> list[float]:
        ms = (C.c_float * 5)()
        self._c(_abi.lib().pbkv_ctx_timings(self._h, ms))
        return list(ms)


def device_count() -> int:
    n = C.c_int()
    _check(_abi.lib().pbkv_device_count(C.byref(n)), None)
    return n.value
