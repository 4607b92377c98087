"""ctypes loaders for the TEST-ONLY checkers (never imported by the product).

* ``Oracle``  -- the C restatement (oracle/pbkv_oracle.c -> _build/libpbkv_oracle.so)
* ``RefTree`` -- the reference itself: a real flowkv::CacheTree plus the
  reference policy functions, compiled from /root/reference headers into
  _ref/libflowkv_ref.so (oracle/ref_capi.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from dataclasses import dataclass, field
from typing import Iterable, Mapping, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2605_06472_b200._abi import PrefetchPlanC, SoAArrays, TreeSoA, ptr, synth_params  # noqa: E402

ORACLE_LIB = os.path.join(HERE, "_build", "libpbkv_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libflowkv_ref.so")


class OracleError(RuntimeError):
    """A ValidationError raised by the checker (message kept verbatim)."""


@dataclass
class Selection:
    victims: list[int] = field(default_factory=list)
    freed: int = 0
    shortfall: bool = False


@dataclass
class Plan:
    candidates: list[tuple[int, float]] = field(default_factory=list)
    budget_space: int = 0
    budget_bw: int = 0
    displacement_budget: int = 0
    selected: list[int] = field(default_factory=list)
    selected_tokens: int = 0


_i32p, _i64p, _f64p = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_double)
_soap = C.POINTER(TreeSoA)

_olib = None
_rlib = None


def have_oracle() -> bool:
    return os.path.exists(ORACLE_LIB)


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def _oracle():
    global _olib
    if _olib is None:
        L = C.CDLL(ORACLE_LIB)
        L.orc_last_error.restype = C.c_char_p
        L.orc_score_nodes.argtypes = [_soap, _i64p, C.c_int64, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, _i32p,
                                      C.c_int64, _f64p]
        L.orc_value_nodes.argtypes = [_soap, _i64p, C.c_int64, C.c_int, C.c_int, _f64p, _i32p, C.c_int64, _f64p]
        L.orc_select.argtypes = [_soap, C.c_int, C.c_int64, _i32p, C.c_int64, _i64p, C.c_int64, _i64p, _i32p,
                                 _i32p, C.c_int64, _i64p, _i64p, C.POINTER(C.c_int)]
        L.orc_plan_prefetch.argtypes = [_soap, _i64p, C.c_int64, C.c_int, C.c_int, _f64p, C.c_int64, C.c_int,
                                        C.c_double, _i32p, _f64p, C.c_int64, _i32p, C.c_int64,
                                        C.POINTER(PrefetchPlanC)]
        _olib = L
    return _olib


def _sorted_forecasts(wf: Sequence[int], P: np.ndarray):
    wf = np.asarray(wf, dtype=np.int64)
    order = np.argsort(wf, kind="stable")
    return np.ascontiguousarray(wf[order]), np.ascontiguousarray(np.asarray(P, dtype=np.float64)[order])


def _rem_csr(remaining: Mapping[int, Sequence[int]] | None):
    if remaining is None:
        return None, 0, None, None
    wf = np.array(sorted(remaining), dtype=np.int64)
    off = np.zeros(wf.size + 1, dtype=np.int64)
    flat: list[int] = []
    for i, w in enumerate(wf.tolist()):
        flat.extend(int(a) for a in remaining[w])
        off[i + 1] = len(flat)
    return wf, wf.size, off, np.array(flat or [0], dtype=np.int32)


class Oracle:
    """C restatement of scoring.hpp / policies.hpp on a SoA snapshot."""

    @staticmethod
    def score_nodes(soa: SoAArrays, wf, P, K: int, gamma: float, ids=None) -> np.ndarray:
        L = _oracle()
        fw, fp = _sorted_forecasts(wf, P)
        s = soa.struct()
        idv = None if ids is None else np.ascontiguousarray(ids, dtype=np.int32)
        n = soa.n_nodes if ids is None else idv.size
        out = np.zeros(max(n, 1), dtype=np.float64)
        rc = L.orc_score_nodes(C.byref(s), ptr(fw, C.c_int64), fw.size, fp.shape[1] if fp.ndim == 3 else 1,
                               fp.shape[2] if fp.ndim == 3 else 2, ptr(fp, C.c_double), K, gamma,
                               ptr(idv, C.c_int32), n, ptr(out, C.c_double))
        if rc:
            raise OracleError(L.orc_last_error().decode())
        return out[:n]

    @staticmethod
    def value_nodes(soa: SoAArrays, wf, P, ids) -> np.ndarray:
        L = _oracle()
        fw, fp = _sorted_forecasts(wf, P)
        s = soa.struct()
        idv = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(max(idv.size, 1), dtype=np.float64)
        rc = L.orc_value_nodes(C.byref(s), ptr(fw, C.c_int64), fw.size, fp.shape[1], fp.shape[2],
                               ptr(fp, C.c_double), ptr(idv, C.c_int32), idv.size, ptr(out, C.c_double))
        if rc:
            raise OracleError(L.orc_last_error().decode())
        return out[: idv.size]

    @staticmethod
    def select(soa: SoAArrays, policy: int, needed: int, locked: Iterable[int] = (),
               remaining: Mapping[int, Sequence[int]] | None = None) -> Selection:
        L = _oracle()
        s = soa.struct()
        lk_list = sorted(set(int(x) for x in locked))
        lk = np.array(lk_list or [0], dtype=np.int32)
        rw, nr, ro, rs = _rem_csr(remaining)
        cap = max(soa.n_nodes, 1)
        v = np.zeros(cap, dtype=np.int32)
        nv, fr, sf = C.c_int64(), C.c_int64(), C.c_int()
        rc = L.orc_select(C.byref(s), policy, int(needed), ptr(lk, C.c_int32), len(lk_list), ptr(rw, C.c_int64), nr,
                          ptr(ro, C.c_int64), ptr(rs, C.c_int32), ptr(v, C.c_int32), cap, C.byref(nv), C.byref(fr),
                          C.byref(sf))
        if rc:
            raise OracleError(L.orc_last_error().decode())
        return Selection(v[: nv.value].tolist(), fr.value, bool(sf.value))

    @staticmethod
    def plan(soa: SoAArrays, wf, P, bandwidth: int, step: int = 1, rho: float = -1.0) -> Plan:
        L = _oracle()
        fw, fp = _sorted_forecasts(wf, P)
        s = soa.struct()
        cap = max(soa.n_nodes, 1)
        cid = np.zeros(cap, dtype=np.int32)
        cv = np.zeros(cap, dtype=np.float64)
        sel = np.zeros(cap, dtype=np.int32)
        pl = PrefetchPlanC()
        H = fp.shape[1] if fp.ndim == 3 and fp.shape[0] else 1
        V1 = fp.shape[2] if fp.ndim == 3 and fp.shape[0] else 2
        rc = L.orc_plan_prefetch(C.byref(s), ptr(fw, C.c_int64), fw.size, H, V1, ptr(fp, C.c_double),
                                 int(bandwidth), int(step), float(rho), ptr(cid, C.c_int32), ptr(cv, C.c_double), cap,
                                 ptr(sel, C.c_int32), cap, C.byref(pl))
        if rc:
            raise OracleError(L.orc_last_error().decode())
        nc, ns = pl.n_candidates, pl.n_selected
        return Plan(list(zip(cid[:nc].tolist(), cv[:nc].tolist())), pl.budget_space, pl.budget_bw,
                    pl.displacement_budget, sel[:ns].tolist(), pl.selected_tokens)


def _ref():
    global _rlib
    if _rlib is None:
        L = C.CDLL(REF_LIB)
        vp = C.c_void_p
        L.fkref_last_error.argtypes = [vp]
        L.fkref_last_error.restype = C.c_char_p
        L.fkref_tree_new.argtypes = [C.c_int64, C.c_int64]
        L.fkref_tree_new.restype = vp
        L.fkref_tree_free.argtypes = [vp]
        L.fkref_apply_ops.argtypes = [vp, _i64p, C.c_int64]
        L.fkref_synth.argtypes = [vp, C.c_void_p]
        L.fkref_shape.argtypes = [vp, _soap]
        L.fkref_export.argtypes = [vp, _soap]
        L.fkref_set_forecasts.argtypes = [vp, _i64p, C.c_int64, C.c_int, C.c_int, _f64p]
        L.fkref_drop_forecast.argtypes = [vp, C.c_int64]
        L.fkref_set_remaining.argtypes = [vp, _i64p, C.c_int64, _i64p, _i32p]
        L.fkref_set_score.argtypes = [vp, C.c_int32, C.c_double]
        L.fkref_refresh_scores.argtypes = [vp, C.c_int64, C.c_int, C.c_double, _i64p]
        L.fkref_refresh_nodes.argtypes = [vp, _i32p, C.c_int64, C.c_int, C.c_double]
        L.fkref_score_nodes.argtypes = [vp, _i32p, C.c_int64, C.c_int, C.c_double, _f64p]
        L.fkref_value_nodes.argtypes = [vp, _i32p, C.c_int64, _f64p]
        L.fkref_select.argtypes = [vp, C.c_int, C.c_int64, _i32p, C.c_int64, _i32p, C.c_int64, _i64p, _i64p,
                                   C.POINTER(C.c_int)]
        L.fkref_plan.argtypes = [vp, C.c_int64, C.c_int, C.c_double, _i32p, _f64p, C.c_int64, _i32p, C.c_int64,
                                 C.POINTER(PrefetchPlanC)]
        L.fkref_touched.argtypes = [vp, C.c_int64, _i32p, C.c_int64, _i64p]
        _rlib = L
    return _rlib


class RefTree:
    """A real flowkv::CacheTree driven through the reference's public API."""

    def __init__(self, device_capacity: int = 1 << 40, host_capacity: int = 1 << 40):
        self.L = _ref()
        self.h = self.L.fkref_tree_new(int(device_capacity), int(host_capacity))
        if not self.h:
            raise OracleError(self.L.fkref_last_error(None).decode())

    def __del__(self):
        try:
            if self.h:
                self.L.fkref_tree_free(self.h)
        except Exception:
            pass

    def _c(self, rc):
        if rc:
            raise OracleError(self.L.fkref_last_error(self.h).decode())

    def apply_ops(self, words):
        w = np.ascontiguousarray(np.asarray(words, dtype=np.int64))
        self._c(self.L.fkref_apply_ops(self.h, ptr(w, C.c_int64), w.size))

    def synth(self, **params):
        p = synth_params(**params)
        self._c(self.L.fkref_synth(self.h, C.cast(C.pointer(p), C.c_void_p)))

    def export(self) -> SoAArrays:
        sh = TreeSoA()
        self.L.fkref_shape(self.h, C.byref(sh))
        arr = SoAArrays(sh.n_nodes, sh.n_entries, dict(
            device_capacity=sh.device_capacity, device_used=sh.device_used,
            retired_device_tokens=sh.retired_device_tokens, host_capacity=sh.host_capacity, host_used=sh.host_used))
        s = arr.struct()
        self.L.fkref_export(self.h, C.byref(s))
        return arr

    def set_forecasts(self, wf, P):
        w = np.ascontiguousarray(wf, dtype=np.int64)
        p = np.ascontiguousarray(P, dtype=np.float64)
        self._c(self.L.fkref_set_forecasts(self.h, ptr(w, C.c_int64), w.size, p.shape[1], p.shape[2],
                                           ptr(p, C.c_double)))

    def drop_forecast(self, w):
        self.L.fkref_drop_forecast(self.h, int(w))

    def set_remaining(self, remaining):
        rw, nr, ro, rs = _rem_csr(remaining)
        self.L.fkref_set_remaining(self.h, ptr(rw, C.c_int64), nr, ptr(ro, C.c_int64), ptr(rs, C.c_int32))

    def set_score(self, node, s):
        self.L.fkref_set_score(self.h, int(node), float(s))

    def refresh_scores(self, w, k, gamma) -> int:
        n = C.c_int64()
        self._c(self.L.fkref_refresh_scores(self.h, int(w), int(k), float(gamma), C.byref(n)))
        return n.value

    def refresh_nodes(self, ids, k, gamma):
        idv = None if ids is None else np.ascontiguousarray(ids, dtype=np.int32)
        self._c(self.L.fkref_refresh_nodes(self.h, ptr(idv, C.c_int32), 0 if idv is None else idv.size, int(k),
                                           float(gamma)))

    def score_nodes(self, ids, k, gamma) -> np.ndarray:
        idv = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(max(idv.size, 1), dtype=np.float64)
        self._c(self.L.fkref_score_nodes(self.h, ptr(idv, C.c_int32), idv.size, int(k), float(gamma),
                                         ptr(out, C.c_double)))
        return out[: idv.size]

    def value_nodes(self, ids) -> np.ndarray:
        idv = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.zeros(max(idv.size, 1), dtype=np.float64)
        self._c(self.L.fkref_value_nodes(self.h, ptr(idv, C.c_int32), idv.size, ptr(out, C.c_double)))
        return out[: idv.size]

    def select(self, policy, needed, locked=()) -> Selection:
        lk_list = sorted(set(int(x) for x in locked))
        lk = np.array(lk_list or [0], dtype=np.int32)
        sh = TreeSoA()
        self.L.fkref_shape(self.h, C.byref(sh))
        cap = max(sh.n_nodes, 1)
        v = np.zeros(cap, dtype=np.int32)
        nv, fr, sf = C.c_int64(), C.c_int64(), C.c_int()
        self._c(self.L.fkref_select(self.h, int(policy), int(needed), ptr(lk, C.c_int32), len(lk_list),
                                    ptr(v, C.c_int32), cap, C.byref(nv), C.byref(fr), C.byref(sf)))
        return Selection(v[: nv.value].tolist(), fr.value, bool(sf.value))

    def plan(self, bandwidth, step=1, rho=-1.0) -> Plan:
        sh = TreeSoA()
        self.L.fkref_shape(self.h, C.byref(sh))
        cap = max(sh.n_nodes, 1)
        cid = np.zeros(cap, dtype=np.int32)
        cv = np.zeros(cap, dtype=np.float64)
        sel = np.zeros(cap, dtype=np.int32)
        pl = PrefetchPlanC()
        self._c(self.L.fkref_plan(self.h, int(bandwidth), int(step), float(rho), ptr(cid, C.c_int32),
                                  ptr(cv, C.c_double), cap, ptr(sel, C.c_int32), cap, C.byref(pl)))
        nc, ns = pl.n_candidates, pl.n_selected
        return Plan(list(zip(cid[:nc].tolist(), cv[:nc].tolist())), pl.budget_space, pl.budget_bw,
                    pl.displacement_budget, sel[:ns].tolist(), pl.selected_tokens)

    def touched(self, w) -> list[int]:
        n = C.c_int64()
        self.L.fkref_touched(self.h, int(w), None, 0, C.byref(n))
        ids = np.zeros(max(n.value, 1), dtype=np.int32)
        self.L.fkref_touched(self.h, int(w), ptr(ids, C.c_int32), n.value, C.byref(n))
        return ids[: n.value].tolist()
