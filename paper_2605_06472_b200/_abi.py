"""ctypes view of the C ABI in include/pbkv.h (structs + library loader).

The library is the in-tree ``libpbkv.so`` built by ``build.py``; there is no
fallback -- if it is missing, importing the package's API raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBKV_LIB") or os.path.join(PKG, "libpbkv.so")  # PBKV_LIB: variant builds (tools)

PBKV_OK, PBKV_EINVAL, PBKV_ECUDA, PBKV_ENOMEM, PBKV_EARG = 0, 1, 2, 3, 4
TIER_DEVICE, TIER_HOST, TIER_ABSENT = 0, 1, 2
POLICY_LRU, POLICY_LAE, POLICY_HE, POLICY_KVFLOW = 0, 1, 2, 3
SCORE_CACHED, SCORE_RECOMPUTE = 0, 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)


class Cfg(C.Structure):
    _fields_ = [("device", C.c_int), ("k", C.c_int), ("gamma", C.c_double), ("num_agents", C.c_int)]


class TreeSoA(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("n_entries", C.c_int64),
        ("parent", _i32p),
        ("len", _i32p),
        ("tier", _u8p),
        ("retired", _u8p),
        ("last_access", _u64p),
        ("ever_tagged", _i32p),
        ("score", _f64p),
        ("device_children", _i32p),
        ("depth", _i32p),
        ("acc_off", _i64p),
        ("acc_wf", _i64p),
        ("acc_bits", _u64p),
        ("device_capacity", C.c_int64),
        ("device_used", C.c_int64),
        ("retired_device_tokens", C.c_int64),
        ("host_capacity", C.c_int64),
        ("host_used", C.c_int64),
    ]


class NodeDelta(C.Structure):
    """pbkv_node_delta"""
    _fields_ = [("id", C.c_int32), ("parent", C.c_int32), ("len", C.c_int32), ("ever_tagged", C.c_int32),
                ("depth", C.c_int32), ("tier", C.c_uint8), ("retired", C.c_uint8), ("pad", C.c_uint8 * 2),
                ("last_access", C.c_uint64), ("score", C.c_double), ("acc_begin", C.c_int64),
                ("acc_end", C.c_int64)]


NODE_DELTA_DTYPE = np.dtype([("id", np.int32), ("parent", np.int32), ("len", np.int32), ("ever_tagged", np.int32),
                             ("depth", np.int32), ("tier", np.uint8), ("retired", np.uint8), ("pad", np.uint8, 2),
                             ("last_access", np.uint64), ("score", np.float64), ("acc_begin", np.int64),
                             ("acc_end", np.int64)], align=True)


class TreeTotals(C.Structure):
    """pbkv_tree_totals"""
    _fields_ = [("device_capacity", C.c_int64), ("device_used", C.c_int64), ("retired_device_tokens", C.c_int64),
                ("host_capacity", C.c_int64), ("host_used", C.c_int64)]


class PrefetchPlanC(C.Structure):
    _fields_ = [
        ("budget_space", C.c_int64),
        ("budget_bw", C.c_int64),
        ("displacement_budget", C.c_int64),
        ("selected_tokens", C.c_int64),
        ("n_candidates", C.c_int64),
        ("n_selected", C.c_int64),
    ]


class SynthParams(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64),
        ("n_workflows", C.c_int64),
        ("agents", C.c_int),
        ("group_size", C.c_int),
        ("shared_len", C.c_int),
        ("group_len", C.c_int),
        ("alphabet", C.c_int),
        ("max_rand_len", C.c_int),
        ("retired_frac", C.c_double),
        ("host_every", C.c_int),
        ("seed", C.c_uint64),
    ]


class PredictorCfg(C.Structure):
    """pbkv_predictor_cfg"""
    _fields_ = [("num_agents", C.c_int), ("horizon", C.c_int), ("dim", C.c_int), ("hidden", C.c_int),
                ("text_dim", C.c_int), ("max_prefix", C.c_int)]


class PredictorWeights(C.Structure):
    """pbkv_predictor_weights"""
    _fields_ = [("embed", C.POINTER(C.c_float)), ("transition", C.POINTER(C.c_float)),
                ("sage1", C.POINTER(C.c_float)), ("sage2", C.POINTER(C.c_float)),
                ("query", C.POINTER(C.c_float)), ("text", C.POINTER(C.c_uint16)),
                ("mlp1", C.POINTER(C.c_float)), ("mlp1_bias", C.POINTER(C.c_float)),
                ("mlp2", C.POINTER(C.c_float)), ("mlp2_bias", C.POINTER(C.c_float))]


def synth_params(n_nodes=10000, n_workflows=256, agents=16, group_size=16, shared_len=32, group_len=8,
                 alphabet=4, max_rand_len=10, retired_frac=0.3, host_every=10, seed=12345) -> SynthParams:
    """SURVEY.md §8(d) synthetic workload (generator: csrc/host/ops.hpp)."""
    return SynthParams(n_nodes, n_workflows, agents, group_size, shared_len, group_len, alphabet,
                       max_rand_len, retired_frac, host_every, seed)


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C ABI must be contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


class SoAArrays:
    """numpy storage behind a TreeSoA struct (the CacheTree read-side image)."""

    FIELDS = {
        "parent": np.int32, "len": np.int32, "tier": np.uint8, "retired": np.uint8,
        "last_access": np.uint64, "ever_tagged": np.int32, "score": np.float64,
        "device_children": np.int32, "depth": np.int32,
    }

    def __init__(self, n_nodes: int, n_entries: int, scalars: dict | None = None):
        self.n_nodes, self.n_entries = int(n_nodes), int(n_entries)
        for f, dt in self.FIELDS.items():
            setattr(self, f, np.zeros(self.n_nodes, dtype=dt))
        self.acc_off = np.zeros(self.n_nodes + 1, dtype=np.int64)
        self.acc_wf = np.zeros(max(self.n_entries, 1), dtype=np.int64)
        self.acc_bits = np.zeros(max(self.n_entries, 1), dtype=np.uint64)
        self.scalars = dict(device_capacity=0, device_used=0, retired_device_tokens=0, host_capacity=0,
                            host_used=0)
        if scalars:
            self.scalars.update(scalars)

    def struct(self, with_depth=True) -> TreeSoA:
        s = TreeSoA()
        s.n_nodes, s.n_entries = self.n_nodes, self.n_entries
        s.parent = ptr(self.parent, C.c_int32)
        s.len = ptr(self.len, C.c_int32)
        s.tier = ptr(self.tier, C.c_uint8)
        s.retired = ptr(self.retired, C.c_uint8)
        s.last_access = ptr(self.last_access, C.c_uint64)
        s.ever_tagged = ptr(self.ever_tagged, C.c_int32)
        s.score = ptr(self.score, C.c_double)
        s.device_children = ptr(self.device_children, C.c_int32)
        s.depth = ptr(self.depth if with_depth else None, C.c_int32)
        s.acc_off = ptr(self.acc_off, C.c_int64)
        s.acc_wf = ptr(self.acc_wf, C.c_int64)
        s.acc_bits = ptr(self.acc_bits, C.c_uint64)
        for k, v in self.scalars.items():
            setattr(s, k, int(v))
        return s

    def copy(self) -> "SoAArrays":
        o = SoAArrays(self.n_nodes, self.n_entries, dict(self.scalars))
        for f in list(self.FIELDS) + ["acc_off", "acc_wf", "acc_bits"]:
            setattr(o, f, getattr(self, f).copy())
        return o

    def entries_of(self, i: int):
        a, b = int(self.acc_off[i]), int(self.acc_off[i + 1])
        return list(zip(self.acc_wf[a:b].tolist(), self.acc_bits[a:b].tolist()))


_lib = None


def lib() -> C.CDLL:
    """Load libpbkv.so (fails loudly: the product has no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libpbkv.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    sig = {
        "pbkv_abi_version": ([], C.c_int),
        "pbkv_last_error": ([vp], C.c_char_p),
        "pbkv_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "pbkv_ctx_create": ([C.POINTER(vp), C.POINTER(Cfg)], C.c_int),
        "pbkv_ctx_destroy": ([vp], C.c_int),
        "pbkv_ctx_sync": ([vp], C.c_int),
        "pbkv_ctx_stream": ([vp, C.POINTER(vp)], C.c_int),
        "pbkv_ctx_timings": ([vp, C.POINTER(C.c_float)], C.c_int),
        "pbkv_ctx_set_timing": ([vp, C.c_int], C.c_int),
        "pbkv_ctx_launches": ([vp, _i64p, _i64p], C.c_int),
        "pbkv_ctx_set_defer": ([vp, C.c_int], C.c_int),
        "pbkv_ctx_kernel_timings": ([vp, C.POINTER(C.c_float)], C.c_int),
        "pbkv_ctx_defer_stats": ([vp, _i64p, _i64p], C.c_int),
        "pbkv_ctx_phase_times": ([vp, _u64p, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "pbkv_mirror_full": ([vp, C.POINTER(TreeSoA)], C.c_int),
        "pbkv_mirror_tree": ([vp, vp], C.c_int),
        "pbkv_mirror_sync": ([vp, vp], C.c_int),
        "pbkv_mirror_delta": ([vp, vp, C.c_int64, _i64p, _u64p, C.POINTER(TreeTotals)], C.c_int),
        "pbkv_mirror_verify": ([vp, C.POINTER(TreeSoA), _i64p], C.c_int),
        "pbkv_mirror_set_scores": ([vp, _i32p, _f64p, C.c_int64], C.c_int),
        "pbkv_mirror_node_count": ([vp, _i64p, _i64p], C.c_int),
        "pbkv_forecast_put": ([vp, _i64p, C.c_int64, C.c_int, C.c_int, _f64p], C.c_int),
        "pbkv_forecast_put_async": ([vp, _i64p, C.c_int64, C.c_int, C.c_int, _f64p], C.c_int),
        "pbkv_forecast_drop": ([vp, _i64p, C.c_int64], C.c_int),
        "pbkv_forecast_clear": ([vp], C.c_int),
        "pbkv_score_all": ([vp, _f64p], C.c_int),
        "pbkv_score_nodes": ([vp, _i32p, C.c_int64, _f64p], C.c_int),
        "pbkv_value_nodes": ([vp, _i32p, C.c_int64, _f64p], C.c_int),
        "pbkv_select": ([vp, C.c_int, C.c_int, C.c_int64, _i32p, C.c_int64, _i32p, C.c_int64, _i64p, _i64p,
                         C.POINTER(C.c_int)], C.c_int),
        "pbkv_select_dev": ([vp, C.c_int, C.c_int, C.c_int64, vp, C.c_int64, vp, C.c_int64, vp], C.c_int),
        "pbkv_set_remaining": ([vp, _i64p, C.c_int64, _i64p, _i32p], C.c_int),
        "pbkv_plan_prefetch": ([vp, C.c_int64, C.c_int, C.c_double, _i32p, _f64p, C.c_int64, _i32p, C.c_int64,
                                C.POINTER(PrefetchPlanC)], C.c_int),
        "pbkv_ctx_wait_stream": ([vp, vp], C.c_int),
        "pbkv_prefetch_round": ([vp, _i32p, C.c_int64, C.c_int64, _i32p, _i64p, _i32p, C.c_int64, _i64p], C.c_int),
        "pbkv_plan_fetch": ([vp, _i32p, _f64p, C.c_int64, _i32p, C.c_int64], C.c_int),
        "pbkv_interval_sums": ([vp, vp, _i64p, _i64p, C.c_int, _f64p], C.c_int),
        "pbkv_predictor_load": ([vp, C.POINTER(PredictorCfg), C.POINTER(PredictorWeights)], C.c_int),
        "pbkv_predict": ([vp, _i64p, C.c_int64, _i64p, _i32p, vp, C.c_int, _f64p], C.c_int),
        "pbkv_tree_create": ([C.POINTER(vp), C.c_int64, C.c_int64], C.c_int),
        "pbkv_tree_destroy": ([vp], C.c_int),
        "pbkv_tree_apply_ops": ([vp, _i64p, C.c_int64], C.c_int),
        "pbkv_tree_synth": ([vp, C.POINTER(SynthParams)], C.c_int),
        "pbkv_tree_shape": ([vp, C.POINTER(TreeSoA)], C.c_int),
        "pbkv_tree_export": ([vp, C.POINTER(TreeSoA)], C.c_int),
        "pbkv_tree_touched": ([vp, C.c_int64, _i32p, C.c_int64, _i64p], C.c_int),
        "pbkv_tree_log": ([vp, C.c_int64, _i64p, _i32p, C.c_int64, _i64p], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Every function name include/pbkv.h declares (parsed from the header)."""
    import re

    hdr = os.path.join(os.path.dirname(PKG), "include", "pbkv.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(pbkv_\w+)\s*\(", src, re.M)))
