"""B200-native PBKV scoring / victim-selection hot path (arXiv 2605.06472).

Drop-in GPU backend for the reference flowkv policy interface
(/root/reference/proj/include/flowkv/{scoring,policies}.hpp): Eq. 2 scoring,
hierarchical victim selection and conservative-prefetch ranking as sm_100a
kernels behind the C ABI in include/pbkv.h.  See DESIGN.md.
"""
from ._abi import (POLICY_HE, POLICY_KVFLOW, POLICY_LAE, POLICY_LRU, SCORE_CACHED, SCORE_RECOMPUTE,
                   TIER_ABSENT, TIER_DEVICE, TIER_HOST, SoAArrays, synth_params)

__all__ = [
    "POLICY_HE", "POLICY_KVFLOW", "POLICY_LAE", "POLICY_LRU", "SCORE_CACHED", "SCORE_RECOMPUTE",
    "TIER_ABSENT", "TIER_DEVICE", "TIER_HOST", "SoAArrays", "synth_params",
]
