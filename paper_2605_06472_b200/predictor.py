"""Stage-1 predictor weights and their random init.

The reference ships no predictor code or checkpoint; the
architecture follows the paper: GraphSAGE x2 over the row-normalised agent
transition matrix, dot-product attention over the prefix, h_txt = ReLU(W_t x),
a two-layer MLP emitting K x (A+1) logits, per-step softmax with END as a
regular class.  With d = 64, h1 = 128, H = 5120, A = 16, K = 8 the model has
~0.37 M parameters ("roughly 350K").
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit patterns, round to nearest even."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


@dataclass
class PredictorWeights:
    num_agents: int
    horizon: int
    dim: int
    hidden: int
    text_dim: int
    embed: np.ndarray       # [A][d] f32
    transition: np.ndarray  # [A][A] f32, rows sum to 1
    sage1: np.ndarray       # [d][2d]
    sage2: np.ndarray       # [d][2d]
    query: np.ndarray       # [d][d]
    text: np.ndarray        # [d][H] bf16 bits (uint16)
    mlp1: np.ndarray        # [h1][3d]
    mlp1_bias: np.ndarray   # [h1]
    mlp2: np.ndarray        # [K*(A+1)][h1]
    mlp2_bias: np.ndarray   # [K*(A+1)]

    @property
    def n_params(self) -> int:
        return sum(int(getattr(self, f).size) for f in
                   ("embed", "sage1", "sage2", "query", "text", "mlp1", "mlp1_bias", "mlp2", "mlp2_bias"))

    @staticmethod
    def random(num_agents: int = 16, horizon: int = 8, dim: int = 64, hidden: int = 128, text_dim: int = 5120,
               seed: int = 7) -> "PredictorWeights":
        rng = np.random.default_rng(seed)
        A, d, h1, H, KV = num_agents, dim, hidden, text_dim, horizon * (num_agents + 1)

        def lin(o, i):
            return (rng.standard_normal((o, i)) / np.sqrt(i)).astype(np.float32)

        counts = rng.random((A, A)) * (rng.random((A, A)) < 0.4) + np.eye(A)[rng.permutation(A)] * 0.5
        trans = (counts / counts.sum(axis=1, keepdims=True)).astype(np.float32)
        return PredictorWeights(
            A, horizon, d, h1, H,
            embed=rng.standard_normal((A, d)).astype(np.float32),
            transition=trans,
            sage1=lin(d, 2 * d), sage2=lin(d, 2 * d), query=lin(d, d),
            text=to_bf16_bits(lin(d, H)),
            mlp1=lin(h1, 3 * d), mlp1_bias=(0.1 * rng.standard_normal(h1)).astype(np.float32),
            mlp2=(2.0 * lin(KV, h1)), mlp2_bias=(0.1 * rng.standard_normal(KV)).astype(np.float32))


def random_inputs(n: int, num_agents: int, text_dim: int, max_prefix: int = 64, seed: int = 11):
    """Synthetic workflow states: prefixes (current agent last) and prefill
    hidden states x (bf16 bits, unit-variance)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_prefix + 1, size=n)
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    prefix = rng.integers(0, num_agents, size=int(off[-1])).astype(np.int32)
    x = to_bf16_bits(rng.standard_normal((n, text_dim)).astype(np.float32))
    return off, prefix, x
