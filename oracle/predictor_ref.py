"""FP64 CPU restatement of the stage-1 predictor (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED: the reference has no predictor code or weights (SPEC.md:8,
:163 put the neural predictor out of scope); this follows PAPER.md equation
by equation and is the checker for the GPU forward under a stated tolerance
(tests/test_predictor.py), not a bit-exact oracle.

  H^(l) = ReLU([H^(l-1) | A H^(l-1)] W^(l)T), l = 1, 2
  h_cur = H2[v_t]; a_i = softmax_{i<t}((W_q h_cur)^T H2[v_i] / sqrt(d))
  h_path = sum_{i<t} a_i H2[v_i]
  h_txt = ReLU(W_t x)
  two-layer MLP over [h_cur | h_path | h_txt] -> K x (A+1) logits,
  per-step softmax, END a regular class

Inputs are the exact values the GPU sees (bf16 x and W_t decoded to float).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def graph_tables(w):
    """H2 [A][d] and the attention logits table QK[u][v] / sqrt(d)."""
    H = w.embed.astype(np.float64)
    A = w.transition.astype(np.float64)
    for W in (w.sage1, w.sage2):
        H = np.maximum(np.concatenate([H, A @ H], axis=1) @ W.astype(np.float64).T, 0.0)
    Q = H @ w.query.astype(np.float64).T
    return H, (Q @ H.T) / np.sqrt(w.dim)


def forward(w, prefix_off: np.ndarray, prefix: np.ndarray, x_bits: np.ndarray) -> np.ndarray:
    """[n, K, A+1] float64 step distributions."""
    H2, QK = graph_tables(w)
    n = len(prefix_off) - 1
    d, K, V1 = w.dim, w.horizon, w.num_agents + 1
    htxt = np.maximum(bf16_to_f64(x_bits) @ bf16_to_f64(w.text).T, 0.0)
    z = np.zeros((n, 3 * d))
    for i in range(n):
        p = prefix[prefix_off[i]:prefix_off[i + 1]]
        cur = int(p[-1])
        z[i, :d] = H2[cur]
        if len(p) > 1:
            s = QK[cur, p[:-1]]
            a = np.exp(s - s.max())
            a /= a.sum()
            z[i, d:2 * d] = a @ H2[p[:-1]]
        z[i, 2 * d:] = htxt[i]
    hid = np.maximum(z @ w.mlp1.astype(np.float64).T + w.mlp1_bias, 0.0)
    logits = (hid @ w.mlp2.astype(np.float64).T + w.mlp2_bias).reshape(n, K, V1)
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    return e / e.sum(axis=2, keepdims=True)
